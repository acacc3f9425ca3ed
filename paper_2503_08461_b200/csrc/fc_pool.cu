// fc_pool.cu -- C ABI of the FastCache B200 pool: state machine, byte
// accounting and the device-resident block allocator (K6).
//
// Byte accounting and handle states restate the reference KVCachePool
// (reference pkg/src/kvservesim/pool.py:87-257): strict admission, one-step
// pooled transition, legacy zombie retention, DoubleFree / InvalidState.
//
// Device allocator: the free list is a LIFO stack of block ids in HBM
// (d_stack) and every handle owns a row of the block-table matrix (d_table).
// All pops and pushes run on the GPU (pop_blocks_kernel / push_blocks_kernel).
// Because every operation's block COUNT is known on the host (it follows from
// token counts alone), the host mirrors only the stack pointer; the block ids
// themselves never leave the device. Batched pops walk the stack in batch
// order and pushes append in request order, ascending logical block, so block
// tables are a deterministic function of the call sequence (oracle/blocks.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "fc_internal.cuh"

namespace fc {

static thread_local char g_err[512] = "";
static thread_local int64_t g_launches = 0;
static thread_local int64_t g_paths[kNumPaths] = {0, 0, 0};

void note_launch() { ++g_launches; }
void note_path(int path) { ++g_paths[path]; }
int64_t path_count(int path) { return g_paths[path]; }

int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
      sms = 148;
    cache[dev] = sms;
  }
  return cache[dev];
}

fc_status set_error(fc_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

fc_status cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return FC_OK;
  return set_error(FC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// allocator kernels
// ---------------------------------------------------------------------------

// Pop: request i's logical block (from + j) <- stack[top - 1 - (off_i + j)].
// With save_raw (legacy compress) the live row is first copied to the
// retained row, then overwritten with fresh blocks.
__global__ void pop_blocks_kernel(int32_t* __restrict__ table, int32_t* __restrict__ rtable,
                                  int32_t stride, const int32_t* __restrict__ stack, int64_t top,
                                  int64_t num_blocks, const __grid_constant__ BlockOpBatch b,
                                  int32_t* __restrict__ err) {
  const BlockOp op = b.op[blockIdx.x];
  int32_t* row = table + (int64_t)op.slot * stride;
  if (b.save_raw) {
    int32_t* rrow = rtable + (int64_t)op.slot * stride;
    for (int j = threadIdx.x; j < b.save_count[blockIdx.x]; j += blockDim.x) rrow[j] = row[j];
    __syncthreads();
  }
  for (int j = threadIdx.x; j < op.count; j += blockDim.x) {
    int64_t pos = top - 1 - (int64_t)(op.off + j);
    int32_t blk = (pos >= 0) ? stack[pos] : -1;
    if (blk < 0 || blk >= num_blocks) atomicCAS(err, 0, 1);
    row[op.from + j] = blk;
  }
}

// Push: stack[top + off_i + j] <- request i's logical block (from + j).
__global__ void push_blocks_kernel(const int32_t* __restrict__ table, int32_t stride,
                                   int32_t* __restrict__ stack, int64_t top,
                                   const __grid_constant__ BlockOpBatch b) {
  const BlockOp op = b.op[blockIdx.x];
  const int32_t* row = table + (int64_t)op.slot * stride;
  for (int j = threadIdx.x; j < op.count; j += blockDim.x) stack[top + op.off + j] = row[op.from + j];
}

__global__ void init_stack_kernel(int32_t* stack, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    stack[i] = (int32_t)(n - 1 - i);
}

}  // namespace fc

using namespace fc;

// ---------------------------------------------------------------------------
// host pool state
// ---------------------------------------------------------------------------
namespace {

enum { ST_RAW = 0, ST_COMPRESSED = 1 };

struct Slot {
  int64_t handle_id = -1;
  int64_t request_id = 0;
  int32_t state = ST_RAW;
  int64_t tokens = 0;      // live tokens (raw, then compressed + decode-appended)
  int32_t n_blocks = 0;    // live blocks in the table row
  int32_t r_blocks = 0;    // retained raw blocks (legacy)
  uint64_t bytes = 0;
  uint64_t retained = 0;   // legacy: raw bytes kept past compression
};

}  // namespace

struct fc_pool {
  fc_model_config cfg{};
  Geom g{};
  int device = 0;
  int mode = FC_POOLED;
  uint64_t capacity = 0, current = 0, peak = 0, zombie_reclaimed = 0;
  int64_t live = 0, alloc_count = 0, retained_handles = 0;
  uint64_t ptb = 0, block_bytes = 0;
  int32_t max_handles = 0;
  int64_t top = 0;  // host mirror of the device stack pointer
  char* arena = nullptr;
  bool owns_arena = false;
  int32_t* d_table = nullptr;
  int32_t* d_rtable = nullptr;
  int32_t* d_stack = nullptr;
  int32_t* d_err = nullptr;
  double* d_wtable = nullptr;
  float* d_ws = nullptr;
  int64_t ws_floats = 0;
  std::vector<Slot> slots;
  std::vector<int32_t> free_slots;
  std::unordered_map<int64_t, int32_t> h2s;
  int64_t next_id = 0;
  bool profiling = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // start, press_end, free_end, end
  int64_t prof_press_launches = 0, prof_total_launches = 0;
  bool prof_valid = false;
  int64_t last_paths[kNumPaths] = {0, 0, 0};  // press launches per path, last compress call
  int last_prefill_tma = -1;                   // kernel of the last prefill write (-1: none yet)
  // host-resident compress (fc_pool_compress_host_batch): a copy stream, two
  // staging slots the DMA fills while the previous slot is scattered into
  // blocks, and a kept-index scratch for the zero-copy V gather.
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t hev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // start, copied[2], scattered[2]
  char* d_stage[2] = {nullptr, nullptr};
  uint64_t stage_bytes = 0;
  int32_t* d_kept = nullptr;
  int64_t kept_cap = 0;
  // decode attention: split-KV partials and per-(request, kv head) arrival counters
  float* d_dec_ws = nullptr;
  int64_t dec_ws_floats = 0;
  int32_t* d_dec_ctr = nullptr;
};

namespace {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

inline int64_t blocks_for(int64_t tokens, int bs) { return (tokens + bs - 1) / bs; }

// kv_bytes with overflow detection (the reference uses Python bigints, kv.py:79-87).
inline bool tok_bytes(const fc_pool* p, int64_t tokens, uint64_t* out) {
  unsigned __int128 v = (unsigned __int128)p->ptb * (unsigned __int128)(uint64_t)tokens;
  if (v > (unsigned __int128)UINT64_MAX) {
    *out = UINT64_MAX;
    return false;
  }
  *out = (uint64_t)v;
  return true;
}

inline uint64_t available(const fc_pool* p) { return p->capacity - p->current; }

void apply(fc_pool* p, int64_t delta) {
  p->current = (uint64_t)((int64_t)p->current + delta);
  if (p->current > p->peak) p->peak = p->current;
}

fc_status lookup(fc_pool* p, int64_t handle_id, int32_t* slot) {
  auto it = p->h2s.find(handle_id);
  if (it == p->h2s.end()) {
    if (handle_id >= 0 && handle_id < p->next_id)
      return set_error(FC_ERR_DOUBLE_FREE, "handle %lld already freed", (long long)handle_id);
    return set_error(FC_ERR_INVALID_ARG, "unknown handle %lld", (long long)handle_id);
  }
  *slot = it->second;
  return FC_OK;
}

// Launch pops (or pushes) for a host-side list of ops, splitting into
// kMaxAllocBatch chunks; updates the host mirror of the stack pointer.
fc_status run_block_ops(fc_pool* p, std::vector<BlockOp>& ops, bool pop, bool save_raw,
                        const std::vector<int32_t>& save_counts, cudaStream_t stream) {
  size_t i = 0;
  while (i < ops.size()) {
    BlockOpBatch b;
    memset(&b, 0, sizeof(b));
    b.save_raw = save_raw ? 1 : 0;
    int32_t off = 0;
    int n = 0;
    for (; i < ops.size() && n < kMaxAllocBatch; ++i, ++n) {
      b.op[n] = ops[i];
      b.op[n].off = off;
      b.save_count[n] = save_raw ? save_counts[i] : 0;
      off += ops[i].count;
    }
    b.n = n;
    if (n == 0) break;
    if (pop) {
      if (off > p->top) return set_error(FC_ERR_CAPACITY, "block pool exhausted");
      if (off > 0 || save_raw) {
        pop_blocks_kernel<<<n, 128, 0, stream>>>(p->d_table, p->d_rtable, p->g.max_bpr, p->d_stack,
                                                 p->top, p->g.num_blocks, b, p->d_err);
        note_launch();
      }
      p->top -= off;
    } else {
      if (off > 0) {
        push_blocks_kernel<<<n, 128, 0, stream>>>(p->d_table, p->g.max_bpr, p->d_stack, p->top, b);
        note_launch();
      }
      p->top += off;
    }
    fc_status st = cuda_check(cudaGetLastError(), pop ? "pop_blocks_kernel" : "push_blocks_kernel");
    if (st != FC_OK) return st;
  }
  return FC_OK;
}

int32_t take_slot(fc_pool* p) {
  int32_t s = p->free_slots.back();
  p->free_slots.pop_back();
  return s;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

int32_t fc_abi_version(void) { return FC_ABI_VERSION; }
const char* fc_last_error(void) { return g_err; }
int64_t fc_launch_count(void) { return g_launches; }

fc_status fc_pool_create(const fc_model_config* cfg, uint64_t capacity_bytes,
                         const fc_pool_options* opts, fc_pool** out) {
  if (!cfg || !opts || !out) return set_error(FC_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  if (cfg->num_layers < 1 || cfg->num_kv_heads < 1 || cfg->head_dim < 1)
    return set_error(FC_ERR_INVALID_ARG, "num_layers, num_kv_heads, head_dim must be >= 1");
  if (cfg->bytes_per_element != 1 && cfg->bytes_per_element != 2 && cfg->bytes_per_element != 4)
    return set_error(FC_ERR_INVALID_ARG, "bytes_per_element must be one of 1, 2, 4");
  static const int dt_bytes[] = {2, 2, 4, 1, 8};
  if (cfg->dtype < 0 || cfg->dtype > FC_U8 || dt_bytes[cfg->dtype] != cfg->bytes_per_element)
    return set_error(FC_ERR_INVALID_ARG, "dtype does not match bytes_per_element");
  if (capacity_bytes < 1) return set_error(FC_ERR_INVALID_ARG, "capacity_bytes must be >= 1");
  if (opts->block_size < 1 || opts->max_handles < 1 || opts->max_blocks_per_handle < 1)
    return set_error(FC_ERR_INVALID_ARG, "block_size, max_handles, max_blocks_per_handle must be >= 1");
  if (cfg->dtype == FC_U8)
    return set_error(FC_ERR_UNSUPPORTED,
                     "device pools need a float KV dtype (f16/bf16/f32): the presses score K");
  if (opts->block_size & (opts->block_size - 1))
    return set_error(FC_ERR_UNSUPPORTED, "block_size must be a power of two");
  if (((int64_t)cfg->head_dim * cfg->bytes_per_element) % 16 != 0)
    return set_error(FC_ERR_UNSUPPORTED, "head_dim * bytes_per_element must be a multiple of 16");

  fc_pool* p = new fc_pool();
  p->cfg = *cfg;
  p->device = opts->device;
  p->mode = opts->mode;
  p->capacity = capacity_bytes;
  p->ptb = 2ull * cfg->num_layers * cfg->num_kv_heads * cfg->head_dim * cfg->bytes_per_element;
  p->block_bytes = p->ptb * (uint64_t)opts->block_size;
  p->max_handles = opts->max_handles;
  Geom& g = p->g;
  g.L = cfg->num_layers;
  g.H = cfg->num_kv_heads;
  g.D = cfg->head_dim;
  g.bs = opts->block_size;
  g.bs_shift = 0;
  while ((1 << g.bs_shift) < g.bs) ++g.bs_shift;
  g.bpe = cfg->bytes_per_element;
  g.max_bpr = opts->max_blocks_per_handle;
  g.num_blocks = opts->num_blocks > 0
                     ? opts->num_blocks
                     : (int64_t)(capacity_bytes / p->block_bytes) +
                           (int64_t)opts->max_handles * (opts->mode == FC_LEGACY_ZOMBIE ? 2 : 1);
  if (g.num_blocks > INT32_MAX) {
    delete p;
    return set_error(FC_ERR_INVALID_ARG, "num_blocks exceeds int32 block ids");
  }
  g.row_bytes = (int64_t)g.D * g.bpe;
  g.block_stride = 2ll * g.H * g.bs * g.row_bytes;
  g.layer_stride = g.num_blocks * g.block_stride;
  const uint64_t arena_bytes = (uint64_t)g.num_blocks * p->block_bytes;

  DeviceGuard guard(p->device);
  fc_status st = FC_OK;
  if (opts->arena) {
    if (opts->arena_bytes < arena_bytes) {
      delete p;
      return set_error(FC_ERR_INVALID_ARG, "external arena too small: %llu < %llu bytes",
                       (unsigned long long)opts->arena_bytes, (unsigned long long)arena_bytes);
    }
    p->arena = (char*)opts->arena;
  } else {
    st = cuda_check(cudaMalloc(&p->arena, arena_bytes), "cudaMalloc(arena)");
    p->owns_arena = true;
  }
  const size_t tbytes = (size_t)p->max_handles * g.max_bpr * sizeof(int32_t);
  if (st == FC_OK) st = cuda_check(cudaMalloc(&p->d_table, tbytes), "cudaMalloc(table)");
  if (st == FC_OK) st = cuda_check(cudaMalloc(&p->d_rtable, tbytes), "cudaMalloc(rtable)");
  if (st == FC_OK)
    st = cuda_check(cudaMalloc(&p->d_stack, g.num_blocks * sizeof(int32_t)), "cudaMalloc(stack)");
  if (st == FC_OK) st = cuda_check(cudaMalloc(&p->d_err, sizeof(int32_t)), "cudaMalloc(err)");
  if (st == FC_OK)
    st = cuda_check(cudaMalloc(&p->d_wtable, 64 * 64 * sizeof(double)), "cudaMalloc(wtable)");
  if (st == FC_OK) st = cuda_check(cudaMemset(p->d_err, 0, sizeof(int32_t)), "cudaMemset");
  if (st == FC_OK) st = cuda_check(cudaMemset(p->d_table, 0xff, tbytes), "cudaMemset");
  if (st == FC_OK) {
    init_stack_kernel<<<256, 256>>>(p->d_stack, g.num_blocks);
    note_launch();
    st = cuda_check(cudaDeviceSynchronize(), "init_stack_kernel");
  }
  if (st != FC_OK) {
    fc_pool_destroy(p);
    return st;
  }
  p->top = g.num_blocks;
  p->slots.resize(p->max_handles);
  for (int32_t s = p->max_handles - 1; s >= 0; --s) p->free_slots.push_back(s);
  *out = p;
  return FC_OK;
}

fc_status fc_pool_destroy(fc_pool* p) {
  if (!p) return FC_OK;
  DeviceGuard guard(p->device);
  cudaDeviceSynchronize();
  if (p->owns_arena) cudaFree(p->arena);
  cudaFree(p->d_table);
  cudaFree(p->d_rtable);
  cudaFree(p->d_stack);
  cudaFree(p->d_err);
  cudaFree(p->d_wtable);
  cudaFree(p->d_ws);
  cudaFree(p->d_stage[0]);
  cudaFree(p->d_stage[1]);
  cudaFree(p->d_kept);
  cudaFree(p->d_dec_ws);
  cudaFree(p->d_dec_ctr);
  for (auto& e : p->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : p->hev)
    if (e) cudaEventDestroy(e);
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  delete p;
  return FC_OK;
}

fc_status fc_pool_arena(fc_pool* p, void** dev_ptr, uint64_t* bytes, int64_t* num_blocks,
                        uint64_t* block_bytes) {
  if (!p) return set_error(FC_ERR_INVALID_ARG, "null pool");
  if (dev_ptr) *dev_ptr = p->arena;
  if (bytes) *bytes = (uint64_t)p->g.num_blocks * p->block_bytes;
  if (num_blocks) *num_blocks = p->g.num_blocks;
  if (block_bytes) *block_bytes = p->block_bytes;
  return FC_OK;
}

fc_status fc_pool_alloc_batch(fc_pool* p, int32_t n, const int64_t* request_ids,
                              const int64_t* tokens, int64_t* handle_ids_out,
                              uint64_t* requested_out, uint64_t* available_out, void* stream) {
  if (!p || n < 0 || (n > 0 && (!tokens || !handle_ids_out)))
    return set_error(FC_ERR_INVALID_ARG, "bad arguments");
  // Validate the whole batch first (atomic: all admitted or none), pool.py:147-165.
  uint64_t cur = p->current;
  int64_t blocks = 0;
  if ((int64_t)n > (int64_t)p->free_slots.size())
    return set_error(FC_ERR_CAPACITY, "more than max_handles=%d live handles", p->max_handles);
  for (int i = 0; i < n; ++i) {
    if (tokens[i] < 0) return set_error(FC_ERR_INVALID_ARG, "tokens must be >= 0");
    uint64_t need;
    bool ok = tok_bytes(p, tokens[i], &need);
    if (!ok || need > p->capacity - cur) {
      if (requested_out) *requested_out = need;
      if (available_out) *available_out = p->capacity - cur;
      return set_error(FC_ERR_CAPACITY, "requested %llu bytes but only %llu available",
                       (unsigned long long)need, (unsigned long long)(p->capacity - cur));
    }
    int64_t nb = blocks_for(tokens[i], p->g.bs);
    if (nb > p->g.max_bpr)
      return set_error(FC_ERR_INVALID_ARG, "request of %lld tokens exceeds max_blocks_per_handle",
                       (long long)tokens[i]);
    cur += need;
    blocks += nb;
  }
  if (blocks > p->top) return set_error(FC_ERR_CAPACITY, "block pool exhausted");
  DeviceGuard guard(p->device);
  std::vector<BlockOp> ops(n);
  for (int i = 0; i < n; ++i) {
    int32_t s = take_slot(p);
    Slot& sl = p->slots[s];
    sl = Slot();
    sl.handle_id = p->next_id++;
    sl.request_id = request_ids ? request_ids[i] : 0;
    sl.state = ST_RAW;
    sl.tokens = tokens[i];
    sl.n_blocks = (int32_t)blocks_for(tokens[i], p->g.bs);
    tok_bytes(p, tokens[i], &sl.bytes);
    p->h2s[sl.handle_id] = s;
    handle_ids_out[i] = sl.handle_id;
    ++p->live;
    ++p->alloc_count;
    apply(p, (int64_t)sl.bytes);
    ops[i] = BlockOp{s, 0, sl.n_blocks, 0};
  }
  return run_block_ops(p, ops, true, false, {}, (cudaStream_t)stream);
}

namespace {

// Every check of a compress call, before any mutation (the batch is atomic).
// Fills the slot and K_r (total, first segment) of every member.
fc_status check_compress(fc_pool* p, int32_t n, const int64_t* handle_ids, const int64_t* seg_tokens,
                         const fc_press_config* press, const fc_press_inputs* inputs,
                         std::vector<int32_t>& slot, std::vector<int32_t>& kept,
                         std::vector<int32_t>& kept0, uint64_t* requested_out,
                         uint64_t* available_out) {
  if (!p || !press || n < 0 || (n > 0 && (!handle_ids || !seg_tokens)))
    return set_error(FC_ERR_INVALID_ARG, "bad arguments");
  if (press->factor < 1) return set_error(FC_ERR_INVALID_ARG, "factor must be >= 1");
  if (press->kind < FC_PRESS_KNORM || press->kind > FC_PRESS_SEEDEDLINEAR)
    return set_error(FC_ERR_INVALID_ARG, "unknown press kind %d", press->kind);
  const bool legacy = p->mode == FC_LEGACY_ZOMBIE;
  const int bs = p->g.bs;
  slot.assign(n, 0);
  kept.assign(n, 0);
  kept0.assign(n, 0);
  uint64_t cur = p->current;
  int64_t new_blocks = 0;
  for (int i = 0; i < n; ++i) {
    fc_status st = lookup(p, handle_ids[i], &slot[i]);
    if (st != FC_OK) return st;
    for (int j = 0; j < i; ++j)
      if (slot[j] == slot[i]) return set_error(FC_ERR_INVALID_ARG, "handle repeated in batch");
    const Slot& sl = p->slots[slot[i]];
    if (sl.state != ST_RAW)
      return set_error(FC_ERR_INVALID_STATE, "transition requires a raw handle, got compressed");
    const int64_t s0 = seg_tokens[2 * i], s1 = seg_tokens[2 * i + 1];
    if (s0 < 0 || s1 < 0 || s0 + s1 != sl.tokens)
      return set_error(FC_ERR_INVALID_ARG, "segment tokens do not sum to the handle's tokens");
    if (sl.tokens == 0) return set_error(FC_ERR_EMPTY_INPUT, "cannot compress an empty cache");
    // K_r: reference ceil rule per modality segment (kv.py:185-193).
    const int64_t k0 = (s0 + press->factor - 1) / press->factor;
    const int64_t k1 = (s1 + press->factor - 1) / press->factor;
    kept0[i] = (int32_t)(s0 > 0 ? k0 : 0);
    kept[i] = (int32_t)(k0 + k1);
    if (press->kind == FC_PRESS_SNAPKV && sl.tokens <= press->window)
      return set_error(FC_ERR_INVALID_ARG, "SnapKV needs more tokens than the window (%d)",
                       press->window);
    if (press->kind == FC_PRESS_EXPECTED_ATTENTION && sl.tokens <= press->n_sink)
      return set_error(FC_ERR_INVALID_ARG, "ExpectedAttention needs more tokens than n_sink (%d)",
                       press->n_sink);
    uint64_t cb;
    tok_bytes(p, kept[i], &cb);
    if (legacy) {
      if (cb > p->capacity - cur) {
        if (requested_out) *requested_out = cb;
        if (available_out) *available_out = p->capacity - cur;
        return set_error(FC_ERR_CAPACITY, "requested %llu bytes but only %llu available",
                         (unsigned long long)cb, (unsigned long long)(p->capacity - cur));
      }
      cur += cb;
      new_blocks += blocks_for(kept[i], bs);
    }
  }
  if (legacy && new_blocks > p->top) return set_error(FC_ERR_CAPACITY, "block pool exhausted");
  if ((press->kind == FC_PRESS_SNAPKV && (!inputs || !inputs->q_window)) ||
      (press->kind == FC_PRESS_EXPECTED_ATTENTION && (!inputs || !inputs->mean_q || !inputs->cov_q)))
    return set_error(FC_ERR_INVALID_ARG, "press inputs missing");
  if ((press->kind == FC_PRESS_SNAPKV || press->kind == FC_PRESS_EXPECTED_ATTENTION) &&
      (press->num_q_heads < p->g.H || press->num_q_heads % p->g.H != 0))
    return set_error(FC_ERR_INVALID_ARG, "num_q_heads must be a multiple of num_kv_heads");
  if (press->kind == FC_PRESS_SEEDEDLINEAR && (press->factor > 64 || !press->chunk_weights))
    return set_error(FC_ERR_UNSUPPORTED, "seeded-linear in-pool compression needs factor <= 64 and weights");
  return FC_OK;
}

}  // namespace

fc_status fc_pool_compress_batch(fc_pool* p, int32_t n, const int64_t* handle_ids,
                                 const int64_t* seg_tokens, const fc_press_config* press,
                                 const fc_press_inputs* inputs, const fc_press_outputs* outputs,
                                 uint64_t* requested_out, uint64_t* available_out, void* stream_) {
  std::vector<int32_t> slot, kept, kept0;
  fc_status st = check_compress(p, n, handle_ids, seg_tokens, press, inputs, slot, kept, kept0,
                                requested_out, available_out);
  if (st != FC_OK || n == 0) return st;
  cudaStream_t stream = (cudaStream_t)stream_;
  const bool legacy = p->mode == FC_LEGACY_ZOMBIE;
  const int bs = p->g.bs;

  DeviceGuard guard(p->device);
  // Plan every launch chunk first: offsets in batch order, launch order LPT
  // (longest request first), chunks of kMaxBatch requests.
  PressParams pp{};
  pp.kind = press->kind;
  pp.factor = press->factor;
  pp.window = press->window;
  pp.pool_kernel = press->pool_kernel;
  pp.n_sink = press->n_sink;
  pp.num_q_heads = press->num_q_heads;
  pp.w_table = p->d_wtable;
  std::vector<int64_t> kept_off(n), score_off(n);
  int64_t ko = 0, so = 0;
  const int64_t LH = (int64_t)p->g.L * p->g.H;
  for (int i = 0; i < n; ++i) {
    kept_off[i] = ko;
    score_off[i] = so;
    ko += (int64_t)kept[i] * LH;
    so += p->slots[slot[i]].tokens * LH;
  }
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return p->slots[slot[a]].tokens > p->slots[slot[b]].tokens;
  });
  std::vector<PressBatch> chunks;
  int64_t need_ws = 0;
  for (int c = 0; c < n; c += kMaxBatch) {
    chunks.emplace_back();
    PressBatch& b = chunks.back();
    memset(&b, 0, sizeof(b));
    b.n = std::min(kMaxBatch, n - c);
    b.per_segment = press->kind <= FC_PRESS_EXPECTED_ATTENTION ? 0 : 1;
    b.in_place = legacy ? 0 : 1;
    b.n_total = n;
    for (int r = 0; r < b.n; ++r) {
      const int i = order[c + r];
      const Slot& sl = p->slots[slot[i]];
      PressReq& q = b.req[r];
      q.slot = slot[i];
      q.T = (int32_t)sl.tokens;
      q.K = kept[i];
      q.seg0 = (int32_t)(seg_tokens[2 * i] > 0 ? seg_tokens[2 * i] : sl.tokens);
      q.K0 = seg_tokens[2 * i] > 0 ? kept0[i] : kept[i];
      q.q_idx = i;
      q.kept_off = kept_off[i];
      q.score_off = score_off[i];
      b.max_T = std::max<int32_t>(b.max_T, q.T);
    }
    if (press->per_segment) b.per_segment = 1;
    need_ws = std::max(need_ws, press_workspace_floats(p->g, press->kind, press->window,
                                                       press->num_q_heads, b.max_T));
  }
  // Dry-run every chunk's launch plan (dtype, head_dim, SMEM budget, tensor-core /
  // SIMT split, tensor maps) and size the workspace BEFORE any pop, push or
  // launch: a refused batch leaves blocks, tables, payload and ledger untouched
  // (the reference's all-or-nothing mutations, pool.py:147-165,167-192).
  const int32_t* src_table = legacy ? p->d_rtable : p->d_table;
  for (const PressBatch& b : chunks) {
    st = launch_press(p->g, p->cfg.dtype, p->arena, src_table, p->d_table, b, pp, inputs, outputs,
                      p->d_ws, p->ws_floats, p->d_err, stream, /*dry_run=*/true);
    if (st != FC_OK) return st;
  }
  if (need_ws > p->ws_floats) {
    cudaStreamSynchronize(stream);
    cudaFree(p->d_ws);
    p->d_ws = nullptr;
    p->ws_floats = 0;
    st = cuda_check(cudaMalloc(&p->d_ws, need_ws * sizeof(float)), "cudaMalloc(workspace)");
    if (st != FC_OK) return st;
    p->ws_floats = need_ws;
  }
  // Host-side weight table for SEEDEDLINEAR (row m-1 = renormalised w[:m]).
  if (press->kind == FC_PRESS_SEEDEDLINEAR) {
    std::vector<double> wt((size_t)press->factor * press->factor, 0.0);
    for (int m = 1; m <= press->factor; ++m) {
      double s = 0;
      for (int i = 0; i < m; ++i) s += press->chunk_weights[i];
      for (int i = 0; i < m; ++i) wt[(size_t)(m - 1) * press->factor + i] = press->chunk_weights[i] / s;
    }
    st = cuda_check(cudaMemcpyAsync(p->d_wtable, wt.data(), wt.size() * sizeof(double),
                                    cudaMemcpyHostToDevice, stream),
                    "upload chunk weights");
    if (st != FC_OK) return st;
  }

  const int64_t launches0 = g_launches;
  int64_t paths0[kNumPaths];
  for (int k = 0; k < kNumPaths; ++k) paths0[k] = path_count(k);
  if (p->profiling) cudaEventRecord(p->ev[0], stream);
  // Legacy: move the raw rows aside and pop fresh destination blocks (batch order).
  if (legacy) {
    std::vector<BlockOp> ops(n);
    std::vector<int32_t> save(n);
    for (int i = 0; i < n; ++i) {
      ops[i] = BlockOp{slot[i], 0, (int32_t)blocks_for(kept[i], bs), 0};
      save[i] = p->slots[slot[i]].n_blocks;
    }
    st = run_block_ops(p, ops, true, true, save, stream);
    if (st != FC_OK) return st;
  }
  for (const PressBatch& b : chunks) {
    st = launch_press(p->g, p->cfg.dtype, p->arena, src_table, p->d_table, b, pp, inputs, outputs,
                      p->d_ws, p->ws_floats, p->d_err, stream);
    if (st != FC_OK) return st;
  }
  for (int k = 0; k < kNumPaths; ++k) p->last_paths[k] = path_count(k) - paths0[k];

  int64_t press_launches = g_launches - launches0;
  if (p->profiling) cudaEventRecord(p->ev[1], stream);
  // Pooled: free the tail blocks in the same stream step (zero-zombie reclaim).
  if (!legacy) {
    std::vector<BlockOp> ops(n);
    for (int i = 0; i < n; ++i) {
      const Slot& sl = p->slots[slot[i]];
      const int32_t keep = (int32_t)blocks_for(kept[i], bs);
      ops[i] = BlockOp{slot[i], keep, sl.n_blocks - keep, 0};
    }
    st = run_block_ops(p, ops, false, false, {}, stream);
    if (st != FC_OK) return st;
  }
  if (p->profiling) {
    cudaEventRecord(p->ev[2], stream);
    cudaEventRecord(p->ev[3], stream);
    p->prof_press_launches = press_launches;
    p->prof_total_launches = g_launches - launches0;
    p->prof_valid = true;
  }

  // Host accounting, batch order (engine.py:501-510 -> pool.py:167-192).
  for (int i = 0; i < n; ++i) {
    Slot& sl = p->slots[slot[i]];
    uint64_t cb;
    tok_bytes(p, kept[i], &cb);
    if (legacy) {
      sl.retained = sl.bytes;
      sl.r_blocks = sl.n_blocks;
      ++p->retained_handles;
      apply(p, (int64_t)cb);
    } else {
      p->zombie_reclaimed += sl.bytes - cb;
      apply(p, (int64_t)cb - (int64_t)sl.bytes);
    }
    sl.bytes = cb;
    sl.tokens = kept[i];
    sl.n_blocks = (int32_t)blocks_for(kept[i], bs);
    sl.state = ST_COMPRESSED;
  }
  return FC_OK;
}

// Host-resident compress: request i's raw KV is a pinned host buffer
// [L][2][H][T_i][D]. Split path (pooled Knorm / SnapKV, whose scores read only
// K): DMA the K planes through two staging slots on the pool's copy stream
// (slot i+1 fills while slot i is scattered into blocks), compress, then read
// only the kept V rows over PCIe (gather_host_rows_kernel) -- 0.5 R + 0.5 C
// bytes cross PCIe instead of R. Other presses / legacy mode DMA all of K and V.
fc_status fc_pool_compress_host_batch(fc_pool* p, int32_t n, const int64_t* handle_ids,
                                      const int64_t* seg_tokens, const fc_press_config* press,
                                      const fc_press_inputs* inputs,
                                      const fc_press_outputs* outputs, const void* const* host_kv,
                                      uint64_t* requested_out, uint64_t* available_out,
                                      void* stream_) {
  std::vector<int32_t> slot, kept, kept0;
  fc_status st = check_compress(p, n, handle_ids, seg_tokens, press, inputs, slot, kept, kept0,
                                requested_out, available_out);
  if (st != FC_OK || n == 0) return st;
  if (!host_kv) return set_error(FC_ERR_INVALID_ARG, "host_kv missing");
  cudaStream_t stream = (cudaStream_t)stream_;
  DeviceGuard guard(p->device);
  const Geom& g = p->g;
  const bool split = p->mode == FC_POOLED &&
                     (press->kind == FC_PRESS_KNORM || press->kind == FC_PRESS_SNAPKV);
  std::vector<const char*> dev_host(n);
  uint64_t max_stage = 0;
  for (int i = 0; i < n; ++i) {
    if (!host_kv[i] || ((uintptr_t)host_kv[i]) % 16)
      return set_error(FC_ERR_INVALID_ARG, "host_kv[%d] missing or not 16-byte aligned", i);
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, host_kv[i]) != cudaSuccess || at.type != cudaMemoryTypeHost ||
        !at.devicePointer) {
      cudaGetLastError();
      return set_error(FC_ERR_INVALID_ARG,
                       "host_kv[%d] must be pinned host memory (cudaHostAlloc / pin_memory)", i);
    }
    dev_host[i] = (const char*)at.devicePointer;
    const uint64_t plane = (uint64_t)g.H * p->slots[slot[i]].tokens * g.row_bytes;
    max_stage = std::max<uint64_t>(max_stage, plane * g.L * (split ? 1 : 2));
  }
  if (!p->copy_stream) {
    st = cuda_check(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking),
                    "cudaStreamCreate(copy)");
    for (auto& e : p->hev)
      if (st == FC_OK) st = cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    if (st != FC_OK) return st;
  }
  if (max_stage > p->stage_bytes) {
    cudaStreamSynchronize(p->copy_stream);
    cudaStreamSynchronize(stream);
    for (auto& b : p->d_stage) {
      cudaFree(b);
      b = nullptr;
    }
    p->stage_bytes = 0;
    for (auto& b : p->d_stage) {
      st = cuda_check(cudaMalloc(&b, max_stage), "cudaMalloc(staging)");
      if (st != FC_OK) return st;
    }
    p->stage_bytes = max_stage;
  }
  // Ingest: DMA into staging slot i%2 on the copy stream, scatter on `stream`.
  cudaEventRecord(p->hev[0], stream);
  cudaStreamWaitEvent(p->copy_stream, p->hev[0], 0);
  for (int i = 0; i < n; ++i) {
    const int b = i & 1;
    const int64_t T = p->slots[slot[i]].tokens;
    const size_t plane = (size_t)g.H * T * g.row_bytes;
    if (i >= 2) cudaStreamWaitEvent(p->copy_stream, p->hev[3 + b], 0);
    if (split)
      st = cuda_check(cudaMemcpy2DAsync(p->d_stage[b], plane, host_kv[i], 2 * plane, plane, g.L,
                                        cudaMemcpyHostToDevice, p->copy_stream),
                      "cudaMemcpy2DAsync(K planes)");
    else
      st = cuda_check(cudaMemcpyAsync(p->d_stage[b], host_kv[i], 2 * plane * g.L,
                                      cudaMemcpyHostToDevice, p->copy_stream),
                      "cudaMemcpyAsync(KV)");
    if (st != FC_OK) return st;
    cudaEventRecord(p->hev[1 + b], p->copy_stream);
    cudaStreamWaitEvent(stream, p->hev[1 + b], 0);
    st = launch_store(g, p->arena, p->d_table + (int64_t)slot[i] * g.max_bpr, 0, T, p->d_stage[b],
                      true, stream, 0, split ? 1 : 2);
    if (st != FC_OK) return st;
    cudaEventRecord(p->hev[3 + b], stream);
  }
  // Compress on the device-resident K (and V); the split path needs the kept indices.
  fc_press_outputs outs{};
  if (outputs) outs = *outputs;
  const int64_t LH = (int64_t)g.L * g.H;
  int64_t sum_kept = 0;
  for (int i = 0; i < n; ++i) sum_kept += (int64_t)kept[i] * LH;
  if (split && !outs.kept_idx) {
    if (sum_kept > p->kept_cap) {
      cudaStreamSynchronize(stream);
      cudaFree(p->d_kept);
      p->d_kept = nullptr;
      p->kept_cap = 0;
      st = cuda_check(cudaMalloc(&p->d_kept, sum_kept * sizeof(int32_t)), "cudaMalloc(kept)");
      if (st != FC_OK) return st;
      p->kept_cap = sum_kept;
    }
    outs.kept_idx = p->d_kept;
  }
  st = fc_pool_compress_batch(p, n, handle_ids, seg_tokens, press, inputs, &outs, requested_out,
                              available_out, stream_);
  if (st != FC_OK || !split) return st;
  // Kept V rows: zero-copy reads of the pinned host buffers into rank slots.
  std::vector<HostGatherReq> reqs(n);
  int64_t ko = 0;
  for (int i = 0; i < n; ++i) {
    reqs[i] = HostGatherReq{slot[i], 0, kept[i], 0, ko, dev_host[i]};
    ko += (int64_t)kept[i] * LH;
  }
  // raw T of request i = the sum of its segments (the slot now holds K_r)
  for (int i = 0; i < n; ++i) reqs[i].T = (int32_t)(seg_tokens[2 * i] + seg_tokens[2 * i + 1]);
  return launch_gather_host(g, p->arena, p->d_table, n, reqs.data(), outs.kept_idx, 1, stream);
}

fc_status fc_pool_append(fc_pool* p, int32_t n, const int64_t* handle_ids, const int64_t* tokens,
                         uint64_t* requested_out, uint64_t* available_out, void* stream) {
  if (!p || n < 0 || (n > 0 && (!handle_ids || !tokens)))
    return set_error(FC_ERR_INVALID_ARG, "bad arguments");
  // Validate the whole batch -- bytes, per-handle block rows AND the block demand
  // on the free stack -- before mutating anything (pool.py:194-211 is strict and
  // all-or-nothing). Members may repeat a handle: each sees its predecessors' growth.
  std::vector<int32_t> slot(n);
  std::vector<int64_t> new_tokens(n);
  std::vector<BlockOp> ops;
  std::unordered_map<int32_t, std::pair<int64_t, int32_t>> grown;  // slot -> (tokens, blocks)
  uint64_t cur = p->current;
  int64_t blocks = 0;
  for (int i = 0; i < n; ++i) {
    fc_status st = lookup(p, handle_ids[i], &slot[i]);
    if (st != FC_OK) return st;
    const Slot& sl = p->slots[slot[i]];
    if (sl.state != ST_COMPRESSED)
      return set_error(FC_ERR_INVALID_STATE, "append requires a compressed handle, got raw");
    if (tokens[i] < 1) return set_error(FC_ERR_INVALID_ARG, "token_count must be >= 1");
    uint64_t need;
    bool ok = tok_bytes(p, tokens[i], &need);
    if (!ok || need > p->capacity - cur) {
      if (requested_out) *requested_out = need;
      if (available_out) *available_out = p->capacity - cur;
      return set_error(FC_ERR_CAPACITY, "requested %llu bytes but only %llu available",
                       (unsigned long long)need, (unsigned long long)(p->capacity - cur));
    }
    cur += need;
    auto it = grown.find(slot[i]);
    const int64_t t0 = it == grown.end() ? sl.tokens : it->second.first;
    const int32_t b0 = it == grown.end() ? sl.n_blocks : it->second.second;
    const int64_t t1 = t0 + tokens[i];
    const int64_t b1 = blocks_for(t1, p->g.bs);
    if (b1 > p->g.max_bpr) return set_error(FC_ERR_INVALID_ARG, "handle exceeds max_blocks_per_handle");
    if (b1 > b0) {
      blocks += b1 - b0;
      ops.push_back(BlockOp{slot[i], b0, (int32_t)(b1 - b0), 0});
    }
    grown[slot[i]] = {t1, (int32_t)std::max<int64_t>(b0, b1)};
    new_tokens[i] = t1;
  }
  if (blocks > p->top) return set_error(FC_ERR_CAPACITY, "block pool exhausted");
  DeviceGuard guard(p->device);
  fc_status st = run_block_ops(p, ops, true, false, {}, (cudaStream_t)stream);
  if (st != FC_OK) return st;
  for (int i = 0; i < n; ++i) {
    Slot& sl = p->slots[slot[i]];
    uint64_t need;
    tok_bytes(p, tokens[i], &need);
    sl.tokens = new_tokens[i];
    sl.n_blocks = (int32_t)blocks_for(sl.tokens, p->g.bs);
    sl.bytes += need;
    apply(p, (int64_t)need);
  }
  return FC_OK;
}

fc_status fc_pool_release_batch(fc_pool* p, int32_t n, const int64_t* handle_ids, void* stream) {
  if (!p || n < 0 || (n > 0 && !handle_ids)) return set_error(FC_ERR_INVALID_ARG, "bad arguments");
  std::vector<int32_t> slot(n);
  for (int i = 0; i < n; ++i) {
    fc_status st = lookup(p, handle_ids[i], &slot[i]);
    if (st != FC_OK) return st;
    for (int j = 0; j < i; ++j)
      if (slot[j] == slot[i])
        return set_error(FC_ERR_DOUBLE_FREE, "handle %lld already freed", (long long)handle_ids[i]);
  }
  DeviceGuard guard(p->device);
  // Push order: request order; live blocks ascending, then retained raw blocks.
  // Retained rows live in d_rtable, so push them with a second op list that
  // reads that table; to keep one contiguous push order we interleave per
  // request by launching live and retained ops in sequence per chunk.
  std::vector<BlockOp> live_ops, raw_ops;
  bool any_raw = false;
  for (int i = 0; i < n; ++i) any_raw |= p->slots[slot[i]].r_blocks > 0;
  fc_status st = FC_OK;
  if (!any_raw) {
    for (int i = 0; i < n; ++i)
      live_ops.push_back(BlockOp{slot[i], 0, p->slots[slot[i]].n_blocks, 0});
    st = run_block_ops(p, live_ops, false, false, {}, (cudaStream_t)stream);
  } else {
    // Legacy releases: per request, live then retained (keeps the oracle order).
    for (int i = 0; i < n && st == FC_OK; ++i) {
      std::vector<BlockOp> one{BlockOp{slot[i], 0, p->slots[slot[i]].n_blocks, 0}};
      st = run_block_ops(p, one, false, false, {}, (cudaStream_t)stream);
      if (st != FC_OK) break;
      if (p->slots[slot[i]].r_blocks > 0) {
        BlockOpBatch b;
        memset(&b, 0, sizeof(b));
        b.n = 1;
        b.op[0] = BlockOp{slot[i], 0, p->slots[slot[i]].r_blocks, 0};
        push_blocks_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(p->d_rtable, p->g.max_bpr,
                                                                p->d_stack, p->top, b);
        note_launch();
        p->top += p->slots[slot[i]].r_blocks;
        st = cuda_check(cudaGetLastError(), "push_blocks_kernel(retained)");
      }
    }
  }
  if (st != FC_OK) return st;
  for (int i = 0; i < n; ++i) {
    Slot& sl = p->slots[slot[i]];
    const uint64_t freed = sl.bytes + sl.retained;
    if (sl.retained > 0) --p->retained_handles;
    apply(p, -(int64_t)freed);
    --p->live;
    p->h2s.erase(sl.handle_id);
    sl = Slot();
    p->free_slots.push_back(slot[i]);
  }
  return FC_OK;
}

// ---------------------------------------------------------------------------
// decode over the compacted blocks
// ---------------------------------------------------------------------------
fc_status fc_pool_write_kv(fc_pool* p, int32_t layer, int32_t n, const int64_t* handle_ids,
                           const int64_t* positions, const void* k, const void* v, void* stream) {
  if (!p || n < 0 || (n > 0 && (!handle_ids || !k || !v)))
    return set_error(FC_ERR_INVALID_ARG, "bad arguments");
  if (layer < 0 || layer >= p->g.L) return set_error(FC_ERR_INVALID_ARG, "layer out of range");
  if (((uintptr_t)k) % 16 || ((uintptr_t)v) % 16)
    return set_error(FC_ERR_INVALID_ARG, "k / v must be 16-byte aligned");
  std::vector<KVWriteReq> reqs(n);
  for (int i = 0; i < n; ++i) {
    int32_t s;
    fc_status st = lookup(p, handle_ids[i], &s);
    if (st != FC_OK) return st;
    const int64_t T = p->slots[s].tokens;
    const int64_t pos = positions ? positions[i] : T - 1;
    if (pos < 0 || pos >= T) return set_error(FC_ERR_INVALID_ARG, "position %lld outside the handle's %lld tokens",
                                              (long long)pos, (long long)T);
    reqs[i] = KVWriteReq{s, (int32_t)pos, i};
  }
  DeviceGuard guard(p->device);
  for (int c = 0; c < n; c += kMaxDecode) {
    KVWriteBatch b;
    memset(&b, 0, sizeof(b));
    b.n = std::min(kMaxDecode, n - c);
    b.layer = layer;
    for (int i = 0; i < b.n; ++i) b.req[i] = reqs[c + i];
    fc_status st = launch_write_kv(p->g, p->arena, p->d_table, b, k, v, (cudaStream_t)stream);
    if (st != FC_OK) return st;
  }
  return FC_OK;
}

fc_status fc_pool_write_prefill_kv(fc_pool* p, int32_t layer, int32_t n, const int64_t* handle_ids,
                                   const int64_t* cu_seqlens, const int64_t* tok_begin,
                                   const void* k, const void* v, void* stream) {
  if (!p || n < 0 || (n > 0 && (!handle_ids || !cu_seqlens || !k || !v)))
    return set_error(FC_ERR_INVALID_ARG, "bad arguments");
  if (layer < 0 || layer >= p->g.L) return set_error(FC_ERR_INVALID_ARG, "layer out of range");
  if (((uintptr_t)k) % 16 || ((uintptr_t)v) % 16)
    return set_error(FC_ERR_INVALID_ARG, "k / v must be 16-byte aligned");
  if (n > 0 && cu_seqlens[0] != 0) return set_error(FC_ERR_INVALID_ARG, "cu_seqlens[0] must be 0");
  std::vector<PrefillReq> reqs(n);
  for (int i = 0; i < n; ++i) {
    int32_t s;
    fc_status st = lookup(p, handle_ids[i], &s);
    if (st != FC_OK) return st;
    for (int j = 0; j < i; ++j)
      if (reqs[j].slot == s) return set_error(FC_ERR_INVALID_ARG, "handle repeated in batch");
    const int64_t cnt = cu_seqlens[i + 1] - cu_seqlens[i];
    const int64_t t0 = tok_begin ? tok_begin[i] : 0;
    if (cnt < 0 || t0 < 0 || t0 + cnt > p->slots[s].tokens)
      return set_error(FC_ERR_INVALID_ARG, "rows of request %d fall outside its %lld tokens", i,
                       (long long)p->slots[s].tokens);
    reqs[i] = PrefillReq{cu_seqlens[i], t0, s, (int32_t)cnt};
  }
  if (n == 0) return FC_OK;
  DeviceGuard guard(p->device);
  return launch_write_prefill(p->g, p->arena, p->d_table, layer, n, reqs.data(), k, v,
                              (cudaStream_t)stream, &p->last_prefill_tma);
}

fc_status fc_pool_decode_attention(fc_pool* p, int32_t layer, int32_t n, const int64_t* handle_ids,
                                   int32_t num_q_heads, float scale, const void* q, void* out,
                                   void* stream) {
  if (!p || n < 0 || (n > 0 && (!handle_ids || !q || !out)))
    return set_error(FC_ERR_INVALID_ARG, "bad arguments");
  if (layer < 0 || layer >= p->g.L) return set_error(FC_ERR_INVALID_ARG, "layer out of range");
  if (num_q_heads < p->g.H || num_q_heads % p->g.H)
    return set_error(FC_ERR_INVALID_ARG, "num_q_heads must be a multiple of num_kv_heads");
  if (((uintptr_t)q) % 16 || ((uintptr_t)out) % 16)
    return set_error(FC_ERR_INVALID_ARG, "q / out must be 16-byte aligned");
  const int gq = num_q_heads / p->g.H;
  std::vector<int32_t> slot(n);
  int64_t total_tok = 0;
  for (int i = 0; i < n; ++i) {
    fc_status st = lookup(p, handle_ids[i], &slot[i]);
    if (st != FC_OK) return st;
    if (p->slots[slot[i]].tokens == 0) return set_error(FC_ERR_EMPTY_INPUT, "handle has no tokens");
    total_tok += p->slots[slot[i]].tokens;
  }
  if (n == 0) return FC_OK;
  if (scale <= 0.f) scale = 1.0f / sqrtf((float)p->g.D);
  const float scale_log2 = scale * 1.4426950408889634f;
  // Split-KV only when (request, kv head) pairs alone cannot fill one wave of
  // 4 CTAs per SM: measured at c2d, 2-16 waves of splits cost 18-30% more
  // than the ragged 1.7-wave unsplit grid (partials + merge + short CTAs).
  const int64_t want_items = (int64_t)sm_count() * 4;
  int split = 1 << 30;
  if ((int64_t)n * p->g.H < want_items) {
    const int64_t s = (total_tok * p->g.H + want_items - 1) / want_items;
    split = (int)std::max<int64_t>(128, (s + 63) / 64 * 64);
  }
  DeviceGuard guard(p->device);
  fc_status st;
  if (!p->d_dec_ctr) {
    st = cuda_check(cudaMalloc(&p->d_dec_ctr, (size_t)kMaxDecode * p->g.H * sizeof(int32_t)),
                    "cudaMalloc(decode counters)");
    if (st != FC_OK) return st;
    st = cuda_check(cudaMemset(p->d_dec_ctr, 0, (size_t)kMaxDecode * p->g.H * sizeof(int32_t)),
                    "cudaMemset(decode counters)");
    if (st != FC_OK) return st;
  }
  for (int c = 0; c < n; c += kMaxDecode) {
    DecodeBatch b;
    memset(&b, 0, sizeof(b));
    b.n = std::min(kMaxDecode, n - c);
    b.Hq = num_q_heads;
    b.layer = layer;
    b.split_tokens = split;
    int items = 0;
    for (int i = 0; i < b.n; ++i) {
      const int64_t T = p->slots[slot[c + i]].tokens;
      const int ns = (int)((T + split - 1) / split);
      b.req[i] = DecodeReq{slot[c + i], (int32_t)T, items, ns, c + i};
      items += p->g.H * ns;
    }
    b.items = items;
    const int64_t need = (int64_t)items * gq * (p->g.D + 2);
    if (need > p->dec_ws_floats) {
      cudaStreamSynchronize((cudaStream_t)stream);
      cudaFree(p->d_dec_ws);
      p->d_dec_ws = nullptr;
      p->dec_ws_floats = 0;
      st = cuda_check(cudaMalloc(&p->d_dec_ws, need * sizeof(float)), "cudaMalloc(decode workspace)");
      if (st != FC_OK) return st;
      p->dec_ws_floats = need;
    }
    st = launch_decode_attention(p->g, p->cfg.dtype, p->arena, p->d_table, b, gq, q, out,
                                 scale_log2, p->d_dec_ws, p->d_dec_ctr, (cudaStream_t)stream);
    if (st != FC_OK) return st;
  }
  return FC_OK;
}

fc_status fc_pool_synchronize(fc_pool* p) {
  if (!p) return set_error(FC_ERR_INVALID_ARG, "null pool");
  DeviceGuard guard(p->device);
  fc_status st = cuda_check(cudaDeviceSynchronize(), "synchronize");
  if (st != FC_OK) return st;
  int32_t err = 0;
  st = cuda_check(cudaMemcpy(&err, p->d_err, sizeof(err), cudaMemcpyDeviceToHost), "read error word");
  if (st != FC_OK) return st;
  if (err) return set_error(FC_ERR_DEVICE, "device error word %d (block-table invariant)", err);
  return FC_OK;
}

fc_status fc_pool_get_stats(fc_pool* p, fc_pool_stats* out) {
  if (!p || !out) return set_error(FC_ERR_INVALID_ARG, "null argument");
  fc_status st = fc_pool_synchronize(p);
  memset(out, 0, sizeof(*out));
  out->current_bytes = p->current;
  out->peak_bytes = p->peak;
  out->capacity_bytes = p->capacity;
  out->live_handles = p->live;
  out->zombie_bytes_reclaimed = p->zombie_reclaimed;
  out->allocation_count = p->alloc_count;
  out->num_blocks = p->g.num_blocks;
  out->free_blocks = p->top;
  out->used_blocks = p->g.num_blocks - p->top;
  out->block_bytes = p->block_bytes;
  uint64_t live_tok = 0;
  for (const auto& kv : p->h2s) {
    const Slot& sl = p->slots[kv.second];
    live_tok += sl.bytes + sl.retained;
  }
  out->live_token_bytes = live_tok;
  const double used = (double)out->used_blocks * (double)p->block_bytes;
  out->fragmentation = used > 0 ? 1.0 - (double)live_tok / used : 0.0;
  out->device_error = st == FC_ERR_DEVICE ? 1 : 0;
  return st;
}

fc_status fc_pool_set_profiling(fc_pool* p, int32_t enable) {
  if (!p) return set_error(FC_ERR_INVALID_ARG, "null pool");
  DeviceGuard guard(p->device);
  if (enable && !p->ev[0]) {
    for (auto& e : p->ev) {
      fc_status st = cuda_check(cudaEventCreate(&e), "cudaEventCreate");
      if (st != FC_OK) return st;
    }
  }
  p->profiling = enable != 0;
  p->prof_valid = false;
  return FC_OK;
}

fc_status fc_pool_last_profile(fc_pool* p, fc_profile* out) {
  if (!p || !out) return set_error(FC_ERR_INVALID_ARG, "null argument");
  if (!p->prof_valid) return set_error(FC_ERR_INVALID_STATE, "no profiled compress call");
  DeviceGuard guard(p->device);
  fc_status st = cuda_check(cudaEventSynchronize(p->ev[3]), "cudaEventSynchronize");
  if (st != FC_OK) return st;
  float a = 0, b = 0, c = 0;
  cudaEventElapsedTime(&a, p->ev[0], p->ev[1]);
  cudaEventElapsedTime(&b, p->ev[1], p->ev[2]);
  cudaEventElapsedTime(&c, p->ev[0], p->ev[3]);
  out->press_ms = a;
  out->free_ms = b;
  out->total_ms = c;
  out->press_launches = p->prof_press_launches;
  out->total_launches = p->prof_total_launches;
  return FC_OK;
}

fc_status fc_pool_last_paths(fc_pool* p, int64_t out[3]) {
  if (!p || !out) return set_error(FC_ERR_INVALID_ARG, "null argument");
  for (int k = 0; k < kNumPaths; ++k) out[k] = p->last_paths[k];
  return FC_OK;
}

fc_status fc_pool_last_prefill_path(fc_pool* p, int32_t* tma) {
  if (!p || !tma) return set_error(FC_ERR_INVALID_ARG, "null argument");
  *tma = p->last_prefill_tma;
  return FC_OK;
}

fc_status fc_pool_block_table(fc_pool* p, int64_t handle_id, const int32_t** dev_row,
                              int32_t* n_blocks, int64_t* n_tokens) {
  if (!p) return set_error(FC_ERR_INVALID_ARG, "null pool");
  int32_t s;
  fc_status st = lookup(p, handle_id, &s);
  if (st != FC_OK) return st;
  if (dev_row) *dev_row = p->d_table + (int64_t)s * p->g.max_bpr;
  if (n_blocks) *n_blocks = p->slots[s].n_blocks;
  if (n_tokens) *n_tokens = p->slots[s].tokens;
  return FC_OK;
}

fc_status fc_pool_store_tokens(fc_pool* p, int64_t handle_id, int64_t tok_begin, int64_t n_tok,
                               const void* src, void* stream) {
  if (!p || !src) return set_error(FC_ERR_INVALID_ARG, "bad arguments");
  int32_t s;
  fc_status st = lookup(p, handle_id, &s);
  if (st != FC_OK) return st;
  if (tok_begin < 0 || n_tok < 0 || tok_begin + n_tok > p->slots[s].tokens)
    return set_error(FC_ERR_INVALID_ARG, "token range outside the handle");
  if (n_tok == 0) return FC_OK;
  DeviceGuard guard(p->device);
  return launch_store(p->g, p->arena, p->d_table + (int64_t)s * p->g.max_bpr, tok_begin, n_tok,
                      src, true, (cudaStream_t)stream);
}

fc_status fc_pool_load_tokens(fc_pool* p, int64_t handle_id, int64_t tok_begin, int64_t n_tok,
                              void* dst, void* stream) {
  if (!p || !dst) return set_error(FC_ERR_INVALID_ARG, "bad arguments");
  int32_t s;
  fc_status st = lookup(p, handle_id, &s);
  if (st != FC_OK) return st;
  if (tok_begin < 0 || n_tok < 0 || tok_begin + n_tok > p->slots[s].tokens)
    return set_error(FC_ERR_INVALID_ARG, "token range outside the handle");
  if (n_tok == 0) return FC_OK;
  DeviceGuard guard(p->device);
  return launch_store(p->g, p->arena, p->d_table + (int64_t)s * p->g.max_bpr, tok_begin, n_tok,
                      dst, false, (cudaStream_t)stream);
}

fc_status fc_synth_fill(fc_pool* p, int32_t n, const int64_t* handle_ids, const int64_t* keys,
                        uint64_t seed, int32_t dist, void* stream) {
  if (!p || n < 0 || (n > 0 && (!handle_ids || !keys)))
    return set_error(FC_ERR_INVALID_ARG, "bad arguments");
  if (p->cfg.dtype > FC_F32) return set_error(FC_ERR_UNSUPPORTED, "synth fill needs f16/bf16/f32");
  std::vector<int32_t> slots(n), toks(n);
  std::vector<uint64_t> k(n);
  for (int i = 0; i < n; ++i) {
    fc_status st = lookup(p, handle_ids[i], &slots[i]);
    if (st != FC_OK) return st;
    toks[i] = (int32_t)p->slots[slots[i]].tokens;
    k[i] = (uint64_t)keys[i];
  }
  DeviceGuard guard(p->device);
  return launch_synth(p->g, p->cfg.dtype, p->arena, p->d_table, n, slots.data(), toks.data(),
                      k.data(), seed, dist, (cudaStream_t)stream);
}

fc_status fc_compress_tensor(const void* src, int64_t n, int64_t d, int32_t dtype,
                             const fc_press_config* press, void* dst, void* stream) {
  if (!src || !dst || !press || d < 1) return set_error(FC_ERR_INVALID_ARG, "bad arguments");
  if (n == 0) return set_error(FC_ERR_EMPTY_INPUT, "cannot compress an empty token sequence");
  if (n < 0 || press->factor < 1) return set_error(FC_ERR_INVALID_ARG, "bad shape or factor");
  if (press->kind != FC_PRESS_MEANPOOL && press->kind != FC_PRESS_SEEDEDLINEAR)
    return set_error(FC_ERR_INVALID_ARG, "compress_tensor supports meanpool / seededlinear");
  if (dtype < FC_F16 || dtype > FC_F64 || dtype == FC_U8)
    return set_error(FC_ERR_UNSUPPORTED, "compress_tensor needs a float dtype");
  PressParams pp{};
  pp.kind = press->kind;
  pp.factor = press->factor;
  double* d_w = nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  if (press->kind == FC_PRESS_SEEDEDLINEAR) {
    if (!press->chunk_weights) return set_error(FC_ERR_INVALID_ARG, "weights missing");
    // Only two chunk sizes occur: full (k) and the tail (n mod k).
    const int k = press->factor;
    const int m_tail = (int)(n % k);
    std::vector<double> wt(2 * (size_t)k, 0.0);
    for (int row = 0; row < 2; ++row) {
      const int m = row == 0 ? k : (m_tail ? m_tail : k);
      double sum = 0;
      for (int i = 0; i < m; ++i) sum += press->chunk_weights[i];
      for (int i = 0; i < m; ++i) wt[(size_t)row * k + i] = press->chunk_weights[i] / sum;
    }
    fc_status st = cuda_check(cudaMallocAsync((void**)&d_w, wt.size() * sizeof(double), s),
                              "cudaMallocAsync(weights)");
    if (st != FC_OK) return st;
    st = cuda_check(cudaMemcpyAsync(d_w, wt.data(), wt.size() * sizeof(double),
                                    cudaMemcpyHostToDevice, s),
                    "upload weights");
    if (st != FC_OK) return st;
    pp.w_table = d_w;
  }
  fc_status st = launch_compress_tensor(src, n, d, dtype, pp, dst, s);
  if (d_w) cudaFreeAsync(d_w, s);
  return st;
}

}  // extern "C"
