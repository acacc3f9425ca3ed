// fc_internal.cuh -- shared device/host internals of the FastCache B200 library.
//
// HBM layout of the paged pool (one arena per fc_pool):
//
//   arena[L][NB][2][Hkv][bs][D]     (element type = pool dtype)
//
// A block holds `bs` tokens of one request for every layer, K|V and kv-head,
// so block_bytes = bs * bytes_per_token (reference kv.py:68-76). Within a
// layer, one (block, K|V, head) chunk is bs*D*bpe contiguous bytes (4 KiB
// for LLaVA fp16 at bs=16): the unit every kernel streams with 128-bit loads.
// A request's token t of (layer l, kv, head h) lives at
//
//   arena + l*layer_stride + table[t / bs]*block_stride + (kv*H + h)*bs*row
//         + (t % bs)*row,      row = D*bpe,  block_stride = 2*H*bs*row,
//                              layer_stride = NB*block_stride.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fastcache.h"

namespace fc {

constexpr int kMaxBatch = 128;      // requests per press launch (kernel-param descriptor)
// Dynamic SMEM a persistent kernel may request: the 227-KB per-CTA opt-in limit
// minus headroom for its static __shared__ scratch (select / barrier words).
constexpr int kDynSmemBudget = 227 * 1024 - 4096;
constexpr int kMaxAllocBatch = 512; // requests per pop/push launch

// Geometry of a pool, passed by value to kernels.
struct Geom {
  int32_t L, H, D, bs;       // layers, kv heads, head dim, block size (tokens)
  int32_t bs_shift;          // log2(bs): block size is a power of two
  int32_t bpe;               // bytes per element
  int32_t max_bpr;           // block-table row stride
  int64_t num_blocks;
  int64_t row_bytes;         // D * bpe
  int64_t block_stride;      // 2 * H * bs * row_bytes  (bytes between blocks in a layer)
  int64_t layer_stride;      // num_blocks * block_stride
  __host__ __device__ __forceinline__ int64_t seg_base(int l, int kv, int h) const {
    return (int64_t)l * layer_stride + ((int64_t)kv * H + h) * bs * row_bytes;
  }
};

// One request of a press batch (kernel-param descriptor, batch order sorted LPT).
struct PressReq {
  int32_t slot;      // device block-table row
  int32_t T;         // raw tokens
  int32_t K;         // kept tokens K_r
  int32_t seg0;      // tokens of the first modality segment (== T if single segment)
  int32_t K0;        // kept of the first segment (per-segment mode)
  int32_t q_idx;     // batch position (index into press inputs)
  int64_t kept_off;  // element offset into fc_press_outputs.kept_idx
  int64_t score_off; // element offset into fc_press_outputs.scores
};

struct PressBatch {
  int32_t n;
  int32_t per_segment;
  int32_t in_place;      // src table == dst table
  int32_t max_T;
  int32_t n_total;       // requests in the whole compress call (press-input rows)
  int32_t reserved;
  PressReq req[kMaxBatch];
};

// One request of a host-resident gather (fc_pool_compress_host_batch).
struct HostGatherReq {
  int32_t slot, T, K, reserved;
  int64_t kept_off;   // element offset of the request's [L][H][K] kept indices
  const char* host;   // device-mapped pointer of the pinned host [L][2][H][T][D] buffer
};
struct HostGatherBatch {
  int32_t n, reserved;
  HostGatherReq req[kMaxBatch];
};

// Decode over the compacted blocks (fc_decode.cu).
constexpr int kMaxDecode = 256;     // requests per decode launch
struct DecodeReq {
  int32_t slot, T;     // block-table row, live tokens
  int32_t item0;       // first CTA of this request (items = H * nsplit)
  int32_t nsplit;      // KV splits per kv head
  int32_t q_row;       // row of q / out
};
struct DecodeBatch {
  int32_t n, Hq, layer, split_tokens, items;
  DecodeReq req[kMaxDecode];
};
struct KVWriteReq {
  int32_t slot, pos, row;
};
struct KVWriteBatch {
  int32_t n, layer;
  KVWriteReq req[kMaxDecode];
};

// One request of a prefill K/V write (fc_pool_write_prefill_kv).
struct PrefillReq {
  int64_t row0;   // first row of this request in the varlen k / v buffers
  int64_t tok0;   // first handle token written
  int32_t slot, n;
};
struct PrefillBatch {
  int32_t n, layer;
  PrefillReq req[kMaxBatch];
};

struct PressParams {
  int32_t kind, factor, window, pool_kernel, n_sink, num_q_heads;
  // SEEDEDLINEAR: device table [factor][factor]; row m-1 = the reference's
  // renormalised weights w[:m] / w[:m].sum() for a chunk of m rows (kv.py:235-237).
  const double* w_table;
};

struct BlockOp {  // one request of a pop/push batch
  int32_t slot;
  int32_t from;   // first logical block
  int32_t count;  // blocks
  int32_t off;    // exclusive prefix of counts in this launch
};

struct BlockOpBatch {
  int32_t n;
  int32_t save_raw;  // legacy compress: copy the live row to the retained row first
  int32_t save_count[kMaxAllocBatch];
  BlockOp op[kMaxAllocBatch];
};

// ---------------------------------------------------------------------------
// element traits
// ---------------------------------------------------------------------------
template <typename T> struct Elem;
template <> struct Elem<__half> {
  static constexpr int kDtype = FC_F16;
  __device__ __forceinline__ static float to_f(__half x) { return __half2float(x); }
  __device__ __forceinline__ static __half from_f(float x) { return __float2half_rn(x); }
};
template <> struct Elem<__nv_bfloat16> {
  static constexpr int kDtype = FC_BF16;
  __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};
template <> struct Elem<float> {
  static constexpr int kDtype = FC_F32;
  __device__ __forceinline__ static float to_f(float x) { return x; }
  __device__ __forceinline__ static float from_f(float x) { return x; }
};

template <> struct Elem<double> {
  static constexpr int kDtype = FC_F64;
  __device__ __forceinline__ static double to_f(double x) { return x; }
  __device__ __forceinline__ static double from_f(double x) { return x; }
};

// 16-byte vector -> fp32 elements.
template <typename T>
__device__ __forceinline__ void unpack16(const uint4& v, float* out) {
  const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
  for (int i = 0; i < (int)(16 / sizeof(T)); ++i) out[i] = Elem<T>::to_f(e[i]);
}

// Streaming 128-bit global accesses. These never allocate in L1, so data this
// kernel later rewrites can never be served stale from L1.
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// Same load without `volatile`: the compiler may batch several of them ahead of their
// uses (only for data this kernel does not rewrite before reading it).
__device__ __forceinline__ uint4 ld_stream_nv(const void* p) {
  uint4 r;
  asm("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(void* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Order-preserving float -> uint32 key (larger float -> larger key).
__device__ __forceinline__ uint32_t float_key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// ---------------------------------------------------------------------------
// host-side launch helpers (defined in fc_pool.cu)
// ---------------------------------------------------------------------------
// SM count of the current device (queried once per device; 148 on B200): grids
// are sized in multiples of it.
int sm_count();
void note_launch();
// Which press implementation a launch used (tensor-core, SIMT, chunk fold): counted
// per thread so a compress call can report the path it took (fc_pool_last_paths).
enum PressPath { kPathTc = 0, kPathSimt = 1, kPathChunk = 2, kNumPaths = 3 };
void note_path(int path);
int64_t path_count(int path);
fc_status set_error(fc_status st, const char* fmt, ...);
fc_status cuda_check(cudaError_t e, const char* what);

// press kernels (fc_press.cu)
fc_status launch_press(const Geom& g, int dtype, char* arena, const int32_t* src_table,
                       int32_t* dst_table, const PressBatch& batch, const PressParams& pp,
                       const fc_press_inputs* in, const fc_press_outputs* out, float* workspace,
                       int64_t workspace_floats, int32_t* d_err, cudaStream_t stream,
                       bool dry_run = false);
bool snapkv_tc_supported(const Geom& g, int dtype, const PressParams& pp, int max_T, int max_K);
fc_status launch_snapkv_tc(const Geom& g, int dtype, char* arena, const int32_t* table,
                           const PressBatch& b, const PressParams& pp, const fc_press_inputs& in,
                           const fc_press_outputs& out, float* ws, int64_t ws_floats,
                           cudaStream_t stream, bool dry_run);
// spill rows of SnapKV tensor-core segments beyond its SMEM plan (0 if none)
int64_t snapkv_tc_workspace_floats(const Geom& g, int max_T, int max_K);
bool ea_tc_supported(const Geom& g, int dtype, const PressParams& pp, int max_T, int max_K);
fc_status launch_ea_tc(const Geom& g, int dtype, char* arena, const int32_t* table,
                       const PressBatch& b, const PressParams& pp, const fc_press_inputs& in,
                       const fc_press_outputs& out, int max_K, float* ws, int64_t ws_floats,
                       cudaStream_t stream, bool dry_run);
// spill rows of ExpectedAttention tensor-core segments beyond its SMEM plan (0 if none)
int64_t ea_tc_workspace_floats(const Geom& g, int num_q_heads, int max_T, int max_K);
int64_t press_workspace_floats(const Geom& g, int kind, int window, int num_q_heads, int max_T);

// decode kernels (fc_decode.cu)
fc_status launch_decode_attention(const Geom& g, int dtype, const char* arena, const int32_t* table,
                                  const DecodeBatch& b, int gq, const void* q, void* out,
                                  float scale_log2, float* ws, int32_t* counters,
                                  cudaStream_t stream);
fc_status launch_write_kv(const Geom& g, char* arena, const int32_t* table, const KVWriteBatch& b,
                          const void* k, const void* v, cudaStream_t stream);

// io kernels (fc_io.cu)
fc_status launch_synth(const Geom& g, int dtype, char* arena, const int32_t* table, int n,
                       const int32_t* slots, const int32_t* tokens, const uint64_t* keys,
                       uint64_t seed, int dist, cudaStream_t stream);
fc_status launch_store(const Geom& g, char* arena, const int32_t* table_row, int64_t tok_begin,
                       int64_t n_tok, const void* src, bool to_blocks, cudaStream_t stream,
                       int kv0 = 0, int nkv = 2);
// *used_tma (optional): 1 when the TMA ingest ran, 0 for the register-copy kernel
fc_status launch_write_prefill(const Geom& g, char* arena, const int32_t* table, int layer, int n,
                               const PrefillReq* reqs, const void* k, const void* v,
                               cudaStream_t stream, int* used_tma = nullptr);
fc_status launch_gather_host(const Geom& g, char* arena, const int32_t* table, int n,
                             const HostGatherReq* reqs, const int32_t* kept_idx, int kv,
                             cudaStream_t stream);
fc_status launch_compress_tensor(const void* src, int64_t n, int64_t d, int dtype,
                                 const PressParams& pp, void* dst, cudaStream_t stream);

}  // namespace fc
