// fc_io.cu -- payload movement kernels: the K8 synthetic KV generator, dense
// <-> paged token copies (prefill ingest, P.Store of PAPER.md:246), and the
// standalone K7 compress_tensor (reference kv.py:211-239).
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

#include "fc_internal.cuh"
#include "fc_tc.cuh"

namespace fc {

// ---------------------------------------------------------------------------
// K8: counter-based generator, bit-identical to oracle/synth.py
// ---------------------------------------------------------------------------
constexpr int kMaxSynth = 256;
struct SynthBatch {
  int32_t n;
  int32_t slot[kMaxSynth];
  int32_t T[kMaxSynth];
  uint64_t key[kMaxSynth];
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t splitmix(uint64_t z) { return mix64(z + 0x9E3779B97F4A7C15ull); }

template <typename T>
__global__ void __launch_bounds__(256)
    synth_fill_kernel(char* __restrict__ arena, const int32_t* __restrict__ table, const Geom g,
                      const __grid_constant__ SynthBatch b, uint64_t seed, int dist) {
  constexpr int kEPV = 16 / (int)sizeof(T);
  const int r = blockIdx.y;
  const int T_len = b.T[r];
  const int vpr = (int)(g.row_bytes / 16);
  const int64_t total = (int64_t)g.L * 2 * g.H * T_len * vpr;
  const uint64_t req = splitmix(seed ^ splitmix(b.key[r]));
  const int32_t* row_tab = table + (int64_t)b.slot[r] * g.max_bpr;
  const float inv_std = 0x1.bb67aep-16f;  // f32(1 / 37837.227), oracle/synth.py INV_STD
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int vec = (int)(v % vpr);
    int64_t rest = v / vpr;
    const int t = (int)(rest % T_len);
    rest /= T_len;
    const int h = (int)(rest % g.H);
    rest /= g.H;
    const int kv = (int)(rest % 2);
    const int l = (int)(rest / 2);
    const uint64_t head = splitmix(req ^ (((uint64_t)l << 24) | ((uint64_t)kv << 23) | (uint64_t)h));
    const uint64_t row = splitmix(head ^ (uint64_t)t);
    float scale = 1.0f;
    if (dist == FC_SYNTH_SCALED) {
      const float a = __fmul_rn(__uint2float_rn((uint32_t)(row >> 40)), 0x1p-24f);
      scale = __fadd_rn(0.5f, __fmul_rn(a, 1.5f));
    }
    T out[kEPV];
#pragma unroll
    for (int e = 0; e < kEPV; ++e) {
      const uint64_t d1 = (uint64_t)(vec * kEPV + e) + 1ull;
      const uint64_t el = mix64(row + d1 * 0x9E3779B97F4A7C15ull);
      const int64_t s = (int64_t)(el & 0xFFFF) + (int64_t)((el >> 16) & 0xFFFF) +
                        (int64_t)((el >> 32) & 0xFFFF) + (int64_t)(el >> 48);
      float x = __fmul_rn(__int2float_rn((int)(s - 131070)), inv_std);
      if (dist == FC_SYNTH_SCALED) x = __fmul_rn(x, scale);
      out[e] = Elem<T>::from_f(x);
    }
    char* dst = arena + g.seg_base(l, kv, h) + (int64_t)row_tab[t / g.bs] * g.block_stride +
                (int64_t)(t % g.bs) * g.row_bytes + vec * 16;
    st_stream(dst, *reinterpret_cast<uint4*>(out));
  }
}

fc_status launch_synth(const Geom& g, int dtype, char* arena, const int32_t* table, int n,
                       const int32_t* slots, const int32_t* tokens, const uint64_t* keys,
                       uint64_t seed, int dist, cudaStream_t stream) {
  for (int c = 0; c < n; c += kMaxSynth) {
    SynthBatch b;
    memset(&b, 0, sizeof(b));
    b.n = n - c < kMaxSynth ? n - c : kMaxSynth;
    int64_t max_vecs = 0;
    for (int i = 0; i < b.n; ++i) {
      b.slot[i] = slots[c + i];
      b.T[i] = tokens[c + i];
      b.key[i] = keys[c + i];
      const int64_t vv = (int64_t)g.L * 2 * g.H * b.T[i] * (g.row_bytes / 16);
      max_vecs = vv > max_vecs ? vv : max_vecs;
    }
    int64_t gx = (max_vecs + 255) / 256;
    const int64_t cap = ((int64_t)sm_count() * 8 * 4 + b.n - 1) / b.n;
    if (gx > cap) gx = cap;
    if (gx < 1) gx = 1;
    dim3 grid((unsigned)gx, (unsigned)b.n);
    switch (dtype) {
      case FC_F16: synth_fill_kernel<__half><<<grid, 256, 0, stream>>>(arena, table, g, b, seed, dist); break;
      case FC_BF16: synth_fill_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(arena, table, g, b, seed, dist); break;
      case FC_F32: synth_fill_kernel<float><<<grid, 256, 0, stream>>>(arena, table, g, b, seed, dist); break;
      default: return set_error(FC_ERR_UNSUPPORTED, "synth fill dtype");
    }
    note_launch();
    fc_status st = cuda_check(cudaGetLastError(), "synth_fill_kernel");
    if (st != FC_OK) return st;
  }
  return FC_OK;
}

// ---------------------------------------------------------------------------
// dense [L][nkv][H][n][D] <-> paged blocks (nkv = 2: K and V; nkv = 1: only
// kv plane kv0, the K-only ingest of the host-resident compress path)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    store_tokens_kernel(char* __restrict__ arena, const int32_t* __restrict__ row_tab, const Geom g,
                        int64_t tok_begin, int64_t n_tok, char* __restrict__ dense, int to_blocks,
                        int kv0, int nkv) {
  const int vpr = (int)(g.row_bytes / 16);
  const int64_t total = (int64_t)g.L * nkv * g.H * n_tok * vpr;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int vec = (int)(v % vpr);
    int64_t rest = v / vpr;
    const int64_t i = rest % n_tok;
    rest /= n_tok;
    const int h = (int)(rest % g.H);
    rest /= g.H;
    const int kv = kv0 + (int)(rest % nkv);
    const int l = (int)(rest / nkv);
    const int64_t t = tok_begin + i;
    char* blk = arena + g.seg_base(l, kv, h) + (int64_t)row_tab[t / g.bs] * g.block_stride +
                (t % g.bs) * g.row_bytes + vec * 16;
    char* dn = dense + v * 16;
    if (to_blocks)
      st_stream(blk, ld_stream(dn));
    else
      st_stream(dn, ld_stream(blk));
  }
}

fc_status launch_store(const Geom& g, char* arena, const int32_t* table_row, int64_t tok_begin,
                       int64_t n_tok, const void* src, bool to_blocks, cudaStream_t stream,
                       int kv0, int nkv) {
  if (((uintptr_t)src) % 16) return set_error(FC_ERR_INVALID_ARG, "dense buffer must be 16-byte aligned");
  const int64_t total = (int64_t)g.L * nkv * g.H * n_tok * (g.row_bytes / 16);
  int64_t grid = (total + 255) / 256;
  if (grid > (int64_t)sm_count() * 16) grid = (int64_t)sm_count() * 16;
  store_tokens_kernel<<<(unsigned)grid, 256, 0, stream>>>(arena, table_row, g, tok_begin, n_tok,
                                                          (char*)src, to_blocks ? 1 : 0, kv0, nkv);
  note_launch();
  return cuda_check(cudaGetLastError(), "store_tokens_kernel");
}

// ---------------------------------------------------------------------------
// Host-resident compress, second half: kept V rows read straight from pinned
// host memory (zero-copy over PCIe, UVA) into rank slots of the request's
// blocks. Host layout per request: [L][2][H][T][D]; V row (l, h, t) is
// row_bytes contiguous bytes. Every thread keeps kUnroll 16-B loads in flight
// so the PCIe read pipe (~2 us latency) stays full; measured 51.5 GB/s for
// 256-B rows at 25-50% density (scripts/pcie_probe.cu).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    gather_host_rows_kernel(char* __restrict__ arena, const int32_t* __restrict__ table,
                            const Geom g, const __grid_constant__ HostGatherBatch b,
                            const int32_t* __restrict__ kept_idx, int kv) {
  constexpr int kUnroll = 4;
  const HostGatherReq q = b.req[blockIdx.y];
  const int vpr = (int)(g.row_bytes / 16);
  const int64_t total = (int64_t)g.L * g.H * q.K * vpr;
  const int32_t* row_tab = table + (int64_t)q.slot * g.max_bpr;
  const int32_t* idx = kept_idx + q.kept_off;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < total;
       v0 += stride * kUnroll) {
    uint4 buf[kUnroll];
    char* dst[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t v = v0 + u * stride;
      dst[u] = nullptr;
      if (v < total) {
        const int vec = (int)(v % vpr);
        const int64_t rest = v / vpr;           // (l*H + h)*K + j
        const int j = (int)(rest % q.K);
        const int lh = (int)(rest / q.K);
        const int l = lh / g.H, h = lh % g.H;
        const int src = idx[rest];
        buf[u] = ld_stream(q.host + ((((int64_t)l * 2 + kv) * g.H + h) * q.T + src) * g.row_bytes +
                           vec * 16);
        dst[u] = arena + g.seg_base(l, kv, h) + (int64_t)row_tab[j >> g.bs_shift] * g.block_stride +
                 (int64_t)(j & (g.bs - 1)) * g.row_bytes + vec * 16;
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (dst[u]) st_stream(dst[u], buf[u]);
  }
}

fc_status launch_gather_host(const Geom& g, char* arena, const int32_t* table, int n,
                             const HostGatherReq* reqs, const int32_t* kept_idx, int kv,
                             cudaStream_t stream) {
  for (int c = 0; c < n; c += kMaxBatch) {
    HostGatherBatch b;
    memset(&b, 0, sizeof(b));
    b.n = n - c < kMaxBatch ? n - c : kMaxBatch;
    int64_t max_vecs = 0;
    for (int i = 0; i < b.n; ++i) {
      b.req[i] = reqs[c + i];
      const int64_t vv = (int64_t)g.L * g.H * b.req[i].K * (g.row_bytes / 16);
      max_vecs = vv > max_vecs ? vv : max_vecs;
    }
    int64_t gx = (max_vecs + 1023) / 1024;
    const int64_t cap = ((int64_t)sm_count() * 8 + b.n - 1) / b.n;
    if (gx > cap) gx = cap;
    if (gx < 1) gx = 1;
    gather_host_rows_kernel<<<dim3((unsigned)gx, (unsigned)b.n), 256, 0, stream>>>(arena, table, g, b,
                                                                                  kept_idx, kv);
    note_launch();
    fc_status st = cuda_check(cudaGetLastError(), "gather_host_rows_kernel");
    if (st != FC_OK) return st;
  }
  return FC_OK;
}

// ---------------------------------------------------------------------------
// K7 standalone: compress_tensor on a dense (n, d) matrix
// ---------------------------------------------------------------------------
template <typename X> struct Acc { using type = float; };
template <> struct Acc<double> { using type = double; };
template <typename X>
__device__ __forceinline__ typename Acc<X>::type to_acc(X x) {
  return (typename Acc<X>::type)Elem<X>::to_f(x);
}

// numpy pairwise_sum of a contiguous run (umath loops_utils), for the (m, 1) case.
template <typename A>
__device__ A pairwise_sum(const A* a, int n) {
  if (n < 8) {
    A r = (A)0;
    for (int i = 0; i < n; ++i) r = r + a[i];
    return r;
  }
  if (n <= 128) {
    A r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = r[j] + a[i + j];
    A res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res = res + a[i];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_sum<A>(a, n2) + pairwise_sum<A>(a + n2, n - n2);
}

template <typename X>
__global__ void __launch_bounds__(256)
    compress_tensor_kernel(const X* __restrict__ src, int64_t n, int64_t d, PressParams pp,
                           void* __restrict__ dst) {
  using A = typename Acc<X>::type;
  const int64_t k = pp.factor;
  const int64_t rows = (n + k - 1) / k;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < rows * d;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = o / d, c = o % d;
    const int64_t first = r * k;
    const int m = (int)((n - first) < k ? (n - first) : k);
    if (pp.kind == FC_PRESS_MEANPOOL) {
      A s;
      if (d == 1 && (sizeof(X) == 4 || sizeof(X) == 8) && Elem<X>::kDtype != FC_BF16) {
        s = pairwise_sum<A>(reinterpret_cast<const A*>(src) + first, m);
      } else {
        s = to_acc<X>(src[first * d + c]);
        for (int i = 1; i < m; ++i) s = s + to_acc<X>(src[(first + i) * d + c]);
      }
      const A mean = s / (A)m;
      reinterpret_cast<X*>(dst)[o] = Elem<X>::from_f(mean);
    } else {
      const double* w = pp.w_table + ((m == k) ? 0 : k);
      double s = 0.0;
      for (int i = 0; i < m; ++i) s = fma(w[i], (double)to_acc<X>(src[(first + i) * d + c]), s);
      reinterpret_cast<double*>(dst)[o] = s;
    }
  }
}

fc_status launch_compress_tensor(const void* src, int64_t n, int64_t d, int dtype,
                                 const PressParams& pp, void* dst, cudaStream_t stream) {
  const int64_t rows = (n + pp.factor - 1) / pp.factor;
  int64_t grid = (rows * d + 255) / 256;
  if (grid > (int64_t)sm_count() * 16) grid = (int64_t)sm_count() * 16;
  if (grid < 1) grid = 1;
  switch (dtype) {
    case FC_F16:
      compress_tensor_kernel<__half><<<(unsigned)grid, 256, 0, stream>>>((const __half*)src, n, d, pp, dst);
      break;
    case FC_BF16:
      compress_tensor_kernel<__nv_bfloat16><<<(unsigned)grid, 256, 0, stream>>>((const __nv_bfloat16*)src, n, d, pp, dst);
      break;
    case FC_F32:
      compress_tensor_kernel<float><<<(unsigned)grid, 256, 0, stream>>>((const float*)src, n, d, pp, dst);
      break;
    case FC_F64:
      compress_tensor_kernel<double><<<(unsigned)grid, 256, 0, stream>>>((const double*)src, n, d, pp, dst);
      break;
    default:
      return set_error(FC_ERR_UNSUPPORTED, "compress_tensor dtype");
  }
  note_launch();
  return cuda_check(cudaGetLastError(), "compress_tensor_kernel");
}


// ---------------------------------------------------------------------------
// P.Store: one layer of the prefill's K/V for a batch of
// requests, varlen layout k, v = [sum_i n_i][H][D] (request i's rows start at
// cu[i]), written to tokens tok0[i] + j of each handle's blocks. One 16-B
// vector per thread; reads are fully coalesced, writes land as 256-B rows in
// the (layer, K|V, head) chunk of their block.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    write_prefill_kernel(char* __restrict__ arena, const int32_t* __restrict__ table, const Geom g,
                         const __grid_constant__ PrefillBatch b, const char* __restrict__ k,
                         const char* __restrict__ v) {
  const PrefillReq rq = b.req[blockIdx.y];
  const int vpr = (int)(g.row_bytes / 16);
  // token-major order: the reads stream the varlen rows; each token's 2*H rows of
  // 256 B land in their (K|V, head) chunks (a chunk-contiguous order that streams
  // the writes instead measured 11% slower)
  const int64_t per_tok = (int64_t)2 * g.H * vpr;
  const int64_t total = (int64_t)rq.n * per_tok;
  const int32_t* row_tab = table + (int64_t)rq.slot * g.max_bpr;
#ifndef FC_PF_UNROLL
#define FC_PF_UNROLL 2
#endif
  constexpr int kUnroll = FC_PF_UNROLL;  // independent 16-B loads in flight per thread
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t x0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x0 < total; x0 += stride * kUnroll) {
    uint4 buf[kUnroll];
    char* dst[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t x = x0 + u * stride;
      dst[u] = nullptr;
      if (x < total) {
        const int64_t j = x / per_tok;
        const int rem = (int)(x - j * per_tok);
        const int kv = rem / (g.H * vpr), hv = rem % (g.H * vpr);
        const int h = hv / vpr, vec = hv % vpr;
        buf[u] = ld_stream((kv ? v : k) + ((rq.row0 + j) * g.H + h) * g.row_bytes + vec * 16);
        const int64_t t = rq.tok0 + j;
        dst[u] = arena + g.seg_base(b.layer, kv, h) + (int64_t)row_tab[t >> g.bs_shift] * g.block_stride +
                 (t & (g.bs - 1)) * g.row_bytes + vec * 16;
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (dst[u]) st_stream(dst[u], buf[u]);
  }
}

// ---------------------------------------------------------------------------
// P.Store through the copy engines: one TMA load brings a (request, pool block,
// K|V, head group) tile -- bs tokens x hg heads of the varlen [rows][H][D] source,
// landed head-major by a 3-D tensor map whose head stride is the inner one -- into a
// 3-stage SMEM ring; each head's bs rows then leave as ONE contiguous bulk store of
// its bs * D * bpe pool chunk (partial blocks at a request's edges go row by row).
// One thread per CTA issues everything: per 64-KB tile one load and hg stores, so
// HBM sees whole 4-KB chunk writes and 8-KB row reads instead of 16-B thread traffic.
// ---------------------------------------------------------------------------
// measured at c2p (16-KB tiles, 5 loads ahead, 2 CTAs per SM): 5.57 ms = 1.00 of the
// copy peak; 3 stages 6.05 ms, 4: 6.16, 7: 5.58; 8 / 12 stages (one CTA per SM) 8.2-9.2 ms;
// 8-KB tiles 6.4-7.9 ms, 32-KB 5.9-6.1 ms; the register kernel below 6.48 ms (0.86)
#ifndef FC_PF_STAGES
#define FC_PF_STAGES 6
#endif
constexpr int kPfStages = FC_PF_STAGES;
#ifndef FC_PF_DEFER   // park the block id one tile later (measured slower: 5.83 vs 5.58 ms)
#define FC_PF_DEFER 0
#endif
#ifndef FC_PF_AHEAD
#define FC_PF_AHEAD (FC_PF_STAGES - 1)
#endif
constexpr int kPfAhead = FC_PF_AHEAD;
static_assert(kPfAhead >= 1 && kPfAhead < kPfStages, "prefill ring: loads ahead < stages");
struct PrefillTmaBatch {
  int32_t n, layer, hg, nhg;
  int32_t item0[kMaxBatch + 1];   // first work item of request i (prefix over requests)
  PrefillReq req[kMaxBatch];
};

__global__ void __launch_bounds__(32, 1)
    write_prefill_tma_kernel(char* __restrict__ arena, const int32_t* __restrict__ table, const Geom g,
                             const __grid_constant__ PrefillTmaBatch b,
                             const __grid_constant__ CUtensorMap kmap,
                             const __grid_constant__ CUtensorMap vmap, int stage_bytes) {
  extern __shared__ __align__(128) unsigned char pf_smem[];
  __shared__ __align__(8) uint64_t full[kPfStages];
  __shared__ int64_t s_dst[kPfStages];   // pool chunk base of the tile's first head
  if (threadIdx.x != 0) return;
  for (int i = 0; i < kPfStages; ++i) tc::mbar_init(&full[i], 1);
  tc::fence_barrier_init();
  tc::tma_prefetch_desc(&kmap);
  tc::tma_prefetch_desc(&vmap);
  const int n_items = b.item0[b.n];
  const int cnt = n_items > (int)blockIdx.x ? (n_items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  struct Tile { int r, kv, hg0; int64_t blk, lo, hi; };
  auto decode = [&](int i) {
    const int item = (int)blockIdx.x + i * (int)gridDim.x;
    int lo_r = 0, hi_r = b.n - 1;   // last request with item0 <= item
    while (lo_r < hi_r) {
      const int mid = (lo_r + hi_r + 1) >> 1;
      if (b.item0[mid] <= item) lo_r = mid; else hi_r = mid - 1;
    }
    const PrefillReq& q = b.req[lo_r];
    int x = item - b.item0[lo_r];
    Tile t;
    t.r = lo_r;
    t.hg0 = (x % b.nhg) * b.hg;
    x /= b.nhg;
    t.kv = x & 1;
    t.blk = (q.tok0 >> g.bs_shift) + (x >> 1);
    t.lo = max(q.tok0, t.blk << g.bs_shift);
    t.hi = min(q.tok0 + q.n, (t.blk + 1) << g.bs_shift);
    return t;
  };
  // the block id of a tile is read when its load is issued (FC_PF_DEFER: parked in
  // s_dst one tile later)
  int32_t pend_blk = 0;
  int pend_st = -1;
  int64_t pend_base = 0;
  auto park = [&]() {
    if (pend_st >= 0) s_dst[pend_st] = pend_base + (int64_t)pend_blk * g.block_stride;
    pend_st = -1;
  };
  auto issue_load = [&](int i) {
    park();
    const int st = i % kPfStages;
    const Tile t = decode(i);
    const PrefillReq& q = b.req[t.r];
    tc::mbar_expect_tx(&full[st], (uint32_t)stage_bytes);
    tc::tma_load_3d(pf_smem + (int64_t)st * stage_bytes, t.kv ? &vmap : &kmap, &full[st], 0,
                    (int)(q.row0 + (t.lo - q.tok0)), t.hg0);
    pend_blk = __ldg(table + (int64_t)q.slot * g.max_bpr + t.blk);
    pend_base = g.seg_base(b.layer, t.kv, t.hg0);
    pend_st = st;
    if (!FC_PF_DEFER) park();
  };
  // kPfAhead loads in flight ahead of the tile being stored; the other
  // kPfStages - kPfAhead stages hold tiles whose bulk stores are still reading SMEM
  for (int i = 0; i < kPfAhead && i < cnt; ++i) issue_load(i);
  const int64_t chunk = (int64_t)g.bs * g.row_bytes;
  for (int i = 0; i < cnt; ++i) {
    const int st = i % kPfStages;
    const Tile t = decode(i);
    tc::mbar_wait(&full[st], (uint32_t)((i / kPfStages) & 1));
    park();
    const unsigned char* src = pf_smem + (int64_t)st * stage_bytes;
    char* dst = arena + s_dst[st];
    const int64_t rows = t.hi - t.lo, r0 = t.lo & (g.bs - 1);
    for (int hh = 0; hh < b.hg; ++hh) {
      // head hh's chunk is H-adjacent in the pool: (K|V, head) chunks follow each other
      char* d = dst + (int64_t)hh * chunk;
      const unsigned char* s_h = src + (int64_t)hh * chunk;
      if (rows == g.bs) {
        tc::bulk_s2g(d, s_h, (uint32_t)chunk);
      } else {
        for (int64_t rr = 0; rr < rows; ++rr)
          tc::bulk_s2g(d + (r0 + rr) * g.row_bytes, s_h + rr * g.row_bytes, (uint32_t)g.row_bytes);
      }
    }
    tc::bulk_commit();
    const int nxt = i + kPfAhead;
    if (nxt < cnt) {
      // tile nxt - kPfStages (the stage's last user) has kPfStages - kPfAhead newer
      // store groups; it must have finished reading SMEM
      tc::bulk_wait_read<kPfStages - kPfAhead>();
      issue_load(nxt);
    }
  }
  tc::bulk_wait_all();
}

static PFN_cuTensorMapEncodeTiled_v12000 io_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// [rows][H][D] varlen source viewed as {D, rows, H} (head stride innermost after D), box
// {D, bs, hg}: the tile lands head-major, each head's bs rows contiguous.
static bool encode_prefill_src(CUtensorMap* map, const void* base, const Geom& g, int64_t rows, int hg) {
  auto enc = io_encode();
  if (!enc) return false;
  const CUtensorMapDataType dt = g.bpe == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : g.bpe == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                              : CU_TENSOR_MAP_DATA_TYPE_UINT32;
  const cuuint64_t dims[3] = {(cuuint64_t)g.D, (cuuint64_t)rows, (cuuint64_t)g.H};
  const cuuint64_t strides[2] = {(cuuint64_t)g.H * g.row_bytes, (cuuint64_t)g.row_bytes};
  const cuuint32_t box[3] = {(cuuint32_t)g.D, (cuuint32_t)g.bs, (cuuint32_t)hg};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#ifndef FC_PF_TMA
#define FC_PF_TMA 1
#endif
#ifndef FC_PF_STAGE_BYTES
#define FC_PF_STAGE_BYTES 16384
#endif

// Returns false (nothing launched) when the geometry does not suit the TMA path.
static bool launch_write_prefill_tma(const Geom& g, char* arena, const int32_t* table, int layer, int n,
                                     const PrefillReq* reqs, const void* k, const void* v,
                                     cudaStream_t stream, fc_status* status) {
  if (!FC_PF_TMA || g.D > 256 || g.bs > 256) return false;
  if ((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) & 15) return false;
  const int64_t chunk = (int64_t)g.bs * g.row_bytes;
  int hg = 1;
  while (hg * 2 <= g.H && g.H % (hg * 2) == 0 && hg * 2 <= 256 && chunk * hg * 2 <= FC_PF_STAGE_BYTES) hg *= 2;
  if (chunk * hg > FC_PF_STAGE_BYTES) return false;
  const int stage_bytes = (int)(chunk * hg);
  const int smem = kPfStages * stage_bytes;
  *status = FC_OK;
  for (int c = 0; c < n; c += kMaxBatch) {
    PrefillTmaBatch b;
    memset(&b, 0, sizeof(b));
    b.n = n - c < kMaxBatch ? n - c : kMaxBatch;
    b.layer = layer;
    b.hg = hg;
    b.nhg = g.H / hg;
    int64_t rows = 1, items = 0;
    for (int i = 0; i < b.n; ++i) {
      const PrefillReq& q = reqs[c + i];
      b.req[i] = q;
      b.item0[i] = (int32_t)items;
      if (q.n > 0) {
        const int64_t nblk = ((q.tok0 + q.n - 1) >> g.bs_shift) - (q.tok0 >> g.bs_shift) + 1;
        items += nblk * 2 * b.nhg;
      }
      rows = std::max<int64_t>(rows, q.row0 + q.n);
    }
    if (items > INT32_MAX) return false;
    b.item0[b.n] = (int32_t)items;
    if (items == 0) continue;
    CUtensorMap kmap, vmap;
    if (!encode_prefill_src(&kmap, k, g, rows, hg) || !encode_prefill_src(&vmap, v, g, rows, hg)) {
      if (c == 0) return false;
      *status = set_error(FC_ERR_CUDA, "cuTensorMapEncodeTiled(prefill) failed");
      return true;
    }
    cudaError_t e = cudaFuncSetAttribute(write_prefill_tma_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) {
      *status = cuda_check(e, "cudaFuncSetAttribute(write_prefill_tma)");
      return true;
    }
    const int grid = (int)std::min<int64_t>(items, (int64_t)sm_count() * std::max(1, (227 * 1024) / (smem + 1024)));
    write_prefill_tma_kernel<<<grid, 32, smem, stream>>>(arena, table, g, b, kmap, vmap, stage_bytes);
    note_launch();
    *status = cuda_check(cudaGetLastError(), "write_prefill_tma_kernel");
    if (*status != FC_OK) return true;
  }
  return true;
}

fc_status launch_write_prefill(const Geom& g, char* arena, const int32_t* table, int layer, int n,
                               const PrefillReq* reqs, const void* k, const void* v,
                               cudaStream_t stream, int* used_tma) {
  fc_status tma_status;
  const bool tma = launch_write_prefill_tma(g, arena, table, layer, n, reqs, k, v, stream, &tma_status);
  if (used_tma) *used_tma = tma ? 1 : 0;
  if (tma) return tma_status;
  for (int c = 0; c < n; c += kMaxBatch) {
    PrefillBatch b;
    memset(&b, 0, sizeof(b));
    b.n = n - c < kMaxBatch ? n - c : kMaxBatch;
    b.layer = layer;
    int64_t max_vecs = 0;
    for (int i = 0; i < b.n; ++i) {
      b.req[i] = reqs[c + i];
      const int64_t vv = (int64_t)b.req[i].n * 2 * g.H * (g.row_bytes / 16);
      max_vecs = vv > max_vecs ? vv : max_vecs;
    }
    if (max_vecs == 0) continue;
#ifndef FC_PF_CTAS
#define FC_PF_CTAS 64
#endif
    int64_t gx = (max_vecs + 4095) / 4096;
    const int64_t cap = ((int64_t)sm_count() * FC_PF_CTAS + b.n - 1) / b.n;
    if (gx > cap) gx = cap;
    if (gx < 1) gx = 1;
    write_prefill_kernel<<<dim3((unsigned)gx, (unsigned)b.n), 256, 0, stream>>>(arena, table, g, b,
                                                                               (const char*)k,
                                                                               (const char*)v);
    note_launch();
    fc_status st = cuda_check(cudaGetLastError(), "write_prefill_kernel");
    if (st != FC_OK) return st;
  }
  return FC_OK;
}

}  // namespace fc
