// fc_press.cu -- batched press kernels of the FastCache compression stage.
//
// One CTA owns one (request, layer, kv-head) segment and runs three phases
// without leaving the SM (K1/K2/K3 -> K4 -> K5 fused):
//
//   1. score   -- stream the segment's K (and V for ExpectedAttention) out of
//                 its paged blocks with 128-bit loads; scores land in SMEM
//                 (T floats), never in HBM.
//   2. select  -- segmented top-K_r by (score desc, index asc): 4-pass 8-bit
//                 radix select on order-preserving uint32 keys, then a
//                 block-wide ballot scan emits the kept positions ascending.
//   3. compact -- copy kept K/V rows j <- idx[j] inside the request's own
//                 blocks. idx is ascending so idx[j] >= j: chunks of W ranks
//                 read all their sources, barrier, then write (safe in place;
//                 later chunks only read positions >= their own ranks). The
//                 identity prefix (idx[j] == j) is never touched.
//
// Algorithmic HBM bytes per segment: Knorm 0.5*R + 2*C;
// SnapKV adds the window queries; ExpectedAttention reads all of K and V.
//
// Reference anchors: K_r is the reference ceil rule (kv.py:169-194) computed
// by the host; the per-handle ledger transition that follows is pool.py:167-192.
#include <cfloat>
#include <climits>

#include "fc_select.cuh"

#ifndef FC_KN_MINB  // Knorm CTAs per SM the register budget is sized for
#define FC_KN_MINB 4
#endif

namespace fc {

// ---------------------------------------------------------------------------
// phase 1 scorers
// ---------------------------------------------------------------------------

// Knorm: s_t = -||K_t||_2, fp32, fixed summation order (oracle/press.py:knorm_scores).
template <typename T, int D>
__device__ __forceinline__ void score_knorm(const char* __restrict__ seg, const Geom& g,
                                            const int32_t* s_tab, int T_len, float* sc) {
  constexpr int kRowBytes = D * (int)sizeof(T);
  constexpr int kVecs = kRowBytes / 16;
  constexpr int kLPR = kVecs < 32 ? kVecs : 32;
  constexpr int kVPL = kVecs / kLPR;
  constexpr int kEPV = RowCfg<T>::kEPV;
  constexpr int kRPP = kThreads / kLPR;
  constexpr int kU = 4;
  // For 16-bit inputs x*x is exact in fp32, so fma(x, x, acc) rounds exactly
  // like fadd(fmul(x, x), acc) (the oracle's order) with half the instructions.
  constexpr bool kExactSquare = sizeof(T) == 2;
  const int lr = threadIdx.x % kLPR, rp = threadIdx.x / kLPR;
  // bulk L2 prefetch of whole block chunks (bs rows each) kPfIters iterations ahead
#ifndef FC_KN_SPF
#define FC_KN_SPF 2
#endif
  constexpr int kPfIters = FC_KN_SPF;
  const int chunk_bytes = g.bs * kRowBytes;
  auto prefetch_rows = [&](int r0, int r1) {
    if (kPfIters == 0) return;
    for (int c = (r0 >> g.bs_shift) + threadIdx.x; c < ((min(r1, T_len) + g.bs - 1) >> g.bs_shift);
         c += kThreads)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                       seg + (int64_t)s_tab[c] * g.block_stride),
                   "r"(chunk_bytes)
                   : "memory");
  };
  prefetch_rows(0, kPfIters * kRPP * kU);
  for (int t0 = 0; t0 < T_len; t0 += kRPP * kU) {
    prefetch_rows(t0 + kPfIters * kRPP * kU, t0 + (kPfIters + 1) * kRPP * kU);
    uint4 v[kU][kVPL];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int t = t0 + u * kRPP + rp;
      if (t < T_len) {
        const char* row = seg + (int64_t)s_tab[t >> g.bs_shift] * g.block_stride +
                          (int64_t)(t & (g.bs - 1)) * kRowBytes;
#pragma unroll
        for (int vv = 0; vv < kVPL; ++vv) v[u][vv] = ld_stream(row + (lr + vv * kLPR) * 16);
      } else {
#pragma unroll
        for (int vv = 0; vv < kVPL; ++vv) v[u][vv] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      float acc = 0.f;
#pragma unroll
      for (int vv = 0; vv < kVPL; ++vv) {
        float x[kEPV];
        unpack16<T>(v[u][vv], x);
#pragma unroll
        for (int e = 0; e < kEPV; ++e)
          acc = kExactSquare ? __fmaf_rn(x[e], x[e], acc) : __fadd_rn(acc, __fmul_rn(x[e], x[e]));
      }
#pragma unroll
      for (int off = kLPR / 2; off >= 1; off >>= 1)
        acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
      const int t = t0 + u * kRPP + rp;
      if (lr == 0 && t < T_len) sc[t] = -sqrtf(acc);
    }
  }
}

// Per-row L2 norm of V (any order; used by ExpectedAttention): sc[t] *= ||V_t||.
template <typename T, int D>
__device__ __forceinline__ void scale_by_vnorm(const char* __restrict__ seg_v, const Geom& g,
                                               const int32_t* s_tab, int t_begin, int T_len,
                                               float* sc) {
  constexpr int kVecs = D * (int)sizeof(T) / 16;
  constexpr int kLPR = kVecs < 32 ? kVecs : 32;
  constexpr int kVPL = kVecs / kLPR;
  constexpr int kEPV = RowCfg<T>::kEPV;
  constexpr int kRPP = kThreads / kLPR;
  const int lr = threadIdx.x % kLPR, rp = threadIdx.x / kLPR;
  for (int t0 = t_begin; t0 < T_len; t0 += kRPP) {
    const int t = t0 + rp;
    float acc = 0.f;
    if (t < T_len) {
      const char* row = seg_v + (int64_t)s_tab[t >> g.bs_shift] * g.block_stride +
                        (int64_t)(t & (g.bs - 1)) * g.row_bytes;
#pragma unroll
      for (int vv = 0; vv < kVPL; ++vv) {
        float x[kEPV];
        unpack16<T>(ld_stream(row + (lr + vv * kLPR) * 16), x);
#pragma unroll
        for (int e = 0; e < kEPV; ++e) acc = fmaf(x[e], x[e], acc);
      }
    }
#pragma unroll
    for (int off = kLPR / 2; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lr == 0 && t < T_len) sc[t] *= sqrtf(acc);
  }
}

// Load rows [t0, t0 + n) of a segment into SMEM as fp32 [n][ld].
template <typename T, int D>
__device__ __forceinline__ void load_rows_f32(const char* __restrict__ seg, const Geom& g,
                                              const int32_t* s_tab, int t0, int n, int T_len,
                                              float* dst, int ld) {
  constexpr int kVecs = D * (int)sizeof(T) / 16;
  constexpr int kEPV = RowCfg<T>::kEPV;
  for (int it = threadIdx.x; it < n * kVecs; it += kThreads) {
    const int r = it / kVecs, vec = it % kVecs;
    const int t = t0 + r;
    float x[kEPV];
    if (t < T_len) {
      const char* row = seg + (int64_t)s_tab[t >> g.bs_shift] * g.block_stride +
                        (int64_t)(t & (g.bs - 1)) * g.row_bytes;
      unpack16<T>(ld_stream(row + vec * 16), x);
    } else {
#pragma unroll
      for (int e = 0; e < kEPV; ++e) x[e] = 0.f;
    }
#pragma unroll
    for (int e = 0; e < kEPV; ++e) dst[r * ld + vec * kEPV + e] = x[e];
  }
}

__device__ __forceinline__ float block_reduce(float v, bool is_max, SelectScratch& s) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const float o = __shfl_xor_sync(0xffffffffu, v, off);
    v = is_max ? fmaxf(v, o) : v + o;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s.red[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = s.red[0];
  for (int w = 1; w < kWarps; ++w) r = is_max ? fmaxf(r, s.red[w]) : r + s.red[w];
  return r;
}

// SnapKV (SIMT, v1): window logits go to a per-CTA global workspace ws[w][T]
// (L2-resident), softmax per query over all T, mean over the window, avg-pool,
// mean over the query-head group; window tokens forced (+inf).
template <typename T, int D>
__device__ void score_snapkv(const char* __restrict__ seg, const Geom& g, const int32_t* s_tab,
                             int T_len, const PressParams& pp, const T* __restrict__ qwin,
                             float* sc, float* scratch, float* s1, float* __restrict__ ws,
                             SelectScratch& ss) {
  constexpr int kTile = 32;
  const int w = pp.window;
  const int gq = pp.num_q_heads / g.H;
  const int n_keep = T_len - w;  // scored positions
  float* qs = scratch;                         // [w][D+1]
  float* ks = qs + w * (D + 1);                // [kTile][D+1]
  float* mz = ks + kTile * (D + 1);            // [2][w]
  // s1 [T]: SMEM after mz, or a global spill row for segments beyond the SMEM plan
  const float inv_sqrt_d = 1.0f / sqrtf((float)D);
  for (int t = threadIdx.x; t < T_len; t += kThreads) sc[t] = 0.f;
  for (int qh = 0; qh < gq; ++qh) {
    const T* q = qwin + (int64_t)qh * w * D;
    for (int i = threadIdx.x; i < w * D; i += kThreads)
      qs[(i / D) * (D + 1) + (i % D)] = Elem<T>::to_f(q[i]);
    __syncthreads();
    // pass 1: logits -> ws, per-query running max
    const int jgroups = kThreads / 8;  // 32 query rows per sweep, 8 threads each
    for (int j0 = 0; j0 < w; j0 += jgroups) {
      const int j = j0 + threadIdx.x / 8;
      const int tt = threadIdx.x % 8;
      float m = -INFINITY;
      for (int t0 = 0; t0 < T_len; t0 += kTile) {
        __syncthreads();
        load_rows_f32<T, D>(seg, g, s_tab, t0, kTile, T_len, ks, D + 1);
        __syncthreads();
        if (j < w) {
          float a[4] = {0.f, 0.f, 0.f, 0.f};
          const float* qr = qs + j * (D + 1);
#pragma unroll 8
          for (int d = 0; d < D; ++d) {
            const float qv = qr[d];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = fmaf(qv, ks[(tt + 8 * i) * (D + 1) + d], a[i]);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int t = t0 + tt + 8 * i;
            if (t < T_len) {
              const float v = (t > T_len - w + j) ? -INFINITY : a[i] * inv_sqrt_d;
              ws[(int64_t)j * T_len + t] = v;
              m = fmaxf(m, v);
            }
          }
        }
      }
#pragma unroll
      for (int off = 4; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
      if (j < w && tt == 0) mz[j] = m;
    }
    __syncthreads();
    // pass 2: Z_j (warp per query row, lanes over t)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = warp; j < w; j += kWarps) {
      const float m = mz[j];
      float z = 0.f;
      for (int t = lane; t < T_len; t += 32) z += expf(ws[(int64_t)j * T_len + t] - m);
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
      if (lane == 0) mz[w + j] = 1.0f / z;
    }
    __syncthreads();
    // pass 3: s1[t] = mean_j softmax_j(t), t < T - w
    for (int t = threadIdx.x; t < n_keep; t += kThreads) {
      float acc = 0.f;
      for (int j = 0; j < w; ++j) acc += expf(ws[(int64_t)j * T_len + t] - mz[j]) * mz[w + j];
      s1[t] = acc / (float)w;
    }
    __syncthreads();
    // avg_pool1d(kernel p, stride 1, zero pad p//2, count_include_pad)
    const int half = pp.pool_kernel / 2;
    for (int t = threadIdx.x; t < n_keep; t += kThreads) {
      float acc = 0.f;
      for (int o = -half; o <= half; ++o) {
        const int u = t + o;
        acc += (u >= 0 && u < n_keep) ? s1[u] : 0.f;
      }
      sc[t] += acc / (float)pp.pool_kernel;
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < T_len; t += kThreads)
    sc[t] = (t >= n_keep) ? INFINITY : (gq > 1 ? sc[t] / (float)gq : sc[t]);
  (void)ss;
}

// ExpectedAttention (SIMT, v1): z_t = mu.K_t/sqrt(D) + K_t^T Sigma K_t/(2D),
// softmax over t >= n_sink, mean over the query group, times ||V_t||.
template <typename T, int D>
__device__ void score_ea(const char* __restrict__ seg, const Geom& g, const int32_t* s_tab,
                         int T_len, const PressParams& pp, const float* __restrict__ mu_g,
                         const float* __restrict__ cov_g, float* sc, float* scratch,
                         float* zt, SelectScratch& ss) {
  constexpr int kTokW = 4;                       // tokens per warp per sweep
  constexpr int kTile = kWarps * kTokW;          // 32 tokens per CTA sweep
  constexpr int kC = D / 32;                     // columns per lane
  const int gq = pp.num_q_heads / g.H;
  const int ns = pp.n_sink;
  float* sig = scratch;                          // [D][D]
  float* mu = sig + D * D;                       // [D]
  float* kt = mu + D;                            // [kTile][D]
  // zt [T]: SMEM after kt, or a global spill row for segments beyond the SMEM plan
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float inv_sqrt_d = 1.0f / sqrtf((float)D);
  const float inv_2d = 1.0f / (2.0f * (float)D);
  for (int t = threadIdx.x; t < T_len; t += kThreads) sc[t] = 0.f;
  for (int qh = 0; qh < gq; ++qh) {
    const float* cov = cov_g + (int64_t)qh * D * D;
    __syncthreads();
    for (int i = threadIdx.x; i < D * D / 4; i += kThreads)
      reinterpret_cast<float4*>(sig)[i] = reinterpret_cast<const float4*>(cov)[i];
    for (int i = threadIdx.x; i < D; i += kThreads) mu[i] = mu_g[(int64_t)qh * D + i];
    for (int t0 = ns; t0 < T_len; t0 += kTile) {
      __syncthreads();
      load_rows_f32<T, D>(seg, g, s_tab, t0, kTile, T_len, kt, D);
      __syncthreads();
      float u[kTokW][kC];
#pragma unroll
      for (int a = 0; a < kTokW; ++a)
#pragma unroll
        for (int c = 0; c < kC; ++c) u[a][c] = 0.f;
      const float* kw = kt + warp * kTokW * D;
      for (int i = 0; i < D; ++i) {
        float sv[kC];
#pragma unroll
        for (int c = 0; c < kC; ++c) sv[c] = sig[i * D + lane + 32 * c];
#pragma unroll
        for (int a = 0; a < kTokW; ++a) {
          const float ki = kw[a * D + i];
#pragma unroll
          for (int c = 0; c < kC; ++c) u[a][c] = fmaf(ki, sv[c], u[a][c]);
        }
      }
#pragma unroll
      for (int a = 0; a < kTokW; ++a) {
        float qf = 0.f, lin = 0.f;
#pragma unroll
        for (int c = 0; c < kC; ++c) {
          const float kj = kw[a * D + lane + 32 * c];
          qf = fmaf(kj, u[a][c], qf);
          lin = fmaf(kj, mu[lane + 32 * c], lin);
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          qf += __shfl_xor_sync(0xffffffffu, qf, off);
          lin += __shfl_xor_sync(0xffffffffu, lin, off);
        }
        const int t = t0 + warp * kTokW + a;
        if (lane == 0 && t < T_len) zt[t] = lin * inv_sqrt_d + qf * inv_2d;
      }
    }
    __syncthreads();
    float m = -INFINITY;
    for (int t = ns + threadIdx.x; t < T_len; t += kThreads) m = fmaxf(m, zt[t]);
    m = block_reduce(m, true, ss);
    float z = 0.f;
    for (int t = ns + threadIdx.x; t < T_len; t += kThreads) z += expf(zt[t] - m);
    z = block_reduce(z, false, ss);
    const float inv_z = 1.0f / z;
    for (int t = ns + threadIdx.x; t < T_len; t += kThreads) sc[t] += expf(zt[t] - m) * inv_z;
  }
  __syncthreads();
  if (gq > 1)
    for (int t = threadIdx.x; t < T_len; t += kThreads) sc[t] /= (float)gq;
  __syncthreads();
  scale_by_vnorm<T, D>(seg + (int64_t)g.H * g.bs * g.row_bytes, g, s_tab, ns, T_len, sc);
  __syncthreads();
  for (int t = threadIdx.x; t < ns && t < T_len; t += kThreads) sc[t] = INFINITY;
}

// ---------------------------------------------------------------------------
// phase 3: in-place compaction of kept rows
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// the fused kernel
// ---------------------------------------------------------------------------
#ifndef FC_KNORM_ASYNC  // Knorm compaction through a cp.async SMEM ring (fc_select.cuh)
#define FC_KNORM_ASYNC 1
#endif
#ifndef FC_KN_RANKS
#define FC_KN_RANKS 16
#endif
#ifndef FC_KN_BUFS
#define FC_KN_BUFS 4
#endif
constexpr int kKnRanks = FC_KN_RANKS, kKnBufs = FC_KN_BUFS;

struct SmemPlan {
  int nb;          // table entries per table
  int tab_bytes;   // both tables
  int sc_bytes;    // scores
  int scratch_bytes;
  int cbuf_bytes;  // Knorm: cp.async compaction ring
  __host__ __device__ int total() const { return tab_bytes + sc_bytes + scratch_bytes + cbuf_bytes; }
};

__host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

// spill: the segment is longer than the SMEM plan allows. Block tables are then read
// straight from global memory, and the T-sized arrays (scores -> keys -> kept indices,
// SnapKV's window mean, EA's logits) live in a per-CTA global row (L2-resident) instead
// of SMEM; nothing else changes. spill_floats() is that row's length.
__host__ __device__ inline SmemPlan smem_plan(int kind, int max_T, int bs, int D, int window,
                                              bool in_place, int row_bytes = 256,
                                              bool spill = false) {
  SmemPlan p;
  p.nb = (max_T + bs - 1) / bs;
  p.tab_bytes = spill ? 0 : align16(p.nb * 4) * (in_place ? 1 : 2);
  p.sc_bytes = spill ? 0 : align16(max_T * 4);
  p.scratch_bytes = 0;
  p.cbuf_bytes = (FC_KNORM_ASYNC && kind == FC_PRESS_KNORM) ? kKnBufs * kKnRanks * 2 * row_bytes : 0;
  const int t_arr = spill ? 0 : ((max_T + 3) & ~3);
  if (kind == FC_PRESS_SNAPKV)
    p.scratch_bytes = align16((window * (D + 1) + 32 * (D + 1) + 2 * window + t_arr) * 4);
  else if (kind == FC_PRESS_EXPECTED_ATTENTION)
    p.scratch_bytes = align16((D * D + D + kWarps * 4 * D + t_arr) * 4);
  return p;
}

__host__ __device__ inline int64_t spill_floats(int kind, int max_T) {
  const int64_t t = (max_T + 3) & ~3;
  return kind == FC_PRESS_KNORM ? t : 2 * t;
}

constexpr int kSmemLimit = 220 * 1024;   // SIMT press plans above this take the spill variant
constexpr int kSpillCtasPerSm = 2;

template <typename T, int D, int KIND, bool kSpill>
__global__ void __launch_bounds__(kThreads, KIND == FC_PRESS_KNORM ? FC_KN_MINB : 2)
    press_kernel(char* __restrict__ arena, const int32_t* __restrict__ src_table,
                 const int32_t* __restrict__ dst_table, const Geom g,
                 const __grid_constant__ PressBatch b, const PressParams pp,
                 const fc_press_inputs in, const fc_press_outputs out, float* __restrict__ ws,
                 int64_t ws_per_cta, int n_items, float* __restrict__ spill) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ SelectScratch ss;
  const SmemPlan plan = smem_plan(KIND, b.max_T, g.bs, D, pp.window, b.in_place != 0,
                                  D * (int)sizeof(T), kSpill);
  int32_t* s_src = reinterpret_cast<int32_t*>(smem);
  int32_t* s_dst = b.in_place ? s_src : s_src + plan.tab_bytes / 8;
  const int64_t t_pad = (b.max_T + 3) & ~3;
  float* sc = kSpill ? spill + (int64_t)blockIdx.x * spill_floats(KIND, b.max_T)
                     : reinterpret_cast<float*>(smem + plan.tab_bytes);
  float* scratch = reinterpret_cast<float*>(smem + plan.tab_bytes + plan.sc_bytes);
  // SnapKV's window mean / EA's logits: after the fixed scratch in SMEM, or spilled
  float* tarr = kSpill ? sc + t_pad
                       : scratch + (KIND == FC_PRESS_SNAPKV
                                        ? pp.window * (D + 1) + 32 * (D + 1) + 2 * pp.window
                                        : D * D + D + kWarps * 4 * D);
  const int LH = g.L * g.H;

  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int r = item / LH, lh = item % LH;
    const int l = lh / g.H, h = lh % g.H;
    const PressReq q = b.req[r];
    const int T_len = q.T, K = q.K;
    const int nb = (T_len + g.bs - 1) / g.bs;
    __syncthreads();  // previous item's SMEM fully consumed
    if (kSpill) {     // tables read in place (the kernel never writes them)
      s_src = const_cast<int32_t*>(src_table) + (int64_t)q.slot * g.max_bpr;
      s_dst = b.in_place ? s_src : const_cast<int32_t*>(dst_table) + (int64_t)q.slot * g.max_bpr;
    } else {
      for (int i = threadIdx.x; i < nb; i += kThreads) {
        s_src[i] = src_table[(int64_t)q.slot * g.max_bpr + i];
        if (!b.in_place) s_dst[i] = dst_table[(int64_t)q.slot * g.max_bpr + i];
      }
    }
    if (threadIdx.x == 0) ss.first_drop = INT_MAX;
    __syncthreads();
    char* seg = arena + g.seg_base(l, 0, h);

    // ---- phase 1: score ----
    if constexpr (KIND == FC_PRESS_KNORM) {
      score_knorm<T, D>(seg, g, s_src, T_len, sc);
    } else if constexpr (KIND == FC_PRESS_SNAPKV) {
      const int gq = pp.num_q_heads / g.H;
      const T* qwin = reinterpret_cast<const T*>(in.q_window) +
                      (((int64_t)q.q_idx * g.L + l) * pp.num_q_heads + (int64_t)h * gq) * pp.window * D;
      score_snapkv<T, D>(seg, g, s_src, T_len, pp, qwin, sc, scratch, tarr,
                         ws + (int64_t)blockIdx.x * ws_per_cta, ss);
    } else {
      const int gq = pp.num_q_heads / g.H;
      const int64_t qoff = ((int64_t)q.q_idx * g.L + l) * pp.num_q_heads + (int64_t)h * gq;
      score_ea<T, D>(seg, g, s_src, T_len, pp, in.mean_q + qoff * D, in.cov_q + qoff * D * D, sc,
                     scratch, tarr, ss);
    }
    __syncthreads();
    if (out.scores) {
      float* so = out.scores + q.score_off + (int64_t)lh * T_len;
      for (int t = threadIdx.x; t < T_len; t += kThreads) so[t] = sc[t];
    }
    uint32_t* keys = reinterpret_cast<uint32_t*>(sc);
    for (int t = threadIdx.x; t < T_len; t += kThreads) keys[t] = float_key(sc[t]);
    __syncthreads();

    // ---- phase 2: select (kept positions overwrite the keys, ascending) ----
    int32_t* idx = reinterpret_cast<int32_t*>(sc);
    select_request(keys, T_len, K, q.seg0, q.K0, b.per_segment, idx, ss);
    if (out.kept_idx) {
      int32_t* ko = out.kept_idx + q.kept_off + (int64_t)lh * K;
      for (int j = threadIdx.x; j < K; j += kThreads) ko[j] = idx[j];
    }
    const int first_moved = b.in_place ? min(ss.first_drop, K) : 0;

    // ---- phase 3: compact K and V rows into the destination blocks ----
    if (FC_KNORM_ASYNC && KIND == FC_PRESS_KNORM)
      compact_rows_async<D * (int)sizeof(T), CtaGroup, kKnRanks, kKnBufs>(
          seg, g, s_src, s_dst, idx, K, first_moved,
          smem + plan.tab_bytes + plan.sc_bytes + plan.scratch_bytes);
    else
      compact_rows<D * (int)sizeof(T)>(seg, g, s_src, s_dst, idx, K, first_moved);
  }
}

// ---------------------------------------------------------------------------
// K7 in-pool chunk compressor (reference compress_tensor per modality segment)
// ---------------------------------------------------------------------------
// Output row r of segment s is the fold of source rows [sb + (r-ob)*k, ...):
// MEAN_POOL: sequential fp32 sum (fp64 for fp64) then IEEE division by the
// row count, cast to the pool dtype (numpy mean semantics, kv.py:227-231);
// SEEDED_LINEAR: fp64 weighted sum with the renormalised weights, rounded to
// the pool dtype (the reference returns fp64; the pool stores its dtype).
#ifndef FC_CHUNK_ITEMS   // output vectors per thread per chunk (c2m: 2 -> 4.69 ms, 4 -> 3.81, 8 spills)
#define FC_CHUNK_ITEMS 4
#endif
#ifndef FC_CHUNK_MINB   // chunk-fold CTAs per SM the register budget is sized for (c2m: 3 -> 4.56 ms, 4 -> 3.81, 5 / 6 spill: 5.63 / 8.12)
#define FC_CHUNK_MINB 4
#endif
template <typename T, int D, bool kSeeded>
__global__ void __launch_bounds__(kThreads, kSeeded ? 2 : FC_CHUNK_MINB)
    chunk_pool_kernel(char* __restrict__ arena, const int32_t* __restrict__ src_table,
                      const int32_t* __restrict__ dst_table, const Geom g,
                      const __grid_constant__ PressBatch b, const PressParams pp) {
  constexpr int kVecs = D * (int)sizeof(T) / 16;
  constexpr int kEPV = RowCfg<T>::kEPV;
  constexpr int kItems = FC_CHUNK_ITEMS;   // output vectors per thread per chunk
  constexpr int kChunk = kThreads * kItems / (2 * kVecs);
  extern __shared__ __align__(16) unsigned char smem[];
  const int LH = g.L * g.H;
  const int r = blockIdx.x / LH, lh = blockIdx.x % LH;
  const int l = lh / g.H, h = lh % g.H;
  const PressReq q = b.req[r];
  const int nb = (q.T + g.bs - 1) / g.bs;
  int32_t* s_src = reinterpret_cast<int32_t*>(smem);
  int32_t* s_dst = b.in_place ? s_src : s_src + align16(nb * 4) / 4;
  for (int i = threadIdx.x; i < nb; i += kThreads) {
    s_src[i] = src_table[(int64_t)q.slot * g.max_bpr + i];
    if (!b.in_place) s_dst[i] = dst_table[(int64_t)q.slot * g.max_bpr + i];
  }
  __syncthreads();
  char* seg = arena + g.seg_base(l, 0, h);
  const int64_t kv_off = (int64_t)g.H * g.bs * g.row_bytes;
  const int k = pp.factor;
  const int seg0 = q.seg0, K0 = q.K0;
  for (int j0 = 0; j0 < q.K; j0 += kChunk) {
    uint4 res[kItems];
    // per item: source base row, row count m, and the byte offset of its vector
    int s_first[kItems], m_rows[kItems];
    int64_t voff[kItems];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int item = it * kThreads + threadIdx.x;
      const int row = item / (2 * kVecs), rem = item % (2 * kVecs);
      const int kv = rem / kVecs, vec = rem % kVecs;
      const int j = j0 + row;
      const bool second = j >= K0;   // output row j's modality segment
      const int sb = second ? seg0 : 0, ob = second ? K0 : 0, se = second ? q.T : seg0;
      s_first[it] = sb + (j - ob) * k;
      m_rows[it] = j < q.K ? min(k, se - s_first[it]) : 0;
      voff[it] = kv * kv_off + vec * 16;
    }
    float accf[kItems][kEPV];
    double accd[kSeeded ? kItems : 1][kEPV];
#pragma unroll
    for (int it = 0; it < kItems; ++it)
#pragma unroll
      for (int e = 0; e < kEPV; ++e) {
        accf[it][e] = 0.f;
        if (kSeeded) accd[it][e] = 0.0;
      }
    // row i of every item's chunk is loaded together (kItems independent 16-B loads in
    // flight per thread), then folded in the reference order: the accumulation chain is
    // per item, so only the HBM latency of one row step is exposed per i
    auto fold = [&](int it, int i, const uint4& raw) {
      float x[kEPV];
      unpack16<T>(raw, x);
      if (!kSeeded) {
#pragma unroll
        for (int e = 0; e < kEPV; ++e) accf[it][e] = (i == 0) ? x[e] : __fadd_rn(accf[it][e], x[e]);
      } else {
        const double wi = pp.w_table[(int64_t)(m_rows[it] - 1) * k + i];
#pragma unroll
        for (int e = 0; e < kEPV; ++e) accd[it][e] = fma(wi, (double)x[e], accd[it][e]);
      }
    };
    auto load = [&](int it, int i) {
      const int src = s_first[it] + i;
      return ld_stream_nv(seg + voff[it] + (int64_t)s_src[src >> g.bs_shift] * g.block_stride +
                          (int64_t)(src & (g.bs - 1)) * g.row_bytes);
    };
    // row i of every item's chunk is loaded together (kItems independent 16-B loads in
    // flight per thread), then folded in the reference's sequential row order. (Two rows
    // per step was measured slower: 5.20 vs 4.52 ms at c2m, the extra registers cost a
    // CTA per SM.)
    for (int i = 0; i < k; ++i) {
      uint4 v[kItems];
#pragma unroll
      for (int it = 0; it < kItems; ++it)
        if (i < m_rows[it]) v[it] = load(it, i);
#pragma unroll
      for (int it = 0; it < kItems; ++it)
        if (i < m_rows[it]) fold(it, i, v[it]);
    }
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      T o[kEPV];
      const int m = max(m_rows[it], 1);
#pragma unroll
      for (int e = 0; e < kEPV; ++e) {
        if (!kSeeded)
          o[e] = Elem<T>::from_f(__fdiv_rn(accf[it][e], (float)m));
        else
          o[e] = Elem<T>::from_f((float)accd[it][e]);
      }
      res[it] = *reinterpret_cast<uint4*>(o);
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int item = it * kThreads + threadIdx.x;
      const int row = item / (2 * kVecs), rem = item % (2 * kVecs);
      const int kv = rem / kVecs, vec = rem % kVecs;
      const int j = j0 + row;
      if (j < q.K)
        st_stream(seg + kv * kv_off + (int64_t)s_dst[j >> g.bs_shift] * g.block_stride +
                      (int64_t)(j & (g.bs - 1)) * g.row_bytes + vec * 16,
                  res[it]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// host dispatch
// ---------------------------------------------------------------------------
// SnapKV SIMT window logits (ws[w][T] per CTA, up to 4 CTAs per SM) + the spill rows of
// segments beyond the SMEM plan (kSpillCtasPerSm per SM).
static int64_t snap_ws_floats(int kind, int window, int max_T) {
  return kind == FC_PRESS_SNAPKV ? (int64_t)sm_count() * 4 * window * max_T : 0;
}

static bool needs_spill(const Geom& g, int kind, int window, int max_T, bool in_place) {
  if (kind > FC_PRESS_EXPECTED_ATTENTION) return false;
  return smem_plan(kind, max_T, g.bs, g.D, window, in_place, g.D * g.bpe).total() > kSmemLimit;
}

int64_t press_workspace_floats(const Geom& g, int kind, int window, int num_q_heads, int max_T) {
  int64_t n = snap_ws_floats(kind, window, max_T);
  if (needs_spill(g, kind, window, max_T, /*in_place=*/false))
    n += (int64_t)sm_count() * kSpillCtasPerSm * spill_floats(kind, max_T);
  if (kind == FC_PRESS_EXPECTED_ATTENTION)   // the tensor-core kernels' spill rows (K <= T)
    n = std::max(n, ea_tc_workspace_floats(g, num_q_heads, max_T, max_T));
  if (kind == FC_PRESS_SNAPKV)
    n = std::max(n, snapkv_tc_workspace_floats(g, max_T, max_T));
  return n;
}

template <typename T, int D, int KIND>
static fc_status launch_one(const Geom& g, char* arena, const int32_t* src, int32_t* dst,
                            const PressBatch& b, const PressParams& pp, const fc_press_inputs& in,
                            const fc_press_outputs& out, float* ws, int64_t ws_floats,
                            cudaStream_t stream, bool dry) {
  const int n_items = b.n * g.L * g.H;
  if (KIND == FC_PRESS_MEANPOOL || KIND == FC_PRESS_SEEDEDLINEAR) {
    const int nb = (b.max_T + g.bs - 1) / g.bs;
    const int smem = align16(nb * 4) * 2;
    if (smem > kDynSmemBudget)
      return set_error(FC_ERR_UNSUPPORTED, "request of %d tokens exceeds the chunk-fold SMEM plan", b.max_T);
    if (dry) return FC_OK;
    auto kern = pp.kind == FC_PRESS_SEEDEDLINEAR ? chunk_pool_kernel<T, D, true>
                                                 : chunk_pool_kernel<T, D, false>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<n_items, kThreads, smem, stream>>>(arena, src, dst, g, b, pp);
    note_launch();
    note_path(kPathChunk);
    return cuda_check(cudaGetLastError(), "chunk_pool_kernel");
  }
  if ((KIND == FC_PRESS_SNAPKV || KIND == FC_PRESS_EXPECTED_ATTENTION) && b.in_place) {
    auto tc_ok = [&](int max_T, int max_K) {
      return KIND == FC_PRESS_SNAPKV ? snapkv_tc_supported(g, Elem<T>::kDtype, pp, max_T, max_K)
                                     : ea_tc_supported(g, Elem<T>::kDtype, pp, max_T, max_K);
    };
    auto run_tc = [&](const PressBatch& bb, int max_K) {
      return KIND == FC_PRESS_SNAPKV
                 ? launch_snapkv_tc(g, Elem<T>::kDtype, arena, src, bb, pp, in, out, ws, ws_floats,
                                    stream, dry)
                 : launch_ea_tc(g, Elem<T>::kDtype, arena, src, bb, pp, in, out, max_K, ws, ws_floats,
                                stream, dry);
    };
    int max_K = 1;
    for (int i = 0; i < b.n; ++i) max_K = max_K > b.req[i].K ? max_K : b.req[i].K;
    if (tc_ok(b.max_T, max_K)) return run_tc(b, max_K);
    // The tensor-core kernels size SMEM by the batch's longest request: when only
    // some requests fit, split -- those go to the tensor-core kernel, the rest to
    // the SIMT kernel (independent segments, so the split changes no result).
    PressBatch fit = b, rest = b;
    fit.n = rest.n = 0;
    fit.max_T = rest.max_T = 0;
    int fit_K = 1;
    for (int i = 0; i < b.n; ++i) {
      const PressReq& q = b.req[i];
      PressBatch& dst = tc_ok(q.T, q.K > 0 ? q.K : 1) ? fit : rest;
      dst.req[dst.n++] = q;
      dst.max_T = std::max(dst.max_T, q.T);
      if (&dst == &fit) fit_K = std::max(fit_K, q.K);
    }
    if (fit.n > 0 && rest.n > 0 && tc_ok(fit.max_T, fit_K)) {
      fc_status st = run_tc(fit, fit_K);
      if (st != FC_OK) return st;
      return launch_one<T, D, KIND>(g, arena, src, dst, rest, pp, in, out, ws, ws_floats, stream, dry);
    }
  }
  constexpr int kKind = KIND == FC_PRESS_KNORM ? FC_PRESS_KNORM
                       : KIND == FC_PRESS_SNAPKV ? FC_PRESS_SNAPKV
                                                 : FC_PRESS_EXPECTED_ATTENTION;
  const bool spill = smem_plan(KIND, b.max_T, g.bs, D, pp.window, b.in_place != 0,
                               D * (int)sizeof(T)).total() > kSmemLimit;
  const SmemPlan plan = smem_plan(KIND, b.max_T, g.bs, D, pp.window, b.in_place != 0,
                                  D * (int)sizeof(T), spill);
  const int smem = plan.total();
  if (smem > kSmemLimit)
    return set_error(FC_ERR_UNSUPPORTED, "request of %d tokens exceeds the SMEM budget", b.max_T);
  const int sms = sm_count();
  const int64_t snap_ws = snap_ws_floats(KIND, pp.window, b.max_T);
  const int64_t spill_row = spill_floats(KIND, b.max_T);
  if (dry) return FC_OK;   // the pool sizes the workspace (press_workspace_floats) next
  if (spill && ws_floats - snap_ws < spill_row)
    return set_error(FC_ERR_INVALID_STATE, "press workspace too small for the spill rows");
  auto kern = spill ? press_kernel<T, D, kKind, true> : press_kernel<T, D, kKind, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute");
  int grid = n_items;
  int64_t ws_per_cta = 0;
  if (KIND == FC_PRESS_SNAPKV) {
    ws_per_cta = (int64_t)pp.window * b.max_T;
    grid = (int)std::min<int64_t>(n_items, std::min<int64_t>((int64_t)sms * 4, snap_ws / ws_per_cta));
  }
  float* spill_base = nullptr;
  if (spill) {
    spill_base = ws + snap_ws;
    grid = (int)std::min<int64_t>(grid, std::min<int64_t>((int64_t)sms * kSpillCtasPerSm,
                                                          (ws_floats - snap_ws) / spill_row));
  }
  kern<<<grid, kThreads, smem, stream>>>(arena, src, dst, g, b, pp, in, out, ws, ws_per_cta,
                                         n_items, spill_base);
  note_launch();
  note_path(kPathSimt);
  return cuda_check(cudaGetLastError(), "press_kernel");
}

template <typename T, int D>
static fc_status dispatch_kind(int kind, const Geom& g, char* arena, const int32_t* src,
                               int32_t* dst, const PressBatch& b, const PressParams& pp,
                               const fc_press_inputs& in, const fc_press_outputs& out, float* ws,
                               int64_t wsf, cudaStream_t s, bool dry) {
  switch (kind) {
    case FC_PRESS_KNORM:
      return launch_one<T, D, FC_PRESS_KNORM>(g, arena, src, dst, b, pp, in, out, ws, wsf, s, dry);
    case FC_PRESS_SNAPKV:
      return launch_one<T, D, FC_PRESS_SNAPKV>(g, arena, src, dst, b, pp, in, out, ws, wsf, s, dry);
    case FC_PRESS_EXPECTED_ATTENTION:
      return launch_one<T, D, FC_PRESS_EXPECTED_ATTENTION>(g, arena, src, dst, b, pp, in, out, ws, wsf, s, dry);
    default:
      return launch_one<T, D, FC_PRESS_MEANPOOL>(g, arena, src, dst, b, pp, in, out, ws, wsf, s, dry);
  }
}

template <typename T>
static fc_status dispatch_dim(int kind, const Geom& g, char* arena, const int32_t* src,
                              int32_t* dst, const PressBatch& b, const PressParams& pp,
                              const fc_press_inputs& in, const fc_press_outputs& out, float* ws,
                              int64_t wsf, cudaStream_t s, bool dry) {
  switch (g.D) {
    case 64: return dispatch_kind<T, 64>(kind, g, arena, src, dst, b, pp, in, out, ws, wsf, s, dry);
    case 128: return dispatch_kind<T, 128>(kind, g, arena, src, dst, b, pp, in, out, ws, wsf, s, dry);
    case 256: return dispatch_kind<T, 256>(kind, g, arena, src, dst, b, pp, in, out, ws, wsf, s, dry);
    default: return set_error(FC_ERR_UNSUPPORTED, "head_dim %d has no compiled press kernel", g.D);
  }
}

fc_status launch_press(const Geom& g, int dtype, char* arena, const int32_t* src_table,
                       int32_t* dst_table, const PressBatch& batch, const PressParams& pp,
                       const fc_press_inputs* in_p, const fc_press_outputs* out_p, float* ws,
                       int64_t ws_floats, int32_t* d_err, cudaStream_t stream, bool dry) {
  (void)d_err;
  fc_press_inputs in{};
  fc_press_outputs out{};
  if (in_p) in = *in_p;
  if (out_p) out = *out_p;
  switch (dtype) {
    case FC_F16:
      return dispatch_dim<__half>(pp.kind, g, arena, src_table, dst_table, batch, pp, in, out, ws, ws_floats, stream, dry);
    case FC_BF16:
      return dispatch_dim<__nv_bfloat16>(pp.kind, g, arena, src_table, dst_table, batch, pp, in, out, ws, ws_floats, stream, dry);
    case FC_F32:
      return dispatch_dim<float>(pp.kind, g, arena, src_table, dst_table, batch, pp, in, out, ws, ws_floats, stream, dry);
    default:
      return set_error(FC_ERR_UNSUPPORTED, "press kernels need an f16/bf16/f32 pool");
  }
}

}  // namespace fc
