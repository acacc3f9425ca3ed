// fc_ea_tc.cu -- ExpectedAttention scoring on the 5th-gen tensor cores (sm_100a).
//
//   z_t = mu . K_t / sqrt(D) + K_t^T Sigma K_t / (2D),  p = softmax_{t >= n_sink}(z),
//   s_t = p_t * ||V_t||,  s_{t < n_sink} = +inf
//
// Persistent and warp-specialised like fc_snapkv_tc.cu. Per (request, layer,
// kv-head) segment the tensor cores compute Y = K_tile . B^T with
//   B = [ Sigma^T ; mu ; 0 ]   (144 x D, fp16),  D_tile[t][n<128] = (K Sigma)[t][n],
//                                                D_tile[t][128]  = K_t . mu,
// where Sigma and mu (fp32 inputs) are split into fp16 hi + lo parts and both
// halves accumulate into the same TMEM tile (~2^-22 relative per element; K
// in fp16 is exact). The consumer warps finish q_t = sum_n Y[t][n] K[t][n]
// in fp32 from the K rows still in SMEM.
//
//   warp 0     TMA producer. Per segment the SMEM ring carries, in order:
//              the segment's K tiles, the NEXT segment's Sigma (2 x 32 KB fp32
//              stages), then the segment's V tiles (for ||V_t||).
//   warp 1     MMA issuer: 2 x 8 tcgen05.mma (M=128, N=144, K=16) per K tile
//              into a 2-slot TMEM ring (2 x 256 columns).
//   warps 2-9  consumers: Sigma -> B conversion (hi/lo split, transpose,
//              128-byte swizzle), z_t epilogue from TMEM + SMEM, softmax,
//              V norms, segmented radix top-k -> hand-off.
//   warps 10-17 compactors: in-place compaction of kept K/V rows.
//
// Algorithmic bytes per segment: R + 2C + (D + D^2) * 4.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstring>
#include <mutex>

#include "fc_select.cuh"
#include "fc_tc.cuh"

namespace fc {

#ifdef FC_TRACE
// Debug build only (make trace): per-CTA, per-segment %globaltimer stamps.
__device__ unsigned long long g_fc_trace_ea[148 * 64 * 8];
__device__ __forceinline__ void ea_stamp(int it, int slot) {
  if (it < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_fc_trace_ea[(blockIdx.x * 64 + it) * 8 + slot] = t;
  }
}
#define EA_STAMP(it, slot) ea_stamp(it, slot)
#else
#define EA_STAMP(it, slot) ((void)0)
#endif

namespace ea {

constexpr int kD = 128;
constexpr int kStages = 3;                      // TMA ring depth (GQA: 2, see ea_stages)
__host__ __device__ constexpr int ea_stages(bool gqa, bool spill = false) {
  return gqa && !spill ? 2 : kStages;
}
constexpr int kTileM = 128;
constexpr int kBRows = 144;                     // 128 Sigma^T rows + mu + 15 zero rows
#ifndef FC_EA_CITEMS  // compactor 16-B loads in flight per thread per chunk
#define FC_EA_CITEMS 8
#endif
#ifndef FC_EA_CPF  // compactor L2 prefetch distance in chunks (0 measured best: 41.2 vs 42.4 ms at 2)
#define FC_EA_CPF 0
#endif
#ifndef FC_EA_SLOTS
#define FC_EA_SLOTS 3
#endif
constexpr int kSlots = FC_EA_SLOTS;              // TMEM ring depth (MMA runs kSlots tiles ahead)
constexpr int kSlotCols = kSlots == 2 ? 256 : 160;  // slot stride (N = 144 used)
constexpr int kTmemCols = 512;                  // power-of-two allocation >= kSlots * kSlotCols
constexpr int kMaxChunks = 16;                  // tile rows / smallest block size (8)
constexpr int kStageBytes = kTileM * kD * 2;    // 32 KB: one K/V tile or half of Sigma (fp32)
constexpr int kBHalf = kBRows * 128;            // one 64-column slab of B (bytes)
constexpr int kBBytes = 2 * kBHalf;             // one full B matrix (hi or lo)
constexpr int kConsumerFirst = 64;
constexpr int kCompactorFirst = kConsumerFirst + kThreads;
#ifndef FC_EA_GQA_COMP_WARPS   // compactor warps of the GQA instantiation (8 = as g = 1)
#define FC_EA_GQA_COMP_WARPS 4
#endif
// GQA: g units of K . Sigma_h per segment keep the consumers busy while the compactors
// idle; 4 compactor warps make the CTA 14 warps, so every warp may hold 128 registers.
#ifndef FC_EA_COMP_WARPS   // compactor warps of the g = 1 instantiation
// (its compaction is bytes-in-flight bound: c4w 43.1 ms at 8 warps x 8 loads, 50.8 ms at
// 6 x 8, 43.1 ms at 6 x 12 with the consumers at 128 registers, 74 ms at 4 x 12)
#define FC_EA_COMP_WARPS 8
#endif
__host__ __device__ constexpr int ea_comp_threads(bool gqa) {
  return 32 * (gqa ? FC_EA_GQA_COMP_WARPS : FC_EA_COMP_WARPS);
}
__host__ __device__ constexpr int ea_threads(bool gqa) { return kCompactorFirst + ea_comp_threads(gqa); }
constexpr int kEaThreads = ea_threads(false);
using Consumers = NamedGroup<kConsumerFirst, 1>;

struct Job {
  int32_t l, h, K, first_moved, slot;
};

struct Smem {
  int max_nb, max_K;
  int off_ring, off_b, off_zt, off_acc, off_idx, off_ctab, off_bar, total;
};

// GQA gives one ring stage (32 KB) to the per-head probability sum so that
// segments up to ~8k tokens still fit the 227-KB SMEM plan. Longer segments take
// the spill variant: z_t / keys, the GQA sum and the kept-index hand-off live in a
// per-CTA global row (spill_row_floats), the compactors read the block table in
// place, and SMEM holds only the TMA ring, B and the barriers -- any T fits.
__host__ __device__ inline Smem plan(int bs, int max_T, int max_K, bool gqa = false,
                                     bool spill = false) {
  Smem p;
  p.max_nb = (max_T + bs - 1) / bs;
  p.max_K = max_K;
  p.off_ring = 0;
  p.off_b = p.off_ring + ea_stages(gqa, spill) * kStageBytes;
  p.off_zt = p.off_b + 2 * kBBytes;
  if (spill) {
    p.off_acc = p.off_idx = p.off_ctab = p.off_bar = p.off_zt;
  } else {
    p.off_acc = p.off_zt + ((max_T * 4 + 15) & ~15);              // GQA: sum over heads of p_t
    p.off_idx = p.off_acc + (gqa ? ((max_T * 4 + 15) & ~15) : 0);
    p.off_ctab = p.off_idx + 2 * ((max_K * 4 + 15) & ~15);
    p.off_bar = p.off_ctab + 2 * ((p.max_nb * 4 + 15) & ~15);
  }
  p.total = p.off_bar + 64 * 8 + 1024;
  return p;
}

__host__ __device__ inline int64_t spill_row_floats(int max_T, int max_K, bool gqa) {
  const int64_t tp = (max_T + 3) & ~3, kp = (max_K + 3) & ~3;
  return tp * (gqa ? 2 : 1) + 2 * kp;
}

// Positions of one segment's stages in the global FIFO ring sequence:
//   [Sigma(first) x2] then per segment: [K tiles][V tiles][Sigma(next) x2 if any].
// The MMA warp waits only on K-tile positions, so it must never be able to
// wait on a stage more than one phase ahead of the producer (mbarrier parity
// waits alias two phases apart). With Sigma(next) LAST, the MMA can only pass
// b_full after the consumers released every earlier position, so the first
// K tile it waits on is exactly one phase ahead of its stage's last release.
// (The old order [K][Sigma(next)][V] let the MMA reach the next K tile while
// V stages were still in flight: a parity alias fed it a V tile, or hung it.)
// GQA (gq query heads per kv head): one "unit" per head, each unit's K tiles
// preceded by its own Sigma, so the sequence per segment is
//   [K(u0)][Sigma(u1) x2][K(u1)] ... [K(u_last)][V tiles][Sigma(next seg, u0) x2]
// and the MMA still only ever waits on K stages right after a Sigma it has
// seen converted (b_full), which keeps the one-phase-ahead invariant.
struct SegPos {
  int k0, v0, sig_next, next, unit_stride;
  __device__ __forceinline__ int k_unit(int u) const { return k0 + u * unit_stride; }
  __device__ __forceinline__ int sig_unit(int u) const { return k0 + (u - 1) * unit_stride + unit_stride - 2; }
};
__device__ __forceinline__ SegPos seg_pos(int start, int ntiles, bool has_next, int gq = 1) {
  SegPos s;
  s.k0 = start;
  s.unit_stride = ntiles + 2;                    // K tiles + the next unit's Sigma
  s.v0 = start + gq * ntiles + 2 * (gq - 1);
  s.sig_next = s.v0 + ntiles;
  s.next = s.sig_next + (has_next ? 2 : 0);
  return s;
}

// byte offset of B[n][k] (fp16) in the 128B-swizzled K-major layout
__device__ __forceinline__ int b_off(int n, int k) {
  const int half = k >> 6, c = (k & 63) >> 3, e = k & 7, r = n & 7;
  return half * kBHalf + (n >> 3) * 1024 + r * 128 + ((c ^ r) << 4) + e * 2;
}

}  // namespace ea

using namespace ea;

// T = __half or __nv_bfloat16: the K/V tiles' type; Sigma / mu are split into
// hi + lo parts of the same type (fp16: ~22 significant bits, bf16: ~16).
template <typename T, bool kGqa, bool kSpill>
__global__ void __launch_bounds__(ea_threads(kGqa), 1)
    ea_tc_kernel(char* __restrict__ arena, const int32_t* __restrict__ table, const Geom g,
                 const __grid_constant__ PressBatch b, const PressParams pp,
                 const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap cmap,
                 const float* __restrict__ mean_q, const fc_press_outputs out, int n_items,
                 int max_K, float* __restrict__ spill) {
  extern __shared__ unsigned char smem_raw[];
  __shared__ SelectScratch ss;
  __shared__ uint32_t s_tmem;
  __shared__ Job s_job[2];
  __shared__ float s_stat[2];

  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  constexpr int kStages = ea_stages(kGqa, kSpill);
  const Smem P = plan(g.bs, b.max_T, max_K, kGqa, kSpill);
  const int gq = kGqa ? pp.num_q_heads / g.H : 1;
  unsigned char* ring = smem + P.off_ring;
  unsigned char* bmat = smem + P.off_b;  // [hi | lo]
  const int k_stride = ((max_K * 4 + 15) & ~15) / 4;
  const int nb_stride = ((P.max_nb * 4 + 15) & ~15) / 4;
  float* const row = kSpill ? spill + (int64_t)blockIdx.x * spill_row_floats(b.max_T, max_K, kGqa)
                            : nullptr;
  const int64_t t_pad = (b.max_T + 3) & ~3;
  float* zt = kSpill ? row : reinterpret_cast<float*>(smem + P.off_zt);
  float* pacc = kSpill ? row + t_pad : reinterpret_cast<float*>(smem + P.off_acc);   // kGqa
  int32_t* idxbuf = kSpill ? reinterpret_cast<int32_t*>(row + t_pad * (kGqa ? 2 : 1))
                           : reinterpret_cast<int32_t*>(smem + P.off_idx);
  int32_t* ctab = reinterpret_cast<int32_t*>(smem + P.off_ctab);   // unused when kSpill
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P.off_bar);
  uint64_t* st_full = bars;                  // [kStages]
  uint64_t* st_empty = bars + kStages;       // [kStages] 8 arrivals (consumer warps)
  uint64_t* sl_full = bars + 2 * kStages;    // [kSlots]
  uint64_t* sl_empty = sl_full + kSlots;     // [kSlots] 8 arrivals
  uint64_t* b_full = sl_empty + kSlots;
  uint64_t* b_empty = b_full + 1;
  uint64_t* job_full = b_empty + 1;          // [2]
  uint64_t* job_empty = job_full + 2;        // [2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int LH = g.L * g.H;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&st_full[i], 1);
      tc::mbar_init(&st_empty[i], kWarps);
    }
    for (int i = 0; i < kSlots; ++i) {
      tc::mbar_init(&sl_full[i], 1);
      tc::mbar_init(&sl_empty[i], kWarps);
    }
    tc::mbar_init(b_full, 1);
    tc::mbar_init(b_empty, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&job_full[i], 1);
      tc::mbar_init(&job_empty[i], 1);
    }
    tc::fence_barrier_init();
    tc::tma_prefetch_desc(&kmap);
    tc::tma_prefetch_desc(&cmap);
  }
  // zero the B rows that carry no data (129..143 of hi and lo) once
  for (int i = threadIdx.x; i < 2 * 2 * 16 * 128 / 16; i += blockDim.x) {
    const int mat = i / (2 * 16 * 8), rem = i % (2 * 16 * 8);
    const int half = rem / (16 * 8), rr = rem % (16 * 8);
    const int n = 128 + rr / 8, c = rr % 8;
    *reinterpret_cast<uint4*>(bmat + mat * kBBytes + half * kBHalf + (n >> 3) * 1024 + (n & 7) * 128 + (c << 4)) =
        make_uint4(0, 0, 0, 0);
  }
  if (warp == 1) tc::tmem_alloc(&s_tmem, kTmemCols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = s_tmem;

  if (warp == 0) {
    // ================= TMA producer =================
    // The whole warp issues: lane c loads chunk c's block id and launches its
    // two TMA boxes, so a 32-KB tile costs one round of issue instead of 16
    // sequential TMA instructions from one lane.
    {
      const int chunks = kTileM / g.bs;
      int pos = 0;
      auto acquire = [&](int p) -> unsigned char* {
        const int st = p % kStages;
        if (lane == 0) tc::mbar_wait(&st_empty[st], ((p / kStages) & 1) ^ 1);
        __syncwarp();
        return ring + st * kStageBytes;
      };
      auto load_sigma = [&](int item, int u) {
        const PressReq q = b.req[item / LH];
        const int lh = item % LH, l = lh / g.H, h = lh % g.H;
        const int row = (int)((((int64_t)q.q_idx * g.L + l) * pp.num_q_heads + h * gq + u) * kD);
        for (int part = 0; part < 2; ++part, ++pos) {
          unsigned char* dst = acquire(pos);
          uint64_t* bar = &st_full[pos % kStages];
          if (lane == 0) {
            tc::mbar_expect_tx(bar, 64 * kD * 4);
            tc::tma_load_2d(dst, &cmap, bar, 0, row + part * 64);
          }
        }
      };
      auto load_tiles = [&](const PressReq& q, int l, int h, int kv) {
        const int nb = (q.T + g.bs - 1) / g.bs, ntiles = (q.T + kTileM - 1) / kTileM;
        const int64_t row_l = ((int64_t)l * g.num_blocks * 2 + kv) * g.H * g.bs + (int64_t)h * g.bs;
        for (int k = 0; k < ntiles; ++k, ++pos) {
          const int n_chunks = min(chunks, nb - k * chunks);
          // block id loaded before the stage wait so its latency hides behind it
          const int blk = lane < n_chunks ? __ldg(table + (int64_t)q.slot * g.max_bpr + k * chunks + lane) : 0;
          unsigned char* dst = acquire(pos);
          uint64_t* bar = &st_full[pos % kStages];
          if (lane == 0) tc::mbar_expect_tx(bar, (uint32_t)(n_chunks * g.bs * kD * 2));
          __syncwarp();
          if (lane < n_chunks) {
            const int64_t row0 = row_l + (int64_t)blk * 2 * g.H * g.bs;
            tc::tma_load_2d(dst + lane * g.bs * 128, &kmap, bar, 0, (int)row0);
            tc::tma_load_2d(dst + kTileM * 128 + lane * g.bs * 128, &kmap, bar, 64, (int)row0);
          }
        }
      };
      if ((int)blockIdx.x < n_items) load_sigma(blockIdx.x, 0);
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int lh = item % LH, l = lh / g.H, h = lh % g.H;
        const PressReq q = b.req[item / LH];
        for (int u = 0; u < gq; ++u) {
          load_tiles(q, l, h, 0);                      // K tiles of unit u
          if (u + 1 < gq) load_sigma(item, u + 1);
        }
        load_tiles(q, l, h, 1);
        if (item + (int)gridDim.x < n_items) load_sigma(item + gridDim.x, 0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_f16(Elem<T>::kDtype == FC_BF16 ? 1 : 0, kTileM, kBRows);
      const uint32_t bh = tc::smem_u32(bmat), bl = bh + kBBytes;
      int pos = 2, gt = 0, un = 0;
      for (int it = 0, item = blockIdx.x; item < n_items; ++it, item += gridDim.x) {
        const PressReq q = b.req[item / LH];
        const int ntiles = (q.T + kTileM - 1) / kTileM;
        const SegPos sp = seg_pos(pos, ntiles, item + (int)gridDim.x < n_items, gq);
        for (int u = 0; u < gq; ++u, ++un) {
        tc::mbar_wait(b_full, un & 1);
        tc::fence_after_sync();
        for (int k = 0; k < ntiles; ++k, ++gt) {
          const int p = sp.k_unit(u) + k, st = p % kStages, sl = gt % kSlots;
          tc::mbar_wait(&sl_empty[sl], ((gt / kSlots) & 1) ^ 1);
          tc::mbar_wait(&st_full[st], (p / kStages) & 1);
          tc::fence_after_sync();
          const uint32_t a = tc::smem_u32(ring + st * kStageBytes);
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            const uint32_t bb = part ? bl : bh;
#pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk) {
              const uint32_t koff = (uint32_t)((kk & 3) * 32);
              tc::mma_f16(tmem + (uint32_t)(sl * kSlotCols),
                          tc::desc_k_sw128(a + (kk >> 2) * kTileM * 128 + koff),
                          tc::desc_k_sw128(bb + (kk >> 2) * kBHalf + koff), idesc,
                          (part | kk) ? 1u : 0u);
            }
          }
          tc::mma_commit(&sl_full[sl]);
        }
        tc::mma_commit(b_empty);
        }
        pos = sp.next;
      }
    }
    __syncwarp();
  } else if (warp >= kCompactorFirst / 32) {
    using Compactors = NamedGroup<kCompactorFirst, 2, ea_comp_threads(kGqa)>;
    // ================= compactors =================
    for (int it = 0, item = blockIdx.x; item < n_items; ++it, item += gridDim.x) {
      const int jb = it & 1;
      tc::mbar_wait(&job_full[jb], (it >> 1) & 1);
      if (Compactors::tid() == 0) EA_STAMP(it, 6);
      const Job job = s_job[jb];
      char* seg = arena + g.seg_base(job.l, 0, job.h);
      const int32_t* tab = kSpill ? table + (int64_t)job.slot * g.max_bpr : ctab + jb * nb_stride;
      compact_rows<kD * 2, Compactors, FC_EA_CITEMS, FC_EA_CPF>(seg, g, tab, tab,
                                          idxbuf + jb * k_stride, job.K, job.first_moved);
      Compactors::sync();
      if (Compactors::tid() == 0) {
        EA_STAMP(it, 7);
        tc::mbar_arrive(&job_empty[jb]);
      }
    }
  } else {
    // ================= consumers =================
    const int ct = Consumers::tid();
    const int cw = warp - kConsumerFirst / 32;
    const int grp = cw >> 2;                    // Y / K columns [64*grp, 64*grp + 64)
    const int quarter = warp & 3;
    const int trow = quarter * 32 + lane;       // TMEM lane = token row in tile
    const float inv_sqrt_d = 1.0f / sqrtf((float)kD);
    const float inv_2d = 1.0f / (2.0f * (float)kD);

    // The consumers read ring stages with generic-proxy loads and the producer
    // refills them with TMA (async proxy): order the reads before the refill
    // with a proxy fence ahead of the release (without it a fast producer's TMA
    // overwrote K/Sigma/V rows still being read -- wrong z_t, or a hang).
    auto release_stage = [&](int p) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&st_empty[p % kStages]);
    };
    // Sigma (fp32, two ring stages) -> B hi/lo (fp16, transposed, swizzled) + mu row
    auto convert_sigma = [&](int p0, int item, int u) {
      const PressReq q = b.req[item / LH];
      const int lh = item % LH, l = lh / g.H, h = lh % g.H;
      const float* mu = mean_q + ((((int64_t)q.q_idx * g.L + l) * pp.num_q_heads + h * gq + u) * kD);
      for (int part = 0; part < 2; ++part) {
        const int p = p0 + part;
        tc::mbar_wait(&st_full[p % kStages], (p / kStages) & 1);
        const float* sig = reinterpret_cast<const float*>(ring + (p % kStages) * kStageBytes);
        // this stage holds Sigma rows k in [64*part, 64*part + 64): B[n][k] = Sigma[k][n]
        for (int i = ct; i < 128 * 8; i += kThreads) {
          const int n = i & 127, c8 = i >> 7;           // 8 chunks of 8 k's
          const int k0 = part * 64 + c8 * 8;
          T hi[8], lo[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float x = sig[(c8 * 8 + e) * kD + n];
            hi[e] = Elem<T>::from_f(x);
            lo[e] = Elem<T>::from_f(x - Elem<T>::to_f(hi[e]));
          }
          *reinterpret_cast<uint4*>(bmat + b_off(n, k0)) = *reinterpret_cast<uint4*>(hi);
          *reinterpret_cast<uint4*>(bmat + kBBytes + b_off(n, k0)) = *reinterpret_cast<uint4*>(lo);
        }
        release_stage(p);
      }
      for (int k = ct; k < kD; k += kThreads) {
        const float x = mu[k];
        const T hi = Elem<T>::from_f(x);
        *reinterpret_cast<T*>(bmat + b_off(128, k)) = hi;
        *reinterpret_cast<T*>(bmat + kBBytes + b_off(128, k)) = Elem<T>::from_f(x - Elem<T>::to_f(hi));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      Consumers::sync();
      if (ct == 0) tc::mbar_arrive(b_full);
    };

    int pos = 2, gt = 0, un = 0;
    if ((int)blockIdx.x < n_items) convert_sigma(0, blockIdx.x, 0);
    for (int it = 0, item = blockIdx.x; item < n_items; ++it, item += gridDim.x) {
      const int r = item / LH, lh = item % LH, l = lh / g.H, h = lh % g.H;
      const PressReq q = b.req[r];
      const int T_len = q.T, K = q.K, ns = pp.n_sink;
      const int nb = (T_len + g.bs - 1) / g.bs, ntiles = (T_len + kTileM - 1) / kTileM;
      const bool has_next = item + (int)gridDim.x < n_items;
      const SegPos sp = seg_pos(pos, ntiles, has_next, gq);
      const int jb = it & 1;
      if (ct == 0) {
        ss.first_drop = INT_MAX;
        EA_STAMP(it, 0);
      }
      if (kGqa)
        for (int t = ct; t < T_len; t += kThreads) pacc[t] = 0.f;
      float m = -INFINITY, inv_z = 0.f;
      for (int u = 0; u < gq; ++u, ++un) {
      for (int t = ct; t < T_len; t += kThreads) zt[t] = 0.f;
      Consumers::sync();
      // ---- z_t from TMEM (Y = K.B^T) and the K rows still in SMEM ----
      for (int k = 0; k < ntiles; ++k, ++gt) {
        const int p = sp.k_unit(u) + k, sl = gt % kSlots;
        tc::mbar_wait(&sl_full[sl], (gt / kSlots) & 1);
        tc::fence_after_sync();
        float y[32];
        float acc = 0.f;
        const int t = k * kTileM + trow;
        const unsigned char* krow = ring + (p % kStages) * kStageBytes + grp * (kTileM * 128) +
                                    (trow >> 3) * 1024 + (trow & 7) * 128;
        const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(sl * kSlotCols + grp * 64);
        // K . mu (column 128) rides along with the first Y load: one wait for both
        uint32_t lin_r = 0;
        if (grp == 0)
          tc::tmem_ld_x1_async(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(sl * kSlotCols + 128), lin_r);
#pragma unroll
        for (int hcol = 0; hcol < 2; ++hcol) {
          tc::tmem_ld_32x32b_x32(taddr + (uint32_t)(hcol * 32), y);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int chunk = hcol * 4 + c;
            const uint4 raw = *reinterpret_cast<const uint4*>(krow + ((chunk ^ (trow & 7)) << 4));
            float kx[8];
            unpack16<T>(raw, kx);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = fmaf(y[c * 8 + e], kx[e], acc);
          }
        }
        tc::reg_after_wait(lin_r);
        const float lin = __uint_as_float(lin_r);
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&sl_empty[sl]);
        release_stage(p);
        if (t < T_len) atomicAdd(&zt[t], grp == 0 ? fmaf(lin, inv_sqrt_d, acc * inv_2d) : acc * inv_2d);
      }
      Consumers::sync();
      if (ct == 0) EA_STAMP(it, 1);
      // ---- softmax over t >= n_sink ----
      m = -INFINITY;
      for (int t = ns + ct; t < T_len; t += kThreads) m = fmaxf(m, zt[t]);
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
      if (lane == 0) ss.red[cw] = m;
      Consumers::sync();
      m = ss.red[0];
      for (int w = 1; w < kWarps; ++w) m = fmaxf(m, ss.red[w]);
      float z = 0.f;
      for (int t = ns + ct; t < T_len; t += kThreads) z += expf(zt[t] - m);
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) z += __shfl_xor_sync(0xffffffffu, z, off);
      Consumers::sync();
      if (lane == 0) ss.red[cw] = z;
      Consumers::sync();
      z = 0.f;
      for (int w = 0; w < kWarps; ++w) z += ss.red[w];
      inv_z = 1.0f / z;
      if (kGqa) {
        // this head's probabilities join the running sum (heads in order: deterministic)
        for (int t = ns + ct; t < T_len; t += kThreads) pacc[t] += expf(zt[t] - m) * inv_z;
        if (u + 1 < gq) {                 // the next head's Sigma while the MMA idles
          tc::mbar_wait(b_empty, un & 1);
          convert_sigma(sp.sig_unit(u + 1), item, u + 1);
        }
      }
      }
      if (ct == 0) EA_STAMP(it, 2);
      if (kGqa) Consumers::sync();
      const float inv_g = 1.0f / (float)gq;
      // ---- V tiles: s_t = p_t * ||V_t|| (two lanes per row) ----
      for (int k = 0; k < ntiles; ++k) {
        const int p = sp.v0 + k;
        tc::mbar_wait(&st_full[p % kStages], (p / kStages) & 1);
        const int row = ct >> 1, half = ct & 1;
        const unsigned char* vrow = ring + (p % kStages) * kStageBytes + half * (kTileM * 128) +
                                    (row >> 3) * 1024 + (row & 7) * 128;
        float sq = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float vx[8];
          // physical chunk c ^ (row & 7): the 128-B swizzle spreads the 16 rows of a warp
          // over all 32 banks (unswizzled offsets put every lane on the same 4 banks)
          unpack16<T>(*reinterpret_cast<const uint4*>(vrow + ((c ^ (row & 7)) << 4)), vx);
#pragma unroll
          for (int e = 0; e < 8; ++e) sq = fmaf(vx[e], vx[e], sq);
        }
        sq += __shfl_xor_sync(0xffffffffu, sq, 1);
        release_stage(p);
        const int t = k * kTileM + row;
        if (half == 0 && t < T_len && t >= ns)
          zt[t] = (kGqa ? pacc[t] * inv_g : expf(zt[t] - m) * inv_z) * sqrtf(sq);
      }
      if (ct == 0) EA_STAMP(it, 3);
      // ---- the next segment's Sigma (last in the ring order, see SegPos) ----
      if (has_next) {
        tc::mbar_wait(b_empty, (un - 1) & 1);   // the MMAs of this segment's last head
        convert_sigma(sp.sig_next, item + gridDim.x, 0);
      }
      Consumers::sync();
      if (ct == 0) EA_STAMP(it, 4);
      for (int t = ct; t < ns && t < T_len; t += kThreads) zt[t] = INFINITY;
      Consumers::sync();
      if (out.scores) {
        float* so = out.scores + q.score_off + (int64_t)lh * T_len;
        for (int t = ct; t < T_len; t += kThreads) so[t] = zt[t];
      }
      uint32_t* keys = reinterpret_cast<uint32_t*>(zt);
      for (int t = ct; t < T_len; t += kThreads) keys[t] = float_key(zt[t]);
      // ---- select into the hand-off buffer ----
      tc::mbar_wait(&job_empty[jb], ((it >> 1) & 1) ^ 1);
      int32_t* idx = idxbuf + jb * k_stride;
      if (!kSpill)
        for (int i = ct; i < nb; i += kThreads) ctab[jb * nb_stride + i] = table[(int64_t)q.slot * g.max_bpr + i];
      Consumers::sync();
      select_request<Consumers>(keys, T_len, K, q.seg0, q.K0, b.per_segment, idx, ss);
      if (out.kept_idx) {
        int32_t* ko = out.kept_idx + q.kept_off + (int64_t)lh * K;
        for (int j = ct; j < K; j += kThreads) ko[j] = idx[j];
      }
      if (ct == 0) s_job[jb] = Job{l, h, K, min(ss.first_drop, K), q.slot};
      Consumers::sync();
      if (ct == 0) {
        EA_STAMP(it, 5);
        tc::mbar_arrive(&job_full[jb]);
      }
      pos = sp.next;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, kTmemCols);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
bool ea_tc_supported(const Geom& g, int dtype, const PressParams& pp, int max_T, int max_K) {
  static const bool forced_simt = [] {
    const char* e = getenv("FASTCACHE_EA_SIMT");
    return e && e[0] == '1';
  }();
  if (forced_simt) return false;
  if ((dtype != FC_F16 && dtype != FC_BF16) || g.D != kD) return false;
  if (pp.num_q_heads % g.H != 0 || pp.num_q_heads / g.H > 8) return false;   // GQA: gq <= 8
  if (g.bs < 8 || g.bs > 128) return false;
  (void)max_T;
  (void)max_K;
  return true;   // any T: segments beyond the SMEM plan take the spill variant
}

static bool ea_needs_spill(const Geom& g, int max_T, int max_K, bool gqa) {
  return plan(g.bs, max_T, max_K, gqa).total > kDynSmemBudget;
}

int64_t ea_tc_workspace_floats(const Geom& g, int num_q_heads, int max_T, int max_K) {
  const bool gqa = num_q_heads != g.H;
  if (!ea_needs_spill(g, max_T, max_K, gqa)) return 0;
  return (int64_t)sm_count() * spill_row_floats(max_T, max_K, gqa);
}

fc_status encode_rows(CUtensorMap* map, const void* base, int dtype, int D, uint64_t rows, int box_rows);

fc_status launch_ea_tc(const Geom& g, int dtype, char* arena, const int32_t* table,
                       const PressBatch& b, const PressParams& pp, const fc_press_inputs& in,
                       const fc_press_outputs& out, int max_K, float* ws, int64_t ws_floats,
                       cudaStream_t stream, bool dry_run) {
  CUtensorMap kmap, cmap;
  const uint64_t rows = (uint64_t)g.L * g.num_blocks * 2 * g.H * g.bs;
  fc_status st = encode_rows(&kmap, arena, dtype, g.D, rows, g.bs);
  if (st != FC_OK) return st;
  st = encode_rows(&cmap, in.cov_q, FC_F32, g.D, (uint64_t)b.n_total * g.L * pp.num_q_heads * g.D, 64);
  if (st != FC_OK) return st;
  const bool gqa = pp.num_q_heads != g.H;
  const bool spill = ea_needs_spill(g, b.max_T, max_K, gqa);
  const Smem P = plan(g.bs, b.max_T, max_K, gqa, spill);
  if (P.total > kDynSmemBudget)
    return set_error(FC_ERR_UNSUPPORTED, "ExpectedAttention tensor-core plan exceeds the SMEM budget");
  if (dry_run) return FC_OK;   // the pool sizes the spill workspace next
  const int n_items = b.n * g.L * g.H;
  const int sms = sm_count();
  int grid = n_items < sms ? n_items : sms;
  if (spill) {
    const int64_t row = spill_row_floats(b.max_T, max_K, gqa);
    if (ws_floats < row) return set_error(FC_ERR_INVALID_STATE, "EA spill workspace too small");
    grid = (int)std::min<int64_t>(grid, ws_floats / row);
  }
  auto launch = [&](auto kern) -> fc_status {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P.total);
    if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute(ea_tc)");
    kern<<<grid, ea_threads(gqa), P.total, stream>>>(arena, table, g, b, pp, kmap, cmap, in.mean_q, out,
                                                n_items, max_K, ws);
    note_launch();
    note_path(kPathTc);
    return cuda_check(cudaGetLastError(), "ea_tc_kernel");
  };
  if (dtype == FC_BF16) {
    if (spill)
      return gqa ? launch(ea_tc_kernel<__nv_bfloat16, true, true>) : launch(ea_tc_kernel<__nv_bfloat16, false, true>);
    return gqa ? launch(ea_tc_kernel<__nv_bfloat16, true, false>) : launch(ea_tc_kernel<__nv_bfloat16, false, false>);
  }
  if (spill) return gqa ? launch(ea_tc_kernel<__half, true, true>) : launch(ea_tc_kernel<__half, false, true>);
  return gqa ? launch(ea_tc_kernel<__half, true, false>) : launch(ea_tc_kernel<__half, false, false>);
}

}  // namespace fc

#ifdef FC_TRACE
extern "C" FC_API fc_status fc_debug_trace_read_ea(void* host, uint64_t bytes) {
  return fc::cuda_check(cudaMemcpyFromSymbol(host, fc::g_fc_trace_ea, bytes), "trace read");
}
#endif
