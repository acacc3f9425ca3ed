// fc_snapkv_tc.cu -- SnapKV scoring on the 5th-gen tensor cores (sm_100a).
//
// Persistent, warp-specialised: one CTA per SM walks a strided list of
// (request, layer, kv-head) segments (longest requests first).
//
//   warp 0      TMA producer: loads the window queries (double-buffered) and
//               streams every K tile (128 tokens x D, fp16/bf16) of every
//               segment from its paged blocks into a 4-stage SMEM ring with
//               cp.async.bulk.tensor (128-byte swizzle).
//   warp 1      MMA issuer: tcgen05.mma  S[tile] = K_tile . Q_win^T
//               (M = 128 tokens, N = 32 queries, K = D, fp32 accumulate) into
//               a 16-slot TMEM ring (16 x 32 columns = all 512 columns). A
//               segment's whole logit matrix stays resident (T <= 2048).
//   warps 2-9   consumers (named barrier 1): per-query max, sum of exp and
//               s'_t = mean_j softmax_j(t) straight from TMEM (tcgen05.ld,
//               each warp group owns 16 of the 32 queries), freeing TMEM slots
//               as they go; then avg-pool, forced window, segmented radix
//               top-k and in-place compaction of K and V (fc_select.cuh).
//
// While the consumers finish segment s, the producer and MMA warps already
// stream and multiply segment s+1 into the freed slots, so HBM stays busy.
// K is read from HBM exactly once; scores never leave the SM. Precision:
// fp16/bf16 products are exact in fp32, only the fp32 accumulation order
// differs from the oracle (scores within 1e-5 relative, tests/test_gpu_press.py).
// Reference anchors: SURVEY.md Appendix A (kvpress SnapKV restated), K_r from
// the reference ceil rule (kv.py:169-194).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <cstring>
#include <mutex>

#include "fc_select.cuh"
#include "fc_tc.cuh"

namespace fc {

#ifdef FC_TRACE
// Debug build only (make trace): per-CTA, per-segment %globaltimer stamps.
__device__ unsigned long long g_fc_trace[148 * 64 * 16];
__device__ __forceinline__ void trace_stamp(int it, int slot) {
  if (it < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_fc_trace[(blockIdx.x * 64 + it) * 16 + slot] = t;
  }
}
#define FC_STAMP(it, slot) trace_stamp(it, slot)
#else
#define FC_STAMP(it, slot) ((void)0)
#endif

#ifndef FC_SNAP_STAGES
#define FC_SNAP_STAGES 3
#endif
constexpr int kTcStages = FC_SNAP_STAGES;
constexpr int kTileM = 128;
constexpr int kSlots = 16;                      // TMEM ring: 16 x 32 fp32 columns
#ifndef FC_SNAP_RESIDENT
#define FC_SNAP_RESIDENT (kSlots - 2)
#endif
// A segment longer than the ring (ntiles > kSlots) is streamed in two passes; the
// last kResident tiles of pass A stay in TMEM for pass B, which re-streams only the
// first ntiles - kResident (two slots stay free so the re-stream starts at once).
constexpr int kResident = FC_SNAP_RESIDENT;
__host__ __device__ __forceinline__ int snap_loads(int ntiles) {
  return ntiles > kSlots ? 2 * ntiles - kResident : ntiles;
}
constexpr int kWin = 32;                        // window queries (UMMA N)
constexpr int kConsumerFirst = 64;              // warps 0,1 = producer, MMA
constexpr int kCompactorFirst = kConsumerFirst + kThreads;
#ifndef FC_SNAP_GQA_COMP_WARPS   // compactor warps of the GQA instantiation (8 = as g = 1)
#define FC_SNAP_GQA_COMP_WARPS 4
#endif
// GQA segments are consumer-bound (g softmax units per segment) with the compactors
// mostly idle: 4 compactor warps make the CTA 14 warps, at most 4 per SM sub-partition,
// so every warp may hold 128 registers (18 warps cap it at 96): c3g 4.09 -> 3.94 ms.
// (Two tiles' TMEM loads per wait on top of that measured 4.03 ms.)
__host__ __device__ constexpr int snap_comp_threads(bool gqa) { return gqa ? 32 * FC_SNAP_GQA_COMP_WARPS : kThreads; }
__host__ __device__ constexpr int snap_threads(bool gqa) { return kCompactorFirst + snap_comp_threads(gqa); }
constexpr int kTcThreads = snap_threads(false);
using Consumers = NamedGroup<kConsumerFirst, 1>;

struct CompactJob {  // consumer -> compactor hand-off of one segment
  int32_t l, h, K, first_moved, slot;
};

#ifndef FC_SNAP_ASYNC_COMPACT
#define FC_SNAP_ASYNC_COMPACT 1
#endif
#ifndef FC_SNAP_L2HINT  // L2 eviction hints on the K tiles (evict-last for a long segment's pass A)
#define FC_SNAP_L2HINT 1
#endif
#ifndef FC_SNAP_CRANKS
#define FC_SNAP_CRANKS 16   // measured at c3: 16 x 6 buffers 5.87 ms, 32 x 4 5.97, 16 x 8 5.95, 16 x 4 6.02, 32 x 3 6.00
#endif
#ifndef FC_SNAP_CBUFS
#define FC_SNAP_CBUFS 6
#endif

struct TcSmem {
  int tile_bytes, q_bytes, max_nb;
  int off_stage, off_q, off_ptab, off_ctab, off_idx, off_sc, off_s1, off_bar, off_cbuf, total;
  bool async_compact;
};

__host__ __device__ inline int snap_k_stride(int max_K) { return ((max_K * 4 + 15) & ~15) / 4; }

// spill: segments too long for the SMEM arrays keep the block tables in global memory
// (read in place) and the T-sized arrays (scores / keys, window means, the kept-index
// hand-off) in a per-CTA global row of snap_spill_floats(); SMEM then holds only the
// TMA ring, the window queries, the barriers and the compaction ring.
__host__ __device__ inline int64_t snap_spill_floats(int max_T, int max_K) {
  const int64_t tp = (max_T + 3) & ~3;
  return tp + (8 + tp) + 2 * snap_k_stride(max_K);
}

__host__ __device__ inline TcSmem tc_smem_plan(int D, int bs, int max_T, int max_K,
                                               bool spill = false) {
  TcSmem p;
  p.tile_bytes = kTileM * D * 2;
  p.q_bytes = (kWin * D * 2 + 1023) & ~1023;
  p.max_nb = (max_T + bs - 1) / bs;
  p.off_stage = 0;  // 1024-aligned base
  p.off_q = p.off_stage + kTcStages * p.tile_bytes;
  p.off_ptab = p.off_q + 2 * p.q_bytes;
  if (spill) {
    p.off_ctab = p.off_idx = p.off_sc = p.off_s1 = p.off_bar = p.off_ptab;
  } else {
    p.off_ctab = p.off_ptab + ((p.max_nb * 4 + 15) & ~15);          // [2][max_nb]
    p.off_idx = p.off_ctab + 2 * ((p.max_nb * 4 + 15) & ~15);        // [2][max_K] kept positions
    p.off_sc = p.off_idx + 2 * snap_k_stride(max_K) * 4;
    p.off_s1 = p.off_sc + ((max_T * 4 + 15) & ~15);                   // [8 zeros][max_T]
    p.off_bar = p.off_s1 + (((max_T + 8) * 4 + 15) & ~15);
  }
  p.off_cbuf = p.off_bar + (((2 * kTcStages + 8 + 2 * kSlots) * 8 + 127) & ~127);
  p.total = p.off_bar + (2 * kTcStages + 8 + 2 * kSlots) * 8 + 1024;
  // the compactors' cp.async ring (D * 2-byte rows, 4 x 32-rank chunks) when it fits
  const int cbuf = FC_SNAP_CBUFS * FC_SNAP_CRANKS * 2 * D * 2;
  p.async_compact = FC_SNAP_ASYNC_COMPACT && p.off_cbuf + cbuf + 1024 <= kDynSmemBudget;
  if (p.async_compact) p.total = p.off_cbuf + cbuf + 1024;
  return p;
}

template <typename T, int D, bool kGqa, bool kSpill>
__global__ void __launch_bounds__(snap_threads(kGqa), 1)
    snapkv_tc_kernel(char* __restrict__ arena, const int32_t* __restrict__ table, const Geom g,
                     const __grid_constant__ PressBatch b, const PressParams pp,
                     const __grid_constant__ CUtensorMap kmap,
                     const __grid_constant__ CUtensorMap qmap, const fc_press_outputs out,
                     int n_items, int max_K, float* __restrict__ spill) {
  constexpr int kHalves = D / 64;  // 128-byte K-dim slabs
  constexpr int kKSteps = D / 16;  // UMMA_K = 16 for 16-bit inputs
  constexpr int kFmt = Elem<T>::kDtype == FC_BF16 ? 1 : 0;
  extern __shared__ unsigned char smem_raw[];
  __shared__ SelectScratch ss;
  __shared__ uint32_t s_tmem;
  __shared__ float s_red[kWarps][16];
  __shared__ float s_m[kWin], s_zinv[kWin];
  __shared__ float s_zpart[kWarps][16];

  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const TcSmem plan = tc_smem_plan(D, g.bs, b.max_T, max_K, kSpill);
  unsigned char* stages = smem + plan.off_stage;
  unsigned char* qbuf = smem + plan.off_q;
  int32_t* ptab = reinterpret_cast<int32_t*>(smem + plan.off_ptab);   // unused when kSpill
  const int nb_stride = ((plan.max_nb * 4 + 15) & ~15) / 4;
  const int k_stride = snap_k_stride(max_K);
  int32_t* ctab = reinterpret_cast<int32_t*>(smem + plan.off_ctab);   // [2][nb_stride]
  __shared__ CompactJob s_job[2];
  float* const row = kSpill ? spill + (int64_t)blockIdx.x * snap_spill_floats(b.max_T, max_K)
                            : nullptr;
  const int64_t t_pad = (b.max_T + 3) & ~3;
  float* sc = kSpill ? row : reinterpret_cast<float*>(smem + plan.off_sc);
  // window means, front-padded with 8 zeros so the pooling window needs no bounds
  float* s1 = (kSpill ? row + t_pad : reinterpret_cast<float*>(smem + plan.off_s1)) + 8;
  int32_t* idxbuf = kSpill ? reinterpret_cast<int32_t*>(row + t_pad + 8 + t_pad)
                           : reinterpret_cast<int32_t*>(smem + plan.off_idx);  // [2][k_stride]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + plan.off_bar);
  uint64_t* st_full = bars;
  uint64_t* st_empty = bars + kTcStages;
  uint64_t* q_full = bars + 2 * kTcStages;
  uint64_t* q_empty = q_full + 2;
  uint64_t* job_full = q_empty + 2;
  uint64_t* job_empty = job_full + 2;
  uint64_t* sl_full = job_empty + 2;
  uint64_t* sl_empty = sl_full + kSlots;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int LH = g.L * g.H;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * kTcStages + 8 + kSlots; ++i) tc::mbar_init(&bars[i], 1);
    for (int i = 0; i < kSlots; ++i) tc::mbar_init(&sl_empty[i], kWarps);  // one arrive per consumer warp
    tc::fence_barrier_init();
    tc::tma_prefetch_desc(&kmap);
    tc::tma_prefetch_desc(&qmap);
  }
  if (warp == 1) tc::tmem_alloc(&s_tmem, kSlots * kWin);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = s_tmem;

  if (warp == 0) {
    // ================= TMA producer =================
    const int chunks = kTileM / g.bs;
    const uint64_t pol_last = tc::l2_policy_evict_last(), pol_first = tc::l2_policy_evict_first();
    int gtile = 0, unit = 0;
    for (int it = 0, item = blockIdx.x; item < n_items; ++it, item += gridDim.x) {
      const int r = item / LH, lh = item % LH, l = lh / g.H, h = lh % g.H;
      const PressReq q = b.req[r];
      const int nb = (q.T + g.bs - 1) / g.bs, ntiles = (q.T + kTileM - 1) / kTileM;
      const int32_t* btab = kSpill ? table + (int64_t)q.slot * g.max_bpr : ptab;
      __syncwarp();
      if (!kSpill)
        for (int i = lane; i < nb; i += 32) ptab[i] = table[(int64_t)q.slot * g.max_bpr + i];
      __syncwarp();
      // GQA: the gq query heads sharing this kv head are scored one after the
      // other ("units"); the first gq - 1 passes over K ask L2 to keep the tiles
      // so the repeats come from L2, not HBM.
      const int gq = kGqa ? pp.num_q_heads / g.H : 1;
      const int64_t row_l = (int64_t)l * g.num_blocks * 2 * g.H * g.bs + (int64_t)h * g.bs;
      // a segment longer than the TMEM ring (T > kSlots * 128) is streamed in two
      // passes: pass A (softmax statistics) over every tile, pass B (normalised
      // window mean) re-streams tiles [0, ntiles - kResident) only
      const int nload = snap_loads(ntiles);
      for (int gi = 0; gi < gq; ++gi, ++unit) {
        if (lane == 0) {
          const int qb = unit & 1;
          tc::mbar_wait(&q_empty[qb], ((unit >> 1) & 1) ^ 1);
          const int qrow = (int)((((int64_t)q.q_idx * g.L + l) * pp.num_q_heads + h * gq + gi) * kWin);
          tc::mbar_expect_tx(&q_full[qb], (uint32_t)(kWin * D * 2));
#pragma unroll
          for (int hf = 0; hf < kHalves; ++hf)
            tc::tma_load_2d(qbuf + qb * plan.q_bytes + hf * kWin * 128, &qmap, &q_full[qb], hf * 64, qrow);
        }
        // K tiles: lane c issues chunk c's boxes (one round of issue per tile)
        for (int kl = 0; kl < nload; ++kl, ++gtile) {
          const int k = kl < ntiles ? kl : kl - ntiles;
          const int st = gtile % kTcStages;
          const int n_chunks = min(chunks, nb - k * chunks);
          if (lane == 0) {
            tc::mbar_wait(&st_empty[st], ((gtile / kTcStages) & 1) ^ 1);
#ifdef FC_TRACE_GQA   // GQA diagnosis (scripts/trace_press.py gqa): unit 1's first / last K tile issue
            if (gi == 1 && kl == 0) FC_STAMP(it, 0);
            if (gi == 1 && kl == ntiles - 1) FC_STAMP(it, 1);
#else
            if (gi == 0 && kl == 0) FC_STAMP(it, 0);
            if (gi == 0 && kl == ntiles - 1) FC_STAMP(it, 1);
#endif
            tc::mbar_expect_tx(&st_full[st], (uint32_t)(n_chunks * g.bs * D * 2));
          }
          __syncwarp();
          unsigned char* dst = stages + st * plan.tile_bytes;
          // evict-last while a later pass (pass B, or the next query head) re-reads
          // the tile; evict-first on its last read
          const bool reread = gi + 1 < gq || (nload > ntiles && kl < ntiles - kResident);
          const uint64_t pol = (FC_SNAP_L2HINT && reread) ? pol_last : pol_first;
          for (int c = lane; c < n_chunks; c += 32) {
            const int64_t row0 = row_l + (int64_t)btab[k * chunks + c] * 2 * g.H * g.bs;
#pragma unroll
            for (int hf = 0; hf < kHalves; ++hf) {
              if (FC_SNAP_L2HINT)
                tc::tma_load_2d_hint(dst + hf * kTileM * 128 + c * g.bs * 128, &kmap, &st_full[st],
                                     hf * 64, (int)row0, pol);
              else
                tc::tma_load_2d(dst + hf * kTileM * 128 + c * g.bs * 128, &kmap, &st_full[st],
                                hf * 64, (int)row0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_f16(kFmt, kTileM, kWin);
      int gtile = 0, unit = 0;
      const int gq = kGqa ? pp.num_q_heads / g.H : 1;
      for (int it = 0, item = blockIdx.x; item < n_items; ++it, item += gridDim.x) {
        const PressReq q = b.req[item / LH];
        const int ntiles = (q.T + kTileM - 1) / kTileM;
        for (int gi = 0; gi < gq; ++gi, ++unit) {
        const int qb = unit & 1;
        tc::mbar_wait(&q_full[qb], (unit >> 1) & 1);
        const uint32_t q_base = tc::smem_u32(qbuf + qb * plan.q_bytes);
        const int nload = snap_loads(ntiles);
        for (int k = 0; k < nload; ++k, ++gtile) {
          const int st = gtile % kTcStages, sl = gtile % kSlots;
          tc::mbar_wait(&sl_empty[sl], ((gtile / kSlots) & 1) ^ 1);
          tc::mbar_wait(&st_full[st], (gtile / kTcStages) & 1);
          tc::fence_after_sync();
          const uint32_t a_base = tc::smem_u32(stages + st * plan.tile_bytes);
#pragma unroll
          for (int kk = 0; kk < kKSteps; ++kk) {
            const uint32_t koff = (uint32_t)((kk & 3) * 32);
            const uint64_t ad = tc::desc_k_sw128(a_base + (kk >> 2) * kTileM * 128 + koff);
            const uint64_t bd = tc::desc_k_sw128(q_base + (kk >> 2) * kWin * 128 + koff);
            tc::mma_f16(tmem + (uint32_t)(sl * kWin), ad, bd, idesc, kk > 0 ? 1u : 0u);
          }
          tc::mma_commit(&st_empty[st]);
          tc::mma_commit(&sl_full[sl]);
#ifdef FC_TRACE_GQA
          if (gi == 1 && k == 0) FC_STAMP(it, 6);   // (the compactor's slots in this build)
          if (gi == 1 && k == nload - 1) FC_STAMP(it, 7);
#endif
        }
        tc::mma_commit(&q_empty[qb]);
        }
        FC_STAMP(it, 2);
      }
    }
    __syncwarp();
  } else if (warp >= kCompactorFirst / 32) {
    using Compactors = NamedGroup<kCompactorFirst, 2, snap_comp_threads(kGqa)>;
    // ================= compactors (8 warps, named barrier 2) =================
    for (int it = 0, item = blockIdx.x; item < n_items; ++it, item += gridDim.x) {
      const int jb = it & 1;
      tc::mbar_wait(&job_full[jb], (it >> 1) & 1);
#ifndef FC_TRACE_GQA
      if (Compactors::tid() == 0) FC_STAMP(it, 6);
#endif
      const CompactJob job = s_job[jb];
      char* seg = arena + g.seg_base(job.l, 0, job.h);
      const int32_t* tab = kSpill ? table + (int64_t)job.slot * g.max_bpr : ctab + jb * nb_stride;
#ifndef FC_NO_COMPACT
      if (plan.async_compact)
        compact_rows_async<D * (int)sizeof(T), Compactors, FC_SNAP_CRANKS, FC_SNAP_CBUFS>(
            seg, g, tab, tab, idxbuf + jb * k_stride, job.K, job.first_moved,
            smem + plan.off_cbuf);
      else
        compact_rows<D * (int)sizeof(T), Compactors, 8>(seg, g, tab, tab, idxbuf + jb * k_stride,
                                                     job.K, job.first_moved);
#endif
      Compactors::sync();
      if (Compactors::tid() == 0) {
#ifndef FC_TRACE_GQA
        FC_STAMP(it, 7);
#endif
        tc::mbar_arrive(&job_empty[jb]);
      }
    }
  } else {
    // ================= consumers (8 warps, named barrier 1) =================
    const int cw = warp - 2;                 // consumer warp 0..7
    const int grp = cw >> 2;                 // owns queries [16*grp, 16*grp + 16)
    const int quarter = warp & 3;            // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(grp * 16);
    // logits in the log2 domain: a_jt * log2(e) = acc * (log2(e) / sqrt(D))
    const float scale = 1.4426950408889634f / sqrtf((float)D);
    const int ct = Consumers::tid();
    int gtile = 0;
    for (int it = 0, item = blockIdx.x; item < n_items; ++it, item += gridDim.x) {
      const int r = item / LH, lh = item % LH, l = lh / g.H, h = lh % g.H;
      const PressReq q = b.req[r];
      const int T_len = q.T, K = q.K;
      const int nb = (T_len + g.bs - 1) / g.bs, ntiles = (T_len + kTileM - 1) / kTileM;
      const int n_keep = T_len - kWin;
      const int jb = it & 1;
      if (ct == 0) ss.first_drop = INT_MAX;

      float acc[16];
      // s1 = the window mean of both query groups (pass 3 adds into it)
      for (int t = ct - 8; t < T_len; t += kThreads) s1[t] = 0.f;
      // GQA: each head's two group addends meet on a zeroed scratch (sc, unused until
      // pooling) and are then added into s1 in head order -- deterministic
      float* const wacc = kGqa ? sc : s1;
      if (kGqa)
        for (int t = ct; t < T_len; t += kThreads) sc[t] = 0.f;
      // GQA: one unit per query head of the group; each adds its window mean
      // (weighted 1/(w * gq)) into s1, in head order
      const int gq = kGqa ? pp.num_q_heads / g.H : 1;
      const float inv_wg = 1.0f / (float)(kWin * gq);
      for (int gi = 0; gi < gq; ++gi) {
        if (ct == 0 && gi == 1) FC_STAMP(it, 11);
        if (ntiles <= kSlots) {
        // pass 1: per-query max over all tokens
  #pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = -INFINITY;
        auto max_tile = [&](int k, const float (&v)[16]) {
          const int t = k * kTileM + row;
          if (t <= T_len - kWin) {   // below the window: no causal mask
  #pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] = fmaxf(acc[j], v[j] * scale);
          } else {
  #pragma unroll
            for (int j = 0; j < 16; ++j)
              if (t < T_len && t <= T_len - kWin + grp * 16 + j) acc[j] = fmaxf(acc[j], v[j] * scale);
          }
        };
        for (int k = 0; k < ntiles; ++k) {
          const int sl = (gtile + k) % kSlots;
          tc::mbar_wait(&sl_full[sl], ((gtile + k) / kSlots) & 1);
          tc::fence_after_sync();
          float v[16];
          tc::tmem_ld_32x32b_x16(lane_addr + (uint32_t)(sl * kWin), v);
          max_tile(k, v);
        }
        if (ct == 0) FC_STAMP(it, 3);
        if (ct == 0 && gi == 1) FC_STAMP(it, 15);
        {
          const float r = tc::warp_reduce16(acc, lane, [](float a, float b) { return fmaxf(a, b); });
          if ((lane & 1) == 0) s_red[cw][lane >> 1] = r;
        }
        Consumers::sync();
        if (ct < kWin) {
          const int gg = ct >> 4, jj = ct & 15;
          float m = s_red[4 * gg][jj];
          for (int i = 1; i < 4; ++i) m = fmaxf(m, s_red[4 * gg + i][jj]);
          s_m[ct] = m;
        }
        Consumers::sync();
        float mj[16];
  #pragma unroll
        for (int j = 0; j < 16; ++j) mj[j] = s_m[grp * 16 + j];
        if (ct == 0) FC_STAMP(it, 8);
        // pass 2: per-query sum of exp
  #pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.f;
        auto exp_tile = [&](int k, float (&v)[16]) {
          const int t = k * kTileM + row;
          if (t <= T_len - kWin) {   // below the window: no causal mask
  #pragma unroll
            for (int j = 0; j < 16; ++j) {
              v[j] = tc::ex2(fmaf(v[j], scale, -mj[j]));
              acc[j] += v[j];
            }
          } else {
  #pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float e = (t < T_len && t <= T_len - kWin + grp * 16 + j) ? tc::ex2(fmaf(v[j], scale, -mj[j])) : 0.f;
              acc[j] += e;
              v[j] = e;
            }
          }
        };
        for (int k = 0; k < ntiles; ++k) {
          const int sl = (gtile + k) % kSlots;
          float v[16];
          tc::tmem_ld_32x32b_x16(lane_addr + (uint32_t)(sl * kWin), v);
          exp_tile(k, v);
          tc::tmem_st_32x32b_x16(lane_addr + (uint32_t)(sl * kWin), v);   // exps replace the logits
        }
        tc::tmem_store_wait();
        if (ct == 0) FC_STAMP(it, 9);
        {
          const float r = tc::warp_reduce16(acc, lane, [](float a, float b) { return a + b; });
          if ((lane & 1) == 0) s_red[cw][lane >> 1] = r;
        }
        Consumers::sync();
        if (ct < kWin) {
          const int gg = ct >> 4, jj = ct & 15;
          float z = 0.f;
          for (int i = 0; i < 4; ++i) z += s_red[4 * gg + i][jj];
          s_zinv[ct] = 1.0f / z;
        }
        Consumers::sync();
        float zj[16];
  #pragma unroll
        for (int j = 0; j < 16; ++j) zj[j] = s_zinv[grp * 16 + j];
        if (ct == 0) FC_STAMP(it, 10);
        // pass 3: window mean of the normalised probabilities; frees TMEM slots. The two
        // warp groups split the tiles (group g: k = g, g + 2, ...) and a thread sums all 32
        // queries of its row, so each token's mean is one plain store: shared-memory fp32
        // atomics are CAS loops on sm_100 (ATOMS.CAST.SPIN), with two warps contending.
        {
          float zall[kWin];
  #pragma unroll
          for (int j = 0; j < kWin; ++j) zall[j] = s_zinv[j];
          const uint32_t row_addr = tmem + ((uint32_t)(quarter * 32) << 16);
          for (int k = grp; k < ntiles; k += 2) {
            const int sl = (gtile + k) % kSlots;
            float v[16];
            float sum = 0.f;
  #pragma unroll
            for (int hq = 0; hq < 2; ++hq) {
              tc::tmem_ld_32x32b_x16(row_addr + (uint32_t)(sl * kWin + hq * 16), v);
  #pragma unroll
              for (int j = 0; j < 16; ++j) sum = fmaf(v[j], zall[hq * 16 + j], sum);   // masked entries are 0
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&sl_empty[sl], 2);   // stands for both groups' warps
            const int t = k * kTileM + row;
            if (t < n_keep) wacc[t] = sum * inv_wg;
          }
        }
        } else {
          // ---- long segment (T > kSlots * 128): two streamed passes ----
          // pass A: per-query running (reference max, sum of exp) as the tiles arrive,
          // each TMEM slot freed at once. Lazy rescaling: the reference moves only when
          // a logit exceeds it by more than 2^8, so the sum stays far from overflow.
          float mref[16], ssum[16];
  #pragma unroll
          for (int j = 0; j < 16; ++j) {
            mref[j] = -INFINITY;
            ssum[j] = 0.f;
          }
          for (int k = 0; k < ntiles; ++k) {
            const int sl = (gtile + k) % kSlots;
            tc::mbar_wait(&sl_full[sl], ((gtile + k) / kSlots) & 1);
            tc::fence_after_sync();
            float v[16];
            tc::tmem_ld_32x32b_x16(lane_addr + (uint32_t)(sl * kWin), v);
            if (k < ntiles - kResident) {   // the last kResident tiles stay for pass B
              tc::fence_before_sync();
              __syncwarp();
              if (lane == 0) tc::mbar_arrive(&sl_empty[sl]);
            }
            const int t = k * kTileM + row;
  #pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (t < T_len && t <= T_len - kWin + grp * 16 + j) {
                const float x = v[j] * scale;
                if (x > mref[j] + 8.f) {
                  ssum[j] = (mref[j] == -INFINITY) ? 0.f : ssum[j] * tc::ex2(mref[j] - x);
                  mref[j] = x;
                }
                ssum[j] += tc::ex2(x - mref[j]);
              }
            }
          }
          if (ct == 0) FC_STAMP(it, 3);
          // combine (reference max, sum) over the warp, then over the 4 lane quarters
          float mw[16];
  #pragma unroll
          for (int j = 0; j < 16; ++j) mw[j] = mref[j];
          const float mwarp = tc::warp_reduce16(mw, lane, [](float x, float y) { return fmaxf(x, y); });
          // broadcast each query's warp max back (lanes 2q, 2q+1 hold query q)
  #pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float mj_w = __shfl_sync(0xffffffffu, mwarp, 2 * j);
            ssum[j] = (mref[j] == -INFINITY) ? 0.f : ssum[j] * tc::ex2(mref[j] - mj_w);
            mw[j] = mj_w;
          }
          const float swarp = tc::warp_reduce16(ssum, lane, [](float x, float y) { return x + y; });
          if ((lane & 1) == 0) {
            s_red[cw][lane >> 1] = mw[lane >> 1];
            s_zpart[cw][lane >> 1] = swarp;
          }
          Consumers::sync();
          if (ct < kWin) {
            const int gg = ct >> 4, jj = ct & 15;
            float m = s_red[4 * gg][jj];
            for (int i = 1; i < 4; ++i) m = fmaxf(m, s_red[4 * gg + i][jj]);
            float z = 0.f;
            for (int i = 0; i < 4; ++i) {
              const float mi = s_red[4 * gg + i][jj];
              if (mi != -INFINITY) z += s_zpart[4 * gg + i][jj] * tc::ex2(mi - m);
            }
            s_m[ct] = m;
            s_zinv[ct] = 1.0f / z;
          }
          Consumers::sync();
          float mj[16], zj[16];
  #pragma unroll
          for (int j = 0; j < 16; ++j) {
            mj[j] = s_m[grp * 16 + j];
            zj[j] = s_zinv[grp * 16 + j];
          }
          if (ct == 0) FC_STAMP(it, 8);
          // pass B: normalised probabilities -> window mean; first the resident tail
          // tiles (their slots free as they go, so the re-stream can start), then the
          // re-streamed tiles [0, ntiles - kResident). As in pass 3 of the resident path,
          // the two warp groups split the tiles and a thread covers all 32 queries of its
          // row (statistics of the other group's queries from SMEM), so the window mean is
          // a plain store instead of two contending shared-memory float atomics.
          for (int kk = grp; kk < ntiles; kk += 2) {
            const bool resident = kk < kResident;
            const int k = resident ? ntiles - kResident + kk : kk - kResident;
            const int gk = resident ? gtile + k : gtile + ntiles + k, sl = gk % kSlots;
            if (!resident) {
              tc::mbar_wait(&sl_full[sl], (gk / kSlots) & 1);
              tc::fence_after_sync();
            }
            const uint32_t row_addr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(sl * kWin);
            float sum = 0.f;
  #pragma unroll
            for (int hq = 0; hq < 2; ++hq) {
              float v[16];
              tc::tmem_ld_32x32b_x16(row_addr + (uint32_t)(hq * 16), v);
              if (hq == grp) {
  #pragma unroll
                for (int j = 0; j < 16; ++j) sum = fmaf(tc::ex2(fmaf(v[j], scale, -mj[j])), zj[j], sum);
              } else {
  #pragma unroll
                for (int j = 0; j < 16; ++j)
                  sum = fmaf(tc::ex2(fmaf(v[j], scale, -s_m[hq * 16 + j])), s_zinv[hq * 16 + j], sum);
              }
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&sl_empty[sl], 2);   // stands for both groups' warps
            const int t = k * kTileM + row;
            if (t < n_keep) wacc[t] = sum * inv_wg;
          }
        }
        gtile += snap_loads(ntiles);
        if (kGqa) {
          Consumers::sync();
          for (int t = ct; t < T_len; t += kThreads) {
            s1[t] += sc[t];
            sc[t] = 0.f;
          }
        }
      }
      if (ct == 0) FC_STAMP(it, 4);
      Consumers::sync();
      // avg-pool (zero pad, count_include_pad), forced window
      const int half = pp.pool_kernel / 2;
      const float inv_p = 1.0f / (float)pp.pool_kernel;
      // scores -> order-preserving keys (and the optional score output) in the same pass
      uint32_t* keys = reinterpret_cast<uint32_t*>(sc);
      float* so = out.scores ? out.scores + q.score_off + (int64_t)lh * T_len : nullptr;
      if (pp.pool_kernel == 7) {
        // s1 is 0 on [-8, 0) and on [n_keep, T_len) (T_len = n_keep + 32), so the
        // fixed 7-term window adds exact zeros where the generic loop stops early
        for (int t = ct; t < T_len; t += kThreads) {
          float v = INFINITY;
          if (t < n_keep) {
            float a = 0.f;
#pragma unroll
            for (int u = -3; u <= 3; ++u) a += s1[t + u];
            v = a * inv_p;
          }
          if (so) so[t] = v;
          keys[t] = float_key(v);
        }
      } else {
        for (int t = ct; t < T_len; t += kThreads) {
          float v = INFINITY;
          if (t < n_keep) {
            float a = 0.f;
            const int u0 = max(0, t - half), u1 = min(n_keep - 1, t + half);
            for (int u = u0; u <= u1; ++u) a += s1[u];
            v = a * inv_p;
          }
          if (so) so[t] = v;
          keys[t] = float_key(v);
        }
      }
      Consumers::sync();
      if (ct == 0) FC_STAMP(it, 12);
      // hand the kept list to the compactors (double-buffered)
      tc::mbar_wait(&job_empty[jb], ((it >> 1) & 1) ^ 1);
      if (ct == 0) FC_STAMP(it, 13);
      int32_t* idx = idxbuf + jb * k_stride;
      if (!kSpill)
        for (int i = ct; i < nb; i += kThreads) ctab[jb * nb_stride + i] = table[(int64_t)q.slot * g.max_bpr + i];
      if (ct == 0) FC_STAMP(it, 14);
      if (b.per_segment && q.seg0 < T_len) {
        select_emit<Consumers, kSpill>(keys, q.seg0, q.K0, idx, 0, 0, ss);
        select_emit<Consumers, kSpill>(keys + q.seg0, T_len - q.seg0, K - q.K0, idx, q.K0, q.seg0, ss);
      } else {
        select_emit<Consumers, kSpill>(keys, T_len, K, idx, 0, 0, ss);
      }
      if (out.kept_idx) {
        int32_t* ko = out.kept_idx + q.kept_off + (int64_t)lh * K;
        for (int j = ct; j < K; j += kThreads) ko[j] = idx[j];
      }
      if (ct == 0) s_job[jb] = CompactJob{l, h, K, min(ss.first_drop, K), q.slot};
      Consumers::sync();  // idx, ctab, job complete; sc / ss reused by the next segment
      if (ct == 0) {
        FC_STAMP(it, 5);
        tc::mbar_arrive(&job_full[jb]);
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, kSlots * kWin);
}

// ---------------------------------------------------------------------------
// host side: tensor maps + dispatch
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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

// 2-D row-major tensor map [rows][D]: box = {box_cols elements, box_rows rows}.
// 16-bit types use the 128-byte swizzle (UMMA K-major operands); fp32 is unswizzled.
fc_status encode_rows(CUtensorMap* map, const void* base, int dtype, int D, uint64_t rows,
                      int box_rows) {
  auto enc = get_encode();
  if (!enc) return set_error(FC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const bool f32 = dtype == FC_F32;
  const int esz = f32 ? 4 : 2;
  const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)D * esz};
  const cuuint32_t box[2] = {f32 ? (cuuint32_t)D : 64u, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                     : (dtype == FC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                         : CU_TENSOR_MAP_DATA_TYPE_FLOAT16);
  CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   f32 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(FC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return FC_OK;
}

bool snapkv_tc_supported(const Geom& g, int dtype, const PressParams& pp, int max_T, int max_K) {
  static const bool forced_simt = [] {
    const char* e = getenv("FASTCACHE_SNAPKV_SIMT");
    return e && e[0] == '1';
  }();
  if (forced_simt) return false;
  if (dtype != FC_F16 && dtype != FC_BF16) return false;
  if (g.D != 64 && g.D != 128) return false;
  if (pp.num_q_heads % g.H != 0 || pp.num_q_heads / g.H > 8) return false;   // GQA: gq <= 8
  if (pp.window != 32) return false;               // one 32x32b.x32 TMEM load per tile
  if (g.bs < 8 || g.bs > 128) return false;
  // segments beyond the TMEM ring (T > kSlots * 128) take the two-pass path, beyond the
  // SMEM arrays the spill variant: any T runs on the tensor cores
  (void)max_T;
  (void)max_K;
  return true;
}

static bool snap_needs_spill(const Geom& g, int max_T, int max_K) {
  return tc_smem_plan(g.D, g.bs, max_T, max_K).total > kDynSmemBudget;
}

int64_t snapkv_tc_workspace_floats(const Geom& g, int max_T, int max_K) {
  return snap_needs_spill(g, max_T, max_K) ? (int64_t)sm_count() * snap_spill_floats(max_T, max_K) : 0;
}

fc_status launch_snapkv_tc(const Geom& g, int dtype, char* arena, const int32_t* table,
                           const PressBatch& b, const PressParams& pp, const fc_press_inputs& in,
                           const fc_press_outputs& out, float* ws, int64_t ws_floats,
                           cudaStream_t stream, bool dry_run) {
  const int n_requests_total = b.n_total;
  CUtensorMap kmap, qmap;
  const uint64_t rows = (uint64_t)g.L * g.num_blocks * 2 * g.H * g.bs;
  fc_status st = encode_rows(&kmap, arena, dtype, g.D, rows, g.bs);
  if (st != FC_OK) return st;
  st = encode_rows(&qmap, in.q_window, dtype, g.D,
                   (uint64_t)n_requests_total * g.L * pp.num_q_heads * pp.window, pp.window);
  if (st != FC_OK) return st;
  int max_K = 1;
  for (int i = 0; i < b.n; ++i) max_K = max_K > b.req[i].K ? max_K : b.req[i].K;
  const bool spill = snap_needs_spill(g, b.max_T, max_K);
  const TcSmem plan = tc_smem_plan(g.D, g.bs, b.max_T, max_K, spill);
  if (plan.total > kDynSmemBudget)
    return set_error(FC_ERR_UNSUPPORTED, "SnapKV tensor-core plan exceeds the SMEM budget");
  if (dry_run) return FC_OK;   // the pool sizes the spill workspace next
  const int n_items = b.n * g.L * g.H;
  const int sms = sm_count();
  int grid = n_items < sms ? n_items : sms;
  if (spill) {
    const int64_t row = snap_spill_floats(b.max_T, max_K);
    if (ws_floats < row) return set_error(FC_ERR_INVALID_STATE, "SnapKV spill workspace too small");
    grid = (int)std::min<int64_t>(grid, ws_floats / row);
  }
  const bool gqa = pp.num_q_heads != g.H;
  auto launch = [&](auto kern) -> fc_status {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, plan.total);
    if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute(snapkv_tc)");
    kern<<<grid, snap_threads(gqa), plan.total, stream>>>(arena, table, g, b, pp, kmap, qmap, out, n_items,
                                                   max_K, ws);
    note_launch();
    note_path(kPathTc);
    return cuda_check(cudaGetLastError(), "snapkv_tc_kernel");
  };
  // g = 1 gets its own instantiation (the unit loop folds away)
  auto pick = [&](auto tag) -> fc_status {
    using T = decltype(tag);
    if (g.D == 64) {
      if (spill) return gqa ? launch(snapkv_tc_kernel<T, 64, true, true>) : launch(snapkv_tc_kernel<T, 64, false, true>);
      return gqa ? launch(snapkv_tc_kernel<T, 64, true, false>) : launch(snapkv_tc_kernel<T, 64, false, false>);
    }
    if (spill) return gqa ? launch(snapkv_tc_kernel<T, 128, true, true>) : launch(snapkv_tc_kernel<T, 128, false, true>);
    return gqa ? launch(snapkv_tc_kernel<T, 128, true, false>) : launch(snapkv_tc_kernel<T, 128, false, false>);
  };
  return dtype == FC_BF16 ? pick(__nv_bfloat16()) : pick(__half());
}

}  // namespace fc

#ifdef FC_TRACE
extern "C" FC_API fc_status fc_debug_trace_read(void* host, uint64_t bytes) {
  return fc::cuda_check(cudaMemcpyFromSymbol(host, fc::g_fc_trace, bytes), "trace read");
}
#endif
