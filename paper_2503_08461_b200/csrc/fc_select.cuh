// fc_select.cuh -- device building blocks shared by the press kernels:
// block scans, the segmented radix top-k (select_emit) and the in-place
// kept-row compaction (compact_rows). See fc_press.cu for the phase contract.
#pragma once

#include <climits>

#include "fc_internal.cuh"

namespace fc {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// A set of 256 threads that cooperates on one segment: the whole CTA, or the
// consumer warps of a warp-specialised kernel synchronising on a named barrier.
struct CtaGroup {
  __device__ __forceinline__ static int tid() { return threadIdx.x; }
  __device__ __forceinline__ static void sync() { __syncthreads(); }
};
template <int kFirstThread, int kBarrierId>
struct NamedGroup {
  __device__ __forceinline__ static int tid() { return threadIdx.x - kFirstThread; }
  __device__ __forceinline__ static void sync() {
    asm volatile("bar.sync %0, %1;" ::"n"(kBarrierId), "n"(kThreads) : "memory");
  }
};

constexpr int kRadixBins = 256;  // 8-bit digits, 4 passes
#ifndef FC_SEL_EXACT
#define FC_SEL_EXACT 1
#endif

struct SelectScratch {
  uint32_t hist[2][kRadixBins];   // double-buffered: pass p counts into hist[p & 1]
  int32_t warp_tot[kWarps];
  uint32_t emit_tot[2][kWarps];   // double-buffered packed (gt | eq << 16) warp counts
  int32_t sel_bin;
  int32_t sel_krem;
  int32_t sel_exact;
  int32_t first_drop;
  float red[kWarps * 4];
};

// Block-wide exclusive scan of a predicate (all threads must call).
template <class G = CtaGroup>
__device__ __forceinline__ int block_excl_scan(bool pred, int32_t* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, warp = G::tid() >> 5;
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  const int in_warp = __popc(m & ((1u << lane) - 1u));
  if (lane == 0) warp_tot[warp] = __popc(m);
  G::sync();
  int before = 0;
  total = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const int c = warp_tot[w];
    before += (w < warp) ? c : 0;
    total += c;
  }
  G::sync();
  return before + in_warp;
}

// Top-K of keys[0..n) by (key desc, index asc); writes idx_base + i of the kept
// i, ascending, to out[out_base ...]; lowers s.first_drop to the first dropped
// idx_base + i. `out` may alias `keys`: kept element i lands at
// G(i) + min(E(i), need) <= i (G/E = greater/equal-to-threshold keys before i).
//
// Threshold: 4-pass radix select on 8-bit digits (one warp scans 8 bins per
// lane; the next pass's histogram reset rides behind the scan's barrier).
// Emission: one ballot scan per 256-key tile carrying both the > tau and == tau
// counts, double-buffered so each tile costs a single barrier.
template <class G = CtaGroup>
__device__ void select_emit(const uint32_t* keys, int n, int K, int32_t* out, int out_base,
                            int idx_base, SelectScratch& s) {
  const int tid = G::tid(), lane = threadIdx.x & 31, warp = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  if (K >= n) {
    for (int i = tid; i < n; i += kThreads) out[out_base + i] = idx_base + i;
    G::sync();
    return;
  }
  uint32_t prefix = 0, mask = 0;
  int krem = K;
  bool exact = false;
  for (int i = tid; i < kRadixBins; i += kThreads) s.hist[0][i] = 0;
  G::sync();
#pragma unroll 1
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    uint32_t* hist = s.hist[pass & 1];
#pragma unroll 4
    for (int base = 0; base < n; base += kThreads) {
      const int i = base + tid;
      if (i < n) {
        const uint32_t k = keys[i];
        if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
      }
    }
    G::sync();
    if (tid >= 32) {
      // the next pass's histogram is cleared while warp 0 scans this one
      for (int i = tid - 32; i < kRadixBins; i += kThreads - 32) s.hist[(pass + 1) & 1][i] = 0;
    } else {
      constexpr int per = kRadixBins / 32;  // 8 bins per lane, lane 31 owns the top
      uint32_t c[per];
      uint32_t local = 0;
#pragma unroll
      for (int b = 0; b < per; ++b) {
        c[b] = hist[lane * per + b];
        local += c[b];
      }
      uint32_t incl = local;  // sum over lanes >= lane
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, incl, off);
        if (lane + off < 32) incl += y;
      }
      const uint32_t above = incl - local;
      if (above < (uint32_t)krem && (uint32_t)krem <= incl) {
        uint32_t cum = above;
#pragma unroll
        for (int b = per - 1; b >= 0; --b) {
          if (cum + c[b] >= (uint32_t)krem) {
            s.sel_bin = lane * per + b;
            s.sel_krem = krem - (int)cum;
            s.sel_exact = (cum + c[b] == (uint32_t)krem) ? 1 : 0;  // the whole bin is kept
            break;
          }
          cum += c[b];
        }
      }
    }
    G::sync();
    prefix |= (uint32_t)s.sel_bin << shift;
    mask |= 255u << shift;
    krem = s.sel_krem;
    // Early exit: the boundary bin is kept whole, so the kept set is exactly
    // {k : (k & mask) >= prefix} = {k : k >= prefix} -- no need to resolve the
    // lower digits (prefix >= 1 here because K < n).
    if (FC_SEL_EXACT && s.sel_exact) {
      exact = true;
      break;
    }
  }
  const uint32_t tau = exact ? prefix - 1u : prefix;
  const int need = exact ? 0 : krem;
  // Emission in super-tiles of kEmitR x 256 keys (warp w owns kEmitR x 32
  // consecutive keys, one ballot per 32): one barrier per super-tile.
#ifndef FC_EMIT_R
#define FC_EMIT_R 4
#endif
  constexpr int kEmitR = FC_EMIT_R;
  int run_gt = 0, run_eq = 0, buf = 0;
  bool drop_found = false;
  for (int base = 0; base < n; base += kThreads * kEmitR, buf ^= 1) {
    const int wbase = base + warp * 32 * kEmitR;
    unsigned bg[kEmitR], be[kEmitR];
    int cg = 0, ce = 0;
#pragma unroll
    for (int r = 0; r < kEmitR; ++r) {
      const int i = wbase + r * 32 + lane;
      const bool valid = i < n;
      const uint32_t k = valid ? keys[i] : 0u;
      bg[r] = __ballot_sync(0xffffffffu, valid && k > tau);
      be[r] = __ballot_sync(0xffffffffu, valid && k == tau);
      cg += __popc(bg[r]);
      ce += __popc(be[r]);
    }
    if (lane == 0) s.emit_tot[buf][warp] = (uint32_t)cg | ((uint32_t)ce << 16);
    G::sync();
    int g_before = 0, e_before = 0, g_tot = 0, e_tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = s.emit_tot[buf][w];
      const int wg = (int)(c & 0xFFFFu), we = (int)(c >> 16);
      g_before += w < warp ? wg : 0;
      e_before += w < warp ? we : 0;
      g_tot += wg;
      e_tot += we;
    }
    int g_run = run_gt + g_before, e_run = run_eq + e_before;
#pragma unroll
    for (int r = 0; r < kEmitR; ++r) {
      const int i = wbase + r * 32 + lane;
      const bool valid = i < n;
      const bool gt = (bg[r] >> lane) & 1u, eq = (be[r] >> lane) & 1u;
      const int G_i = g_run + __popc(bg[r] & lt_mask);
      const int E_i = e_run + __popc(be[r] & lt_mask);
      const bool kept = gt || (eq && E_i < need);
      if (kept) out[out_base + G_i + min(E_i, need)] = idx_base + i;
      if (!drop_found) {
        const unsigned dropped = __ballot_sync(0xffffffffu, valid && !kept);
        if (dropped) {
          if (lane == 0) atomicMin(&s.first_drop, idx_base + wbase + r * 32 + __ffs(dropped) - 1);
          drop_found = true;  // later keys of this warp only hold larger indices
        }
      }
      g_run += __popc(bg[r]);
      e_run += __popc(be[r]);
    }
    run_gt += g_tot;
    run_eq += e_tot;
  }
  G::sync();
}

template <typename T>
struct RowCfg {
  static constexpr int kEPV = 16 / sizeof(T);
};

template <int kRowBytes, int kItems, class G = CtaGroup>
struct Compactor {
  static constexpr int kVecs = kRowBytes / 16;
  static constexpr int kChunk = kThreads * kItems / (2 * kVecs);  // ranks per chunk
  char* seg;
  const Geom& g;
  const int32_t* s_src;
  const int32_t* s_dst;
  const int32_t* idx;
  int K;
  int64_t kv_off;

  __device__ __forceinline__ void load(int j0, uint4 (&buf)[kItems]) const {
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int item = it * kThreads + G::tid();
      const int row = item / (2 * kVecs), rem = item % (2 * kVecs);
      const int kv = rem / kVecs, vec = rem % kVecs;
      const int j = j0 + row;
      if (j < K) {
        const int src = idx[j];
        buf[it] = ld_stream(seg + kv * kv_off + (int64_t)s_src[src >> g.bs_shift] * g.block_stride +
                            (int64_t)(src & (g.bs - 1)) * kRowBytes + vec * 16);
      }
    }
  }
  // Pull the source rows (K and V) of ranks [j0, j0 + kChunk) towards L2 so the
  // later register loads hit L2: one bulk prefetch per row, no registers held.
  __device__ __forceinline__ void prefetch(int j0) const {
    for (int r = G::tid(); r < 2 * kChunk; r += kThreads) {
      const int kv = r >= kChunk, j = j0 + (kv ? r - kChunk : r);
      if (j < K) {
        const int src = idx[j];
        const char* p = seg + kv * kv_off + (int64_t)s_src[src >> g.bs_shift] * g.block_stride +
                        (int64_t)(src & (g.bs - 1)) * kRowBytes;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "n"(kRowBytes) : "memory");
      }
    }
  }
  __device__ __forceinline__ void store(int j0, const uint4 (&buf)[kItems]) const {
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int item = it * kThreads + G::tid();
      const int row = item / (2 * kVecs), rem = item % (2 * kVecs);
      const int kv = rem / kVecs, vec = rem % kVecs;
      const int j = j0 + row;
      if (j < K)
        st_stream(seg + kv * kv_off + (int64_t)s_dst[j >> g.bs_shift] * g.block_stride +
                      (int64_t)(j & (g.bs - 1)) * kRowBytes + vec * 16,
                  buf[it]);
    }
  }
};

// Copy kept rows j <- idx[j] (K and V), chunks of kChunk ranks, software
// pipelined: loads of chunk c+1 are in flight while chunk c is stored. Safe in
// place because idx is ascending (idx[j] >= j): chunk c writes ranks
// [cW, (c+1)W) while chunk c+1 only reads positions >= (c+1)W, and the barrier
// before chunk c+1's stores orders them after every read of chunks <= c+1.
#ifndef FC_PF
#define FC_PF 2
#endif
template <int kRowBytes, class G = CtaGroup, int kItems = 4, int kPrefetch = FC_PF>
__device__ __forceinline__ void compact_rows(char* __restrict__ seg, const Geom& g,
                                             const int32_t* s_src, const int32_t* s_dst,
                                             const int32_t* idx, int K, int j_start) {
  using C = Compactor<kRowBytes, kItems, G>;
  const C c{seg, g, s_src, s_dst, idx, K, (int64_t)g.H * g.bs * kRowBytes};
  if (j_start >= K) return;
  uint4 a[kItems], b[kItems];
  int j0 = j_start;
#pragma unroll
  for (int d = 1; d <= kPrefetch; ++d) c.prefetch(j0 + d * C::kChunk);
  c.load(j0, a);
  G::sync();
  while (true) {
    const int j1 = j0 + C::kChunk;
    if (kPrefetch > 0) c.prefetch(j1 + kPrefetch * C::kChunk);
    if (j1 < K) c.load(j1, b);
    c.store(j0, a);
    if (j1 >= K) break;
    G::sync();
    const int j2 = j1 + C::kChunk;
    if (kPrefetch > 0) c.prefetch(j2 + kPrefetch * C::kChunk);
    if (j2 < K) c.load(j2, a);
    c.store(j1, b);
    if (j2 >= K) break;
    G::sync();
    j0 = j2;
  }
}


// Same contract as compact_rows, but the rows travel through an SMEM ring of
// kNBuf chunks with cp.async (LDGSTS), so kNBuf - 1 chunks of loads are in
// flight without holding registers (the register version keeps one chunk
// ahead). Chunk c = kRanks ranks x {K, V}. Iteration c: wait for chunk c,
// barrier, issue the loads of chunk c + kNBuf - 1 into the buffer chunk c - 1
// used, then store chunk c from SMEM. In place: chunk c stores ranks
// [cW, (c+1)W) only after every load of chunks <= c completed (the barrier),
// and every load still in flight reads positions >= (c+1)W.
template <int kRowBytes, class G, int kRanks, int kNBuf>
struct AsyncCompactor {
  static constexpr int kVecs = kRowBytes / 16;
  static constexpr int kItems = kRanks * 2 * kVecs / kThreads;  // 16-B pieces per thread
  static_assert(kItems * kThreads == kRanks * 2 * kVecs, "chunk must split evenly over the group");
  static constexpr int kChunkBytes = kRanks * 2 * kRowBytes;
  static constexpr int kSmemBytes = kNBuf * kChunkBytes;
};

template <int kRowBytes, class G, int kRanks = 32, int kNBuf = 4>
__device__ __forceinline__ void compact_rows_async(char* __restrict__ seg, const Geom& g,
                                                   const int32_t* s_src, const int32_t* s_dst,
                                                   const int32_t* idx, int K, int j_start,
                                                   unsigned char* smem) {
  using A = AsyncCompactor<kRowBytes, G, kRanks, kNBuf>;
  constexpr int kVecs = A::kVecs;
  if (j_start >= K) return;
  const int64_t kv_off = (int64_t)g.H * g.bs * kRowBytes;
  const int nchunks = (K - j_start + kRanks - 1) / kRanks;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  auto issue = [&](int c) {
    if (c < nchunks) {
      const uint32_t buf = sbase + (uint32_t)((c % kNBuf) * A::kChunkBytes);
#pragma unroll
      for (int it = 0; it < A::kItems; ++it) {
        const int v = it * kThreads + G::tid();
        const int rank = v / (2 * kVecs), rem = v % (2 * kVecs);
        const int kv = rem / kVecs, vec = rem % kVecs;
        const int j = j_start + c * kRanks + rank;
        if (j < K) {
          const int src = idx[j];
          const char* gp = seg + kv * kv_off + (int64_t)s_src[src >> g.bs_shift] * g.block_stride +
                           (int64_t)(src & (g.bs - 1)) * kRowBytes + vec * 16;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(buf + v * 16), "l"(gp)
                       : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");  // uniform group count, even if empty
  };
#pragma unroll
  for (int c = 0; c < kNBuf - 1; ++c) issue(c);
  for (int c = 0; c < nchunks; ++c) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kNBuf - 2) : "memory");
    G::sync();  // chunk c landed everywhere; chunk c-1's buffer fully read
    issue(c + kNBuf - 1);
    const unsigned char* buf = smem + (c % kNBuf) * A::kChunkBytes;
#pragma unroll
    for (int it = 0; it < A::kItems; ++it) {
      const int v = it * kThreads + G::tid();
      const int rank = v / (2 * kVecs), rem = v % (2 * kVecs);
      const int kv = rem / kVecs, vec = rem % kVecs;
      const int j = j_start + c * kRanks + rank;
      if (j < K)
        st_stream(seg + kv * kv_off + (int64_t)s_dst[j >> g.bs_shift] * g.block_stride +
                      (int64_t)(j & (g.bs - 1)) * kRowBytes + vec * 16,
                  *reinterpret_cast<const uint4*>(buf + v * 16));
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

}  // namespace fc
