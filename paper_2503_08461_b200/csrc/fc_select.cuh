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
  static constexpr int kSize = kThreads;
  __device__ __forceinline__ static int tid() { return threadIdx.x; }
  __device__ __forceinline__ static void sync() { __syncthreads(); }
};
// kCount threads from kFirstThread on (kThreads for the select / press groups; the
// compaction helpers also run on smaller groups)
template <int kFirstThread, int kBarrierId, int kCount = kThreads>
struct NamedGroup {
  static constexpr int kSize = kCount;
  __device__ __forceinline__ static int tid() { return threadIdx.x - kFirstThread; }
  __device__ __forceinline__ static void sync() {
    asm volatile("bar.sync %0, %1;" ::"n"(kBarrierId), "n"(kCount) : "memory");
  }
};

#ifndef FC_SEL_MARK
#define FC_SEL_MARK(i) ((void)0)  // phase stamps (scripts/select_bench.cu)
#endif
#ifndef FC_SEL_EXACT
#define FC_SEL_EXACT 1
#endif


constexpr int kHistWords = 512;     // 1024 packed 16-bit bins, or 512 32-bit bins

struct alignas(16) SelectScratch {
  uint32_t hist[kHistWords];      // radix histogram (warp 0 zeroes it while scanning)
  int32_t warp_tot[kWarps];
  uint32_t emit_tot[2][kWarps];   // emission: per-warp (> tau, == tau) counts
  int32_t sel_bin;
  int32_t sel_krem;
  int32_t sel_exact;
  int32_t first_drop;
  float red[kWarps * 4];
  uint32_t rng[3][kWarps];        // per-warp (min finite key, max finite key, forced-keep count)
};

// Key of +inf: forced keeps (SnapKV window, EA sinks) score +inf and sit above
// every finite key.
constexpr uint32_t kKeyInf = 0xFF800000u;

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

// keys[i .. i+3] (16-B load when the array is 16-B aligned); lanes past n read 0
// and are masked out by the callers' index checks.
__device__ __forceinline__ uint4 load_quad(const uint32_t* keys, int i, int n, bool vec) {
  if (vec && i + 3 < n) return *reinterpret_cast<const uint4*>(keys + i);
  uint4 v;
  v.x = i < n ? keys[i] : 0u;
  v.y = i + 1 < n ? keys[i + 1] : 0u;
  v.z = i + 2 < n ? keys[i + 2] : 0u;
  v.w = i + 3 < n ? keys[i + 3] : 0u;
  return v;
}
__device__ __forceinline__ uint32_t quad_at(const uint4& v, int e) {
  return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
}
// Predicated shared-memory add (no branch or reconvergence point per key) and a
// conditional store.
__device__ __forceinline__ void red_add_if(uint32_t* addr, uint32_t v, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q red.shared.add.u32 [%0], %1;\n}" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(addr)),
               "r"(v), "r"((uint32_t)p)
               : "memory");
}
__device__ __forceinline__ void st_if(int32_t* addr, int32_t v, bool p) {
  if (p) *addr = v;   // plain C++: the compiler keeps the address space (STS for SMEM buffers)
}

// Warp 0 of a select: find the bin holding the krem-th largest counted key
// (s.sel_bin / sel_krem / sel_exact) and clear the histogram for the next pass.
// Lane l owns words [16l, 16l + 16): bins [32l, 32l + 32) packed, [16l, 16l + 16)
// not. Level 1 picks the lane by a suffix scan of the lanes' totals, level 2 the
// bin inside it by a suffix scan over that lane's bins, one bin per lane.
__device__ __forceinline__ void hist_boundary(SelectScratch& s, bool packed, int krem, int lane) {
  uint32_t w[16];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint4 x = *reinterpret_cast<const uint4*>(&s.hist[16 * lane + 4 * c]);
    w[4 * c] = x.x;
    w[4 * c + 1] = x.y;
    w[4 * c + 2] = x.z;
    w[4 * c + 3] = x.w;
  }
  uint32_t local = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) local += packed ? (w[c] & 0xFFFFu) + (w[c] >> 16) : w[c];
  uint32_t incl = local;  // sum over lanes >= lane
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_down_sync(0xffffffffu, incl, off);
    if (lane + off < 32) incl += y;
  }
  // level 1: the lane whose bins hold the krem-th largest finite key
  const unsigned hit = __ballot_sync(0xffffffffu, incl - local < (uint32_t)krem && (uint32_t)krem <= incl);
  const int L = __ffs(hit) - 1;
  const uint32_t above_L = __shfl_sync(0xffffffffu, incl - local, L);
  // level 2: lane j takes bin j of lane L's range (packed: 32 bins, else 16)
  const int per = packed ? 32 : 16;
  const int bin = L * per + lane;
  const uint32_t wv = s.hist[packed ? bin >> 1 : min(bin, kHistWords - 1)];
  const uint32_t cnt = lane < per ? (packed ? (wv >> ((bin & 1) << 4)) & 0xFFFFu : wv) : 0u;
  uint32_t sfx = cnt;     // sum over bins >= this one within lane L's range
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_down_sync(0xffffffffu, sfx, off);
    if (lane + off < 32) sfx += y;
  }
  const uint32_t cum = above_L + sfx - cnt;   // keys in bins above this one
  if (lane < per && cum < (uint32_t)krem && (uint32_t)krem <= cum + cnt) {
    s.sel_bin = bin;
    s.sel_krem = krem - (int)cum;
    s.sel_exact = (cum + cnt == (uint32_t)krem) ? 1 : 0;  // the whole bin is kept
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c)   // clear this lane's words for the next pass
    *reinterpret_cast<uint4*>(&s.hist[16 * lane + 4 * c]) = make_uint4(0, 0, 0, 0);
}

// ---------------------------------------------------------------------------
// Segmented top-K: select_emit = threshold (tau, need) + emission.
//
// Top-K of keys[0..n) by (key desc, index asc); writes idx_base + i of the kept
// i, ascending, to out[out_base ...]; lowers s.first_drop to the first dropped
// idx_base + i. Kept: every key > tau, plus the first `need` keys == tau.
// `out` may alias `keys`: kept element i lands at G(i) + min(E(i), need) <= i
// (G/E = greater/equal-to-threshold keys before i).
//
// The select is latency-bound (8 warps, 25-45-cycle SHFL / REDUX / LDS / barrier
// links measured on B200, scripts/lat_probe.cu), so each piece is shaped to cut
// dependent steps and barriers (scripts/select_bench.cu times them in isolation):
//
// Threshold, n <= kSmallN: radix select on absolute 8-bit digits, a pass ending
//   early once its boundary bin is kept whole (one warp scans 8 bins per lane; the
//   next pass's histogram is cleared behind the scan's barrier).
// Threshold, n > kSmallN: digits of the offset r = k - kmin from the smallest finite
//   key, 10 bits wide with packed 16-bit counters (n < 65536; else 9 bits / 32-bit),
//   starting at the highest bit the finite keys span: one segment's scores share
//   their sign and most exponent bits, so absolute top digits put almost every key
//   in a few bins (a wasted pass); offsets spread them and ~8k keys resolve in two
//   passes instead of three or four. Forced keeps (+inf keys) are counted apart and
//   kept first. Warp 0 finds the boundary bin with a two-level warp scan.
// Emission, kSmallN < n <= 8192 (emit_packed): each warp owns a contiguous range of
//   128-key rounds. One read classifies its keys (> tau, == tau) into 4 + 4 bits per
//   lane per round held in registers, with the per-round counts packed into 8-bit
//   fields: one 5-step warp scan serves every round, one barrier exchanges the warp
//   totals, and no key is read after it, so writing `out` over `keys` is safe.
// Emission otherwise (emit_supertile): 1024-key super-tiles, one ballot scan and one
//   barrier per super-tile. For ~1k keys this measured better inside the
//   SnapKV kernel (its compactors are the bottleneck there and the packed form's
//   extra issue slows them: c3 6.22 vs 6.38 ms), while for EA's ~8k-key segments the
//   packed form halves the emission (scripts/select_bench.cu: 24.9k -> 14.5k cycles
//   per EA-like select in all).
constexpr int kSmallN = 4096;

template <class G>
__device__ __forceinline__ void threshold_abs8(const uint32_t* keys, int n, int K,
                                               SelectScratch& s, uint32_t& tau, int& need) {
  const int tid = G::tid(), lane = threadIdx.x & 31;
  uint32_t prefix = 0, mask = 0;
  int krem = K;
  bool exact = false;
  for (int i = tid; i < 256; i += kThreads) s.hist[i] = 0;
  G::sync();
#pragma unroll 1
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    uint32_t* hist = s.hist + (pass & 1) * 256;
#pragma unroll 4
    for (int base = 0; base < n; base += kThreads) {
      const int i = base + tid;
      if (i < n) {
        const uint32_t k = keys[i];
        if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
      }
    }
    G::sync();
    FC_SEL_MARK(2 + pass * 2);
    if (tid >= 32) {
      // the next pass's histogram is cleared while warp 0 scans this one
      for (int i = tid - 32; i < 256; i += kThreads - 32) s.hist[((pass + 1) & 1) * 256 + i] = 0;
    } else {
      constexpr int per = 8;  // 8 bins per lane, lane 31 owns the top
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
    FC_SEL_MARK(3 + pass * 2);
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
  tau = exact ? prefix - 1u : prefix;
  need = exact ? 0 : krem;
}

template <class G>
__device__ __forceinline__ void threshold_rel(const uint32_t* keys, int n, int K, SelectScratch& s,
                                              uint32_t& tau, int& need) {
  const int tid = G::tid(), lane = threadIdx.x & 31, warp = tid >> 5;
  const bool vec = (reinterpret_cast<uintptr_t>(keys) & 15u) == 0;
  const int nq = (n + 3) >> 2;
  constexpr int kB = 4;   // quads in flight per thread
  // ---- range of the finite keys, forced-keep count ----
  uint32_t kmin = 0xFFFFFFFFu, kmax = 0u, ninf = 0u;
  for (int q0 = tid; q0 < nq; q0 += kB * kThreads) {
    uint4 v[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) v[u] = load_quad(keys, 4 * (q0 + u * kThreads), n, vec);
#pragma unroll
    for (int u = 0; u < kB; ++u)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t k = quad_at(v[u], e);
        const bool valid = 4 * (q0 + u * kThreads) + e < n;
        const bool inf = k >= kKeyInf;
        ninf += (valid && inf) ? 1u : 0u;
        kmin = (valid && !inf) ? min(kmin, k) : kmin;
        kmax = (valid && !inf) ? max(kmax, k) : kmax;
      }
  }
  kmin = __reduce_min_sync(0xffffffffu, kmin);
  kmax = __reduce_max_sync(0xffffffffu, kmax);
  ninf = __reduce_add_sync(0xffffffffu, ninf);
  if (lane == 0) {
    s.rng[0][warp] = kmin;
    s.rng[1][warp] = kmax;
    s.rng[2][warp] = ninf;
  }
  for (int i = tid; i < kHistWords; i += kThreads) s.hist[i] = 0;
  G::sync();
  kmin = s.rng[0][0];
  kmax = s.rng[1][0];
  ninf = s.rng[2][0];
#pragma unroll
  for (int w = 1; w < kWarps; ++w) {
    kmin = min(kmin, s.rng[0][w]);
    kmax = max(kmax, s.rng[1][w]);
    ninf += s.rng[2][w];
  }
  FC_SEL_MARK(1);
  if ((uint32_t)K <= ninf) {
    tau = kKeyInf;   // only forced keeps survive: the first K of them by index
    need = K;
    return;
  }
  // n - ninf > K - ninf >= 1 finite keys, so kmin <= kmax
  const bool packed = n < 65536;
  const int dbits = packed ? 10 : 9;
  const uint32_t range = kmax - kmin;
  int hi = range ? 32 - __clz((int)range) : 0;   // bits of r still unresolved: [0, hi)
  uint32_t prefix = 0, mask = 0;
  int krem = K - (int)ninf;
  bool exact = false;
#pragma unroll 1
  for (int pass = 0; hi > 0; ++pass) {
    const int lo = hi > dbits ? hi - dbits : 0;
    const uint32_t dmask = (1u << (hi - lo)) - 1u;
    for (int q0 = tid; q0 < nq; q0 += kB * kThreads) {
      uint4 v[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) v[u] = load_quad(keys, 4 * (q0 + u * kThreads), n, vec);
#pragma unroll
      for (int u = 0; u < kB; ++u)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t k = quad_at(v[u], e);
          const uint32_t r = k - kmin;
          const bool hit = 4 * (q0 + u * kThreads) + e < n && k < kKeyInf && (r & mask) == prefix;
          const uint32_t b = (r >> lo) & dmask;
          red_add_if(&s.hist[packed ? b >> 1 : b], packed ? 1u << ((b & 1u) << 4) : 1u, hit);
        }
    }
    G::sync();
    FC_SEL_MARK(2 + min(pass, 3) * 2);
    if (tid < 32) hist_boundary(s, packed, krem, lane);
    G::sync();
    FC_SEL_MARK(3 + min(pass, 3) * 2);
    prefix |= (uint32_t)s.sel_bin << lo;
    mask |= dmask << lo;
    krem = s.sel_krem;
    hi = lo;
    // Early exit: the boundary bin is kept whole, so the finite kept set is
    // exactly {r : (r & mask) >= prefix} = {r : r >= prefix} -- no need to
    // resolve the lower digits (prefix >= 1 here: some finite key is dropped).
    if (FC_SEL_EXACT && s.sel_exact) {
      exact = true;
      break;
    }
  }
  tau = kmin + (exact ? prefix - 1u : prefix);
  need = exact ? 0 : krem;
}

constexpr int kEmitMaxRounds = 8;   // packed emission: n <= 8 warps x 8 x 128 keys

// Emission for n <= 8192. Warp w owns rounds [0, rounds) of 128 keys at
// w * rounds * 128 (lane l: 4 keys per round). Per lane the (> tau, == tau) bits
// of every round sit in two words (4 bits per round) and their counts in 8-bit
// fields of two 64-bit words; ONE 5-step warp scan of those packed counts gives
// every round's lane prefix at once (fields never carry: <= 32 x 4 per round).
template <class G>
__device__ __forceinline__ void emit_packed(const uint32_t* keys, int n, int32_t* out,
                                            int out_base, int idx_base, SelectScratch& s,
                                            uint32_t tau, int need, int rounds) {
  const int tid = G::tid(), lane = threadIdx.x & 31, warp = tid >> 5;
  const bool vec = (reinterpret_cast<uintptr_t>(keys) & 15u) == 0;
  const int a = warp * rounds * 128 + lane * 4;
  uint32_t gm = 0, em = 0;       // bits 4j..4j+3: round j
  uint64_t gc = 0, ec = 0;       // byte j: popc of round j
#pragma unroll 1
  for (int j0 = 0; j0 < rounds; j0 += 2) {
    uint4 v[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) v[u] = load_quad(keys, a + (j0 + u) * 128, n, vec);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = j0 + u, i0 = a + j * 128;
      const int nvalid = j < rounds ? min(max(n - i0, 0), 4) : 0;
      const uint32_t vm = (1u << nvalid) - 1u;
      const uint32_t gb = ((v[u].x > tau) | ((v[u].y > tau) << 1) | ((v[u].z > tau) << 2) |
                           ((v[u].w > tau) << 3)) & vm;
      const uint32_t eb = ((v[u].x == tau) | ((v[u].y == tau) << 1) | ((v[u].z == tau) << 2) |
                           ((v[u].w == tau) << 3)) & vm;
      gm |= gb << (4 * j);
      em |= eb << (4 * j);
      gc |= (uint64_t)__popc(gb) << (8 * j);
      ec |= (uint64_t)__popc(eb) << (8 * j);
    }
  }
  // inclusive lane scans of the packed per-round counts (independent chains)
  uint64_t gi = gc, ei = ec;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint64_t yg = __shfl_up_sync(0xffffffffu, gi, off);
    const uint64_t ye = __shfl_up_sync(0xffffffffu, ei, off);
    gi += lane >= off ? yg : 0ull;
    ei += lane >= off ? ye : 0ull;
  }
  const uint64_t gt_tot = __shfl_sync(0xffffffffu, gi, 31), eq_tot = __shfl_sync(0xffffffffu, ei, 31);
  if (lane == 0) {
    uint32_t tg = 0, te = 0;
    for (int j = 0; j < rounds; ++j) {
      tg += (uint32_t)(gt_tot >> (8 * j)) & 0xFFu;
      te += (uint32_t)(eq_tot >> (8 * j)) & 0xFFu;
    }
    s.emit_tot[0][warp] = tg;
    s.emit_tot[1][warp] = te;
  }
  G::sync();   // every key of the segment has been read: `out` may now overwrite them
  int g_run = 0, e_run = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    g_run += w < warp ? (int)s.emit_tot[0][w] : 0;
    e_run += w < warp ? (int)s.emit_tot[1][w] : 0;
  }
  const uint64_t gx = gi - gc, ex = ei - ec;   // exclusive lane prefixes, per round byte
  int first_drop = INT_MAX;
#pragma unroll 1
  for (int j = 0; j < rounds; ++j) {
    const uint32_t gb = (gm >> (4 * j)) & 15u, eb = (em >> (4 * j)) & 15u;
    int gpos = g_run + (int)((gx >> (8 * j)) & 0xFFu);
    int epos = e_run + (int)((ex >> (8 * j)) & 0xFFu);
    const int i0 = a + j * 128;
    const int nvalid = min(max(n - i0, 0), 4);
    uint32_t keptb = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const bool gt = (gb >> e) & 1u, eq = (eb >> e) & 1u;
      const bool kept = gt || (eq && epos < need);
      st_if(out + out_base + gpos + min(epos, need), idx_base + i0 + e, kept);
      keptb |= kept ? 1u << e : 0u;
      gpos += gt;
      epos += eq;
    }
    const uint32_t dropb = ((1u << nvalid) - 1u) & ~keptb;
    first_drop = (first_drop == INT_MAX && dropb) ? i0 + __ffs(dropb) - 1 : first_drop;
    g_run += (int)((gt_tot >> (8 * j)) & 0xFFu);
    e_run += (int)((eq_tot >> (8 * j)) & 0xFFu);
  }
  first_drop = __reduce_min_sync(0xffffffffu, first_drop);
  if (lane == 0 && first_drop != INT_MAX) atomicMin(&s.first_drop, idx_base + first_drop);
}

#ifndef FC_EMIT_R
#define FC_EMIT_R 4
#endif
template <class G>
__device__ __forceinline__ void emit_supertile(const uint32_t* keys, int n, int32_t* out,
                                               int out_base, int idx_base, SelectScratch& s,
                                               uint32_t tau, int need) {
  const int tid = G::tid(), lane = threadIdx.x & 31, warp = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
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
}

// kWide = false compiles only the absolute-digit threshold and the super-tile
// emission (the short-segment forms): kernels whose hot segments are short keep
// the smaller code (the warp-specialised SnapKV kernel is ~10k instructions and
// measurably sensitive to its layout).
template <class G = CtaGroup, bool kWide = true>
__device__ void select_emit(const uint32_t* keys, int n, int K, int32_t* out, int out_base,
                            int idx_base, SelectScratch& s) {
  const int tid = G::tid();
  if (K >= n) {
    for (int i = tid; i < n; i += kThreads) out[out_base + i] = idx_base + i;
    G::sync();
    return;
  }
  FC_SEL_MARK(0);
  uint32_t tau;
  int need;
  if (!kWide || n <= kSmallN)
    threshold_abs8<G>(keys, n, K, s, tau, need);
  else
    threshold_rel<G>(keys, n, K, s, tau, need);
  FC_SEL_MARK(9);
  const int rounds = (((n + kWarps - 1) / kWarps) + 127) >> 7;
  if (kWide && n > kSmallN && rounds <= kEmitMaxRounds)
    emit_packed<G>(keys, n, out, out_base, idx_base, s, tau, need, rounds);
  else
    emit_supertile<G>(keys, n, out, out_base, idx_base, s, tau, need);
  FC_SEL_MARK(10);
  G::sync();
  FC_SEL_MARK(11);
}

// One request's select: the whole segment, or (per-segment budgets) its two modality
// segments one after the other -- a single inlined select_emit either way.
template <class G = CtaGroup, bool kWide = true>
__device__ __forceinline__ void select_request(const uint32_t* keys, int T, int K, int seg0, int K0,
                                               bool per_segment, int32_t* idx, SelectScratch& s) {
  const int nseg = (per_segment && seg0 < T) ? 2 : 1;
#pragma unroll 1
  for (int sg = 0; sg < nseg; ++sg) {
    const int lo = nseg == 2 && sg == 1 ? seg0 : 0;
    const int n = nseg == 2 ? (sg == 0 ? seg0 : T - seg0) : T;
    const int k = nseg == 2 ? (sg == 0 ? K0 : K - K0) : K;
    const int ob = nseg == 2 && sg == 1 ? K0 : 0;
    select_emit<G, kWide>(keys + lo, n, k, idx, ob, lo, s);
  }
}

template <typename T>
struct RowCfg {
  static constexpr int kEPV = 16 / sizeof(T);
};

template <int kRowBytes, int kItems, class G = CtaGroup>
struct Compactor {
  static constexpr int kVecs = kRowBytes / 16;
  static constexpr int kChunk = G::kSize * kItems / (2 * kVecs);  // ranks per chunk
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
      const int item = it * G::kSize + G::tid();
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
    for (int r = G::tid(); r < 2 * kChunk; r += G::kSize) {
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
      const int item = it * G::kSize + G::tid();
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
  static constexpr int kItems = kRanks * 2 * kVecs / G::kSize;  // 16-B pieces per thread
  static_assert(kItems * G::kSize == kRanks * 2 * kVecs, "chunk must split evenly over the group");
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
        const int v = it * G::kSize + G::tid();
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
      const int v = it * G::kSize + G::tid();
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
