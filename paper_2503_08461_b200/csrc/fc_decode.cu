// fc_decode.cu -- the step after the hot path: decode
// over the compacted paged blocks.
//
//   write_decode_kv_kernel  one new token's K/V per request for one layer into
//                           its slot (the UpdateKVCache of PAPER.md:255-261;
//                           the block itself was popped by fc_pool_append,
//                           reference pool.py:194-211)
//   decode_attn_kernel      paged attention of one query token per request
//                           over every live token of its handle, one layer:
//                           split-KV (flash-decoding) with the last CTA of a
//                           (request, kv-head) merging the split partials.
//
// Roofline: HBM. Per (request, kv-head) the kernel reads T*2*D*bpe bytes of
// K/V and does 4*D*g flops per token (g = query heads per kv head), i.e. g
// flops per byte at fp16 -- far below even the SIMT ridge, so the design goal
// is bytes in flight, not math: every lane owns one 16-B vector of a row and
// keeps kTile rows of K and V (2 x kTile x 16 B) in flight before it reduces.
#include <cstring>

#include "fc_internal.cuh"

namespace fc {

#ifndef FC_DEC_WARPS
#define FC_DEC_WARPS 4
#endif
constexpr int kDecodeWarps = FC_DEC_WARPS;
constexpr int kDecodeThreads = kDecodeWarps * 32;

// The lane-group geometry of a row: kVpr 16-B vectors per row, kRows rows per
// warp-wide load, kTile row-groups in flight per lane.
template <typename T, int D, int G>
struct DecodeCfg {
  static constexpr int kEPV = 16 / (int)sizeof(T);
  static constexpr int kVpr = D / kEPV;
  static_assert(kVpr >= 1 && kVpr <= 32 && (32 % kVpr) == 0, "row must split evenly over a warp");
  static constexpr int kRows = 32 / kVpr;
#ifndef FC_DEC_TILE1
#define FC_DEC_TILE1 4
#endif
  static constexpr int kTile = G >= 4 ? 4 : (G == 1 ? FC_DEC_TILE1 : 8);  // rows in flight vs registers
};

__device__ __forceinline__ void merge_state(float& m, float& l, float* acc, float m_o, float l_o,
                                            const float* acc_o, int n) {
  const float mn = fmaxf(m, m_o);
  const float a = (m == -INFINITY) ? 0.f : exp2f(m - mn);
  const float b = (m_o == -INFINITY) ? 0.f : exp2f(m_o - mn);
  l = l * a + l_o * b;
  for (int e = 0; e < n; ++e) acc[e] = acc[e] * a + acc_o[e] * b;
  m = mn;
}

#ifndef FC_DEC_MINB1
#define FC_DEC_MINB1 6
#endif
template <typename T, int D, int G>
__global__ void __launch_bounds__(kDecodeThreads, G == 1 ? FC_DEC_MINB1 : 1)
    decode_attn_kernel(const char* __restrict__ arena, const int32_t* __restrict__ table,
                       const Geom g, const __grid_constant__ DecodeBatch b,
                       const T* __restrict__ q, T* __restrict__ out, float scale_log2,
                       float* __restrict__ ws, int32_t* __restrict__ counters) {
  using C = DecodeCfg<T, D, G>;
  constexpr int kEPV = C::kEPV, kVpr = C::kVpr, kRows = C::kRows, kTile = C::kTile;
  __shared__ float s_part[kDecodeWarps][G][D + 2];
  __shared__ int s_last;

  // item -> (request, kv head, split)
  const int item = blockIdx.x;
  int lo = 0, hi = b.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (b.req[mid].item0 <= item) lo = mid; else hi = mid - 1;
  }
  const DecodeReq rq = b.req[lo];
  const int local = item - rq.item0;
  const int h = local / rq.nsplit, split = local % rq.nsplit;
  const int t_begin = split * b.split_tokens;
  const int t_end = min(rq.T, t_begin + b.split_tokens);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / kVpr, vec = lane % kVpr;
  const int hq0 = h * G;

  // query slice of this lane, pre-scaled into the exp2 domain
  float qf[G][kEPV];
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
    const uint4 raw = *reinterpret_cast<const uint4*>(q + ((int64_t)rq.q_row * b.Hq + hq0 + gi) * D +
                                                      vec * kEPV);
    unpack16<T>(raw, qf[gi]);
#pragma unroll
    for (int e = 0; e < kEPV; ++e) qf[gi][e] *= scale_log2;
  }
  float m[G], l[G], acc[G][kEPV];
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
    m[gi] = -INFINITY;
    l[gi] = 0.f;
#pragma unroll
    for (int e = 0; e < kEPV; ++e) acc[gi][e] = 0.f;
  }

  const int32_t* row_tab = table + (int64_t)rq.slot * g.max_bpr;
  const char* kbase = arena + g.seg_base(b.layer, 0, h) + vec * 16;
  const int64_t v_off = (int64_t)g.H * g.bs * g.row_bytes;
  constexpr int kTileTok = kTile * kRows;
  constexpr int kStride = kDecodeWarps * kTileTok;
  for (int t0 = t_begin + warp * kTileTok; t0 < t_end; t0 += kStride) {
    uint4 kr[kTile], vr[kTile];
#pragma unroll
    for (int u = 0; u < kTile; ++u) {
      const int t = t0 + u * kRows + sub;
      if (t < t_end) {
        const char* p = kbase + (int64_t)row_tab[t >> g.bs_shift] * g.block_stride +
                        (int64_t)(t & (g.bs - 1)) * g.row_bytes;
        kr[u] = ld_stream(p);
        vr[u] = ld_stream(p + v_off);
      }
    }
#pragma unroll
    for (int gi = 0; gi < G; ++gi) {
      float s[kTile];
      float tmax = -INFINITY;
#pragma unroll
      for (int u = 0; u < kTile; ++u) {
        float kf[kEPV];
        unpack16<T>(kr[u], kf);
        float d = 0.f;
#pragma unroll
        for (int e = 0; e < kEPV; ++e) d = fmaf(qf[gi][e], kf[e], d);
#pragma unroll
        for (int off = kVpr / 2; off > 0; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
        const int t = t0 + u * kRows + sub;
        s[u] = (t < t_end) ? d : -INFINITY;
        tmax = fmaxf(tmax, s[u]);
      }
      if (tmax == -INFINITY) continue;  // no live row for this lane group
      const float mn = fmaxf(m[gi], tmax);
      const float corr = (m[gi] == -INFINITY) ? 0.f : exp2f(m[gi] - mn);
      l[gi] *= corr;
#pragma unroll
      for (int e = 0; e < kEPV; ++e) acc[gi][e] *= corr;
#pragma unroll
      for (int u = 0; u < kTile; ++u) {
        if (s[u] == -INFINITY) continue;
        const float p = exp2f(s[u] - mn);
        l[gi] += p;
        float vf[kEPV];
        unpack16<T>(vr[u], vf);
#pragma unroll
        for (int e = 0; e < kEPV; ++e) acc[gi][e] = fmaf(p, vf[e], acc[gi][e]);
      }
      m[gi] = mn;
    }
  }
  // merge the kRows lane groups of the warp, then the warps through SMEM
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
#pragma unroll
    for (int off = kVpr; off < 32; off <<= 1) {
      const float m_o = __shfl_xor_sync(0xffffffffu, m[gi], off);
      const float l_o = __shfl_xor_sync(0xffffffffu, l[gi], off);
      float acc_o[kEPV];
#pragma unroll
      for (int e = 0; e < kEPV; ++e) acc_o[e] = __shfl_xor_sync(0xffffffffu, acc[gi][e], off);
      merge_state(m[gi], l[gi], acc[gi], m_o, l_o, acc_o, kEPV);
    }
    if (lane < kVpr) {
#pragma unroll
      for (int e = 0; e < kEPV; ++e) s_part[warp][gi][vec * kEPV + e] = acc[gi][e];
      if (lane == 0) {
        s_part[warp][gi][D] = m[gi];
        s_part[warp][gi][D + 1] = l[gi];
      }
    }
  }
  __syncthreads();
  // threads (gi, d) merge the warps; D*G <= 128*8 -> a few per thread
  float* part = ws + (int64_t)item * G * (D + 2);
  for (int x = threadIdx.x; x < G * D; x += kDecodeThreads) {
    const int gi = x / D, d = x % D;
    float mm = -INFINITY, ll = 0.f, aa = 0.f;
#pragma unroll
    for (int w = 0; w < kDecodeWarps; ++w)
      merge_state(mm, ll, &aa, s_part[w][gi][D], s_part[w][gi][D + 1], &s_part[w][gi][d], 1);
    if (rq.nsplit == 1) {
      out[((int64_t)rq.q_row * b.Hq + hq0 + gi) * D + d] = Elem<T>::from_f(ll > 0.f ? aa / ll : 0.f);
    } else {
      part[gi * (D + 2) + d] = aa;
      if (d == 0) {
        part[gi * (D + 2) + D] = mm;
        part[gi * (D + 2) + D + 1] = ll;
      }
    }
  }
  if (rq.nsplit == 1) return;
  // split-KV: the last CTA of this (request, kv head) merges every split
  __threadfence();
  __syncthreads();
  int32_t* ctr = counters + (int64_t)lo * g.H + h;
  if (threadIdx.x == 0) s_last = (atomicAdd(ctr, 1) == rq.nsplit - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const float* base = ws + (int64_t)(rq.item0 + h * rq.nsplit) * G * (D + 2);
  for (int x = threadIdx.x; x < G * D; x += kDecodeThreads) {
    const int gi = x / D, d = x % D;
    float mm = -INFINITY, ll = 0.f, aa = 0.f;
    for (int sp = 0; sp < rq.nsplit; ++sp) {
      const volatile float* pp = base + ((int64_t)sp * G + gi) * (D + 2);
      const float a_o = pp[d];
      merge_state(mm, ll, &aa, pp[D], pp[D + 1], &a_o, 1);
    }
    out[((int64_t)rq.q_row * b.Hq + hq0 + gi) * D + d] = Elem<T>::from_f(ll > 0.f ? aa / ll : 0.f);
  }
  if (threadIdx.x == 0) *ctr = 0;  // ready for the next launch
}

template <typename T, int D>
fc_status launch_decode_t(const Geom& g, const char* arena, const int32_t* table,
                          const DecodeBatch& b, int gq, const void* q, void* out, float scale_log2,
                          float* ws, int32_t* counters, cudaStream_t stream) {
  const dim3 grid((unsigned)b.items);
#define FC_DEC(G)                                                                              \
  decode_attn_kernel<T, D, G><<<grid, kDecodeThreads, 0, stream>>>(                           \
      arena, table, g, b, (const T*)q, (T*)out, scale_log2, ws, counters)
  switch (gq) {
    case 1: FC_DEC(1); break;
    case 2: FC_DEC(2); break;
    case 4: FC_DEC(4); break;
    case 8: FC_DEC(8); break;
    default: return set_error(FC_ERR_UNSUPPORTED, "decode attention: query heads per kv head must be 1, 2, 4 or 8");
  }
#undef FC_DEC
  note_launch();
  return cuda_check(cudaGetLastError(), "decode_attn_kernel");
}

fc_status launch_decode_attention(const Geom& g, int dtype, const char* arena, const int32_t* table,
                                  const DecodeBatch& b, int gq, const void* q, void* out,
                                  float scale_log2, float* ws, int32_t* counters,
                                  cudaStream_t stream) {
  if (b.items == 0) return FC_OK;
  switch (dtype) {
    case FC_F16:
      if (g.D == 128) return launch_decode_t<__half, 128>(g, arena, table, b, gq, q, out, scale_log2, ws, counters, stream);
      if (g.D == 64) return launch_decode_t<__half, 64>(g, arena, table, b, gq, q, out, scale_log2, ws, counters, stream);
      break;
    case FC_BF16:
      if (g.D == 128) return launch_decode_t<__nv_bfloat16, 128>(g, arena, table, b, gq, q, out, scale_log2, ws, counters, stream);
      if (g.D == 64) return launch_decode_t<__nv_bfloat16, 64>(g, arena, table, b, gq, q, out, scale_log2, ws, counters, stream);
      break;
    case FC_F32:
      if (g.D == 128) return launch_decode_t<float, 128>(g, arena, table, b, gq, q, out, scale_log2, ws, counters, stream);
      if (g.D == 64) return launch_decode_t<float, 64>(g, arena, table, b, gq, q, out, scale_log2, ws, counters, stream);
      break;
    default:
      break;
  }
  return set_error(FC_ERR_UNSUPPORTED, "decode attention needs f16/bf16/f32 and head_dim 64 or 128");
}

// ---------------------------------------------------------------------------
// one new token's K/V per request, one layer
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    write_decode_kv_kernel(char* __restrict__ arena, const int32_t* __restrict__ table, const Geom g,
                           const __grid_constant__ KVWriteBatch b, const char* __restrict__ k,
                           const char* __restrict__ v) {
  const KVWriteReq rq = b.req[blockIdx.y];
  const int vpr = (int)(g.row_bytes / 16);
  const int total = 2 * g.H * vpr;
  const int32_t* row_tab = table + (int64_t)rq.slot * g.max_bpr;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < total; x += gridDim.x * blockDim.x) {
    const int vec = x % vpr, h = (x / vpr) % g.H, kv = x / (vpr * g.H);
    const char* src = (kv ? v : k) + ((int64_t)rq.row * g.H + h) * g.row_bytes + vec * 16;
    char* dst = arena + g.seg_base(b.layer, kv, h) + (int64_t)row_tab[rq.pos >> g.bs_shift] * g.block_stride +
                (int64_t)(rq.pos & (g.bs - 1)) * g.row_bytes + vec * 16;
    st_stream(dst, ld_stream(src));
  }
}

fc_status launch_write_kv(const Geom& g, char* arena, const int32_t* table, const KVWriteBatch& b,
                          const void* k, const void* v, cudaStream_t stream) {
  const int total = 2 * g.H * (int)(g.row_bytes / 16);
  const int gx = (total + 255) / 256;
  write_decode_kv_kernel<<<dim3((unsigned)gx, (unsigned)b.n), 256, 0, stream>>>(
      arena, table, g, b, (const char*)k, (const char*)v);
  note_launch();
  return cuda_check(cudaGetLastError(), "write_decode_kv_kernel");
}

}  // namespace fc
