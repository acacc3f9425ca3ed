// fc_snapkv_tc.cu -- SnapKV scoring on the 5th-gen tensor cores (sm_100a).
//
// One CTA per (request, layer, kv-head) segment, 256 threads:
//
//   thread 0   TMA producer + MMA issuer: streams the segment's K tiles
//              (128 tokens x D, fp16/bf16) from its paged blocks into a
//              3-stage SMEM ring with cp.async.bulk.tensor (128-byte swizzle),
//              and issues tcgen05.mma  S[tile] = K_tile . Q_win^T  (M=128
//              tokens, N=w queries, K=D) into TMEM columns [tile*w, tile*w+w).
//              The whole segment's window logits stay resident in TMEM
//              (ceil(T/128)*w <= 512 columns, i.e. T <= 2048 at w = 32).
//   all warps  epilogue from TMEM (tcgen05.ld 32x32b): per-query max, then
//              sum of exp, then s'_t = mean_j softmax_j(t); avg-pool, window
//              forced keep; then the shared segmented top-k and in-place
//              compaction (fc_select.cuh).
//
// K is read from HBM exactly once; scores never leave the SM. Precision:
// fp16/bf16 products are exact in fp32, only the fp32 accumulation order
// differs from the oracle (scores within 1e-5 relative, tests/test_gpu_press.py).
// Reference anchors: SURVEY.md Appendix A (kvpress SnapKV restated), K_r from
// the reference ceil rule (kv.py:169-194).
#include <cudaTypedefs.h>

#include <cfloat>
#include <cstring>
#include <mutex>

#include "fc_select.cuh"
#include "fc_tc.cuh"

namespace fc {

constexpr int kTcStages = 3;
constexpr int kTileM = 128;

struct TcSmem {
  int D, w, bs, max_T;
  int tile_bytes, q_bytes;
  int off_stage, off_q, off_tab, off_sc, off_s1, off_bar, total;
};

__host__ __device__ inline TcSmem tc_smem_plan(int D, int w, int bs, int max_T) {
  TcSmem p;
  p.D = D;
  p.w = w;
  p.bs = bs;
  p.max_T = max_T;
  p.tile_bytes = kTileM * D * 2;
  p.q_bytes = w * D * 2;
  p.off_stage = 0;                                            // 1024-aligned base
  p.off_q = p.off_stage + kTcStages * p.tile_bytes;
  p.off_tab = p.off_q + ((p.q_bytes + 1023) & ~1023);
  const int nb = (max_T + bs - 1) / bs;
  // Scores (sc) and window means (s1) live in the K stage ring: they are only
  // written after the last MMA has consumed the last stage (mma_done).
  p.off_sc = p.off_stage;
  p.off_s1 = p.off_sc + ((max_T * 4 + 15) & ~15);
  p.off_bar = p.off_tab + ((nb * 4 + 15) & ~15);
  p.total = p.off_bar + 16 * 8 + 1024;                        // barriers + alignment slack
  return p;
}

template <typename T, int D>
__global__ void __launch_bounds__(kThreads, 2)
    snapkv_tc_kernel(char* __restrict__ arena, const int32_t* __restrict__ table, const Geom g,
                     const __grid_constant__ PressBatch b, const PressParams pp,
                     const __grid_constant__ CUtensorMap kmap,
                     const __grid_constant__ CUtensorMap qmap, const fc_press_outputs out) {
  constexpr int kHalves = D / 64;              // 128-byte K-dim slabs
  constexpr int kKSteps = D / 16;              // UMMA_K = 16 for 16-bit inputs
  constexpr int kFmt = sizeof(T) == 2 && Elem<T>::kDtype == FC_BF16 ? 1 : 0;
  extern __shared__ unsigned char smem_raw[];
  __shared__ SelectScratch ss;
  __shared__ uint32_t s_tmem;
  __shared__ float s_red[kWarps][32];
  __shared__ float s_m[32], s_zinv[32];

  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int w = pp.window;
  const TcSmem plan = tc_smem_plan(D, w, g.bs, b.max_T);
  unsigned char* stages = smem + plan.off_stage;
  unsigned char* qs = smem + plan.off_q;
  int32_t* s_tab = reinterpret_cast<int32_t*>(smem + plan.off_tab);
  float* sc = reinterpret_cast<float*>(smem + plan.off_sc);
  float* s1 = reinterpret_cast<float*>(smem + plan.off_s1);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + plan.off_bar);
  uint64_t* full = bars;                 // [kTcStages]
  uint64_t* empty = bars + kTcStages;    // [kTcStages]
  uint64_t* q_full = bars + 2 * kTcStages;
  uint64_t* mma_done = q_full + 1;

  const int LH = g.L * g.H;
  const int r = blockIdx.x / LH, lh = blockIdx.x % LH;
  const int l = lh / g.H, h = lh % g.H;
  const PressReq q = b.req[r];
  const int T_len = q.T, K = q.K;
  const int nb = (T_len + g.bs - 1) / g.bs;
  const int ntiles = (T_len + kTileM - 1) / kTileM;
  uint32_t ncols = 32;
  while (ncols < (uint32_t)(ntiles * w)) ncols <<= 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  for (int i = threadIdx.x; i < nb; i += kThreads) s_tab[i] = table[(int64_t)q.slot * g.max_bpr + i];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2 * kTcStages + 2; ++i) tc::mbar_init(&bars[i], 1);
    tc::fence_barrier_init();
    ss.first_drop = INT_MAX;
    tc::tma_prefetch_desc(&kmap);
    tc::tma_prefetch_desc(&qmap);
  }
  if (warp == 1) tc::tmem_alloc(&s_tmem, ncols);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = s_tmem;

  // ---- producer + MMA issuer (one thread) ----
  if (threadIdx.x == 0) {
    const int chunks = kTileM / g.bs;
    const int64_t row_l = (int64_t)l * g.num_blocks * 2 * g.H * g.bs + (int64_t)h * g.bs;
    auto issue_tile = [&](int k, int st) {
      int n_chunks = min(chunks, nb - k * chunks);
      tc::mbar_expect_tx(&full[st], (uint32_t)(n_chunks * g.bs * D * 2));
      unsigned char* dst = stages + st * plan.tile_bytes;
      for (int c = 0; c < n_chunks; ++c) {
        const int64_t row0 = row_l + (int64_t)s_tab[k * chunks + c] * 2 * g.H * g.bs;
#pragma unroll
        for (int hf = 0; hf < kHalves; ++hf)
          tc::tma_load_2d(dst + hf * kTileM * 128 + c * g.bs * 128, &kmap, &full[st], hf * 64,
                          (int)row0);
      }
    };
    // window queries of this (request, layer, kv-head): rows [qrow, qrow + w)
    const int qrow = (int)(((int64_t)q.q_idx * g.L + l) * pp.num_q_heads + h) * w;
    tc::mbar_expect_tx(q_full, (uint32_t)(w * D * 2));
#pragma unroll
    for (int hf = 0; hf < kHalves; ++hf) tc::tma_load_2d(qs + hf * w * 128, &qmap, q_full, hf * 64, qrow);
    for (int k = 0; k < min(kTcStages, ntiles); ++k) issue_tile(k, k);
    tc::mbar_wait(q_full, 0);
    const uint32_t idesc = tc::idesc_f16(kFmt, kTileM, w);
    const uint32_t q_base = tc::smem_u32(qs);
    for (int k = 0; k < ntiles; ++k) {
      const int st = k % kTcStages;
      const uint32_t ph = (uint32_t)(k / kTcStages) & 1u;
      tc::mbar_wait(&full[st], ph);
      tc::fence_after_sync();
      const uint32_t a_base = tc::smem_u32(stages + st * plan.tile_bytes);
#pragma unroll
      for (int kk = 0; kk < kKSteps; ++kk) {
        const uint32_t koff = (uint32_t)((kk & 3) * 32);
        const uint64_t ad = tc::desc_k_sw128(a_base + (kk >> 2) * kTileM * 128 + koff);
        const uint64_t bd = tc::desc_k_sw128(q_base + (kk >> 2) * w * 128 + koff);
        tc::mma_f16(tmem + (uint32_t)(k * w), ad, bd, idesc, kk > 0 ? 1u : 0u);
      }
      tc::mma_commit(&empty[st]);
      if (k + kTcStages < ntiles) {
        tc::mbar_wait(&empty[st], ph);
        issue_tile(k + kTcStages, st);
      }
    }
    tc::mma_commit(mma_done);
  }
  __syncwarp();
  tc::mbar_wait(mma_done, 0);
  tc::fence_after_sync();

  // ---- epilogue: softmax over all T per window query, from TMEM ----
  const float inv_sqrt_d = 1.0f / sqrtf((float)D);
  const int quarter = warp & 3, parity = warp >> 2;
  const int row = quarter * 32 + lane;
  const uint32_t lane_addr = tmem + ((uint32_t)(quarter * 32) << 16);
  const int n_keep = T_len - w;
  float acc[32];
  // pass 1: per-query max
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] = -INFINITY;
  for (int k = parity; k < ntiles; k += 2) {
    float v[32];
    tc::tmem_ld_32x32b_x32(lane_addr + (uint32_t)(k * w), v);
    const int t = k * kTileM + row;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const bool ok = j < w && t < T_len && t <= T_len - w + j;
      if (ok) acc[j] = fmaxf(acc[j], v[j] * inv_sqrt_d);
    }
  }
#pragma unroll
  for (int j = 0; j < 32; ++j)
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc[j] = fmaxf(acc[j], __shfl_xor_sync(0xffffffffu, acc[j], off));
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (lane == j) s_red[warp][j] = acc[j];
  __syncthreads();
  if (threadIdx.x < 32) {
    float m = s_red[0][threadIdx.x];
    for (int i = 1; i < kWarps; ++i) m = fmaxf(m, s_red[i][threadIdx.x]);
    s_m[threadIdx.x] = m;
  }
  __syncthreads();
  float mj[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) mj[j] = s_m[j];
  // pass 2: per-query sum of exp
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] = 0.f;
  for (int k = parity; k < ntiles; k += 2) {
    float v[32];
    tc::tmem_ld_32x32b_x32(lane_addr + (uint32_t)(k * w), v);
    const int t = k * kTileM + row;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const bool ok = j < w && t < T_len && t <= T_len - w + j;
      if (ok) acc[j] += expf(v[j] * inv_sqrt_d - mj[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < 32; ++j)
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], off);
#pragma unroll
  for (int j = 0; j < 32; ++j)
    if (lane == j) s_red[warp][j] = acc[j];
  __syncthreads();
  if (threadIdx.x < 32) {
    float z = 0.f;
    for (int i = 0; i < kWarps; ++i) z += s_red[i][threadIdx.x];
    s_zinv[threadIdx.x] = 1.0f / z;
  }
  __syncthreads();
  float zj[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) zj[j] = s_zinv[j];
  // pass 3: s'_t = mean over the window of the normalised probabilities
  for (int k = parity; k < ntiles; k += 2) {
    float v[32];
    tc::tmem_ld_32x32b_x32(lane_addr + (uint32_t)(k * w), v);
    const int t = k * kTileM + row;
    if (t < n_keep) {
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < w && t <= T_len - w + j) s += expf(v[j] * inv_sqrt_d - mj[j]) * zj[j];
      s1[t] = s / (float)w;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, ncols);

  // ---- avg-pool (zero pad), forced window, then the shared select + compact ----
  const int half = pp.pool_kernel / 2;
  for (int t = threadIdx.x; t < T_len; t += kThreads) {
    float v = INFINITY;
    if (t < n_keep) {
      float a = 0.f;
      for (int o = -half; o <= half; ++o) {
        const int u = t + o;
        a += (u >= 0 && u < n_keep) ? s1[u] : 0.f;
      }
      v = a / (float)pp.pool_kernel;
    }
    sc[t] = v;
  }
  __syncthreads();
  if (out.scores) {
    float* so = out.scores + q.score_off + (int64_t)lh * T_len;
    for (int t = threadIdx.x; t < T_len; t += kThreads) so[t] = sc[t];
  }
  uint32_t* keys = reinterpret_cast<uint32_t*>(sc);
  for (int t = threadIdx.x; t < T_len; t += kThreads) keys[t] = float_key(sc[t]);
  __syncthreads();
  int32_t* idx = reinterpret_cast<int32_t*>(sc);
  if (b.per_segment && q.seg0 < T_len) {
    select_emit(keys, q.seg0, q.K0, idx, 0, 0, ss);
    select_emit(keys + q.seg0, T_len - q.seg0, K - q.K0, idx, q.K0, q.seg0, ss);
  } else {
    select_emit(keys, T_len, K, idx, 0, 0, ss);
  }
  if (out.kept_idx) {
    int32_t* ko = out.kept_idx + q.kept_off + (int64_t)lh * K;
    for (int j = threadIdx.x; j < K; j += kThreads) ko[j] = idx[j];
  }
  char* seg = arena + g.seg_base(l, 0, h);
  compact_rows<D * (int)sizeof(T)>(seg, g, s_tab, s_tab, idx, K, min(ss.first_drop, K));
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

static fc_status encode_rows(CUtensorMap* map, const void* base, int dtype, int D, uint64_t rows,
                             int box_rows) {
  auto enc = get_encode();
  if (!enc) return set_error(FC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, dtype == FC_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                   2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(FC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return FC_OK;
}

bool snapkv_tc_supported(const Geom& g, int dtype, const PressParams& pp, int max_T) {
  static const bool forced_simt = [] {
    const char* e = getenv("FASTCACHE_SNAPKV_SIMT");
    return e && e[0] == '1';
  }();
  if (forced_simt) return false;
  if (dtype != FC_F16 && dtype != FC_BF16) return false;
  if (g.D != 64 && g.D != 128) return false;
  if (pp.num_q_heads != g.H) return false;          // one query head per kv head
  if (pp.window != 32) return false;               // one 32x32b.x32 TMEM load per tile
  if (g.bs < 8 || g.bs > 128) return false;
  if ((max_T + kTileM - 1) / kTileM * pp.window > 512) return false;
  return true;
}

fc_status launch_snapkv_tc(const Geom& g, int dtype, char* arena, const int32_t* table,
                           const PressBatch& b, const PressParams& pp, const fc_press_inputs& in,
                           const fc_press_outputs& out, cudaStream_t stream) {
  const int n_requests_total = b.n_total;
  CUtensorMap kmap, qmap;
  const uint64_t rows = (uint64_t)g.L * g.num_blocks * 2 * g.H * g.bs;
  fc_status st = encode_rows(&kmap, arena, dtype, g.D, rows, g.bs);
  if (st != FC_OK) return st;
  st = encode_rows(&qmap, in.q_window, dtype, g.D,
                   (uint64_t)n_requests_total * g.L * pp.num_q_heads * pp.window, pp.window);
  if (st != FC_OK) return st;
  const TcSmem plan = tc_smem_plan(g.D, pp.window, g.bs, b.max_T);
  const int n_items = b.n * g.L * g.H;
  auto launch = [&](auto kern) -> fc_status {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, plan.total);
    if (e != cudaSuccess) return cuda_check(e, "cudaFuncSetAttribute(snapkv_tc)");
    kern<<<n_items, kThreads, plan.total, stream>>>(arena, table, g, b, pp, kmap, qmap, out);
    note_launch();
    return cuda_check(cudaGetLastError(), "snapkv_tc_kernel");
  };
  if (dtype == FC_BF16)
    return g.D == 64 ? launch(snapkv_tc_kernel<__nv_bfloat16, 64>) : launch(snapkv_tc_kernel<__nv_bfloat16, 128>);
  return g.D == 64 ? launch(snapkv_tc_kernel<__half, 64>) : launch(snapkv_tc_kernel<__half, 128>);
}

}  // namespace fc
