/*
 * fastcache.h -- C ABI of the B200-native FastCache compression-stage hot path.
 *
 * One opaque fc_pool per (process, GPU) owns a paged KV arena in HBM, the
 * device-resident block tables and free-list stack, and a host mirror of the
 * reference's byte accounting. Every entry point is a plain C function with
 * POD arguments; no C++ exception and no torch type crosses it. All device
 * work is stream-ordered on the caller's cudaStream_t (passed as void*; NULL
 * means the legacy default stream). A pool is NOT thread-safe: the caller
 * serialises calls, as the reference's single-writer engine does
 * (engine.py:563-575).
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/kvservesim):
 *   fc_pool_create          <- KVCachePool.__init__            pool.py:95-117
 *   fc_pool_alloc_batch     <- KVCachePool.allocate            pool.py:147-165  (batched)
 *   fc_pool_compress_batch  <- compressed_spec + KVCachePool.transition_compressed
 *                              kv.py:173-194, pool.py:167-192; driven per batch from
 *                              Simulator._on_stage_complete(COMPRESS) engine.py:501-510
 *   fc_pool_compress_host_batch <- same as fc_pool_compress_batch, raw KV still in pinned
 *                              host memory (the P.Store -> compress hand-off)
 *   fc_pool_append          <- KVCachePool.append_decode_tokens pool.py:194-211
 *   fc_pool_write_kv / fc_pool_decode_attention <- the decode stage over compressed
 *                              caches (engine.py:514-548 drives append_decode_tokens per
 *                              step; UpdateKVCache PAPER.md:255-261)
 *   fc_pool_release_batch   <- KVCachePool.release             pool.py:213-224  (batched)
 *   fc_pool_get_stats       <- KVCachePool.stats / verify_conservation pool.py:228-257
 *   fc_compress_tensor      <- compress_tensor                 kv.py:211-239
 *   fc_synth_fill           <- (bench input generator; stands in for P.Store(M.Prefill)
 *                              PAPER.md:246)
 *   fc_pool_store_tokens    <- P.Store (prefill KV ingest)
 *   fc_pool_write_prefill_kv <- P.Store per layer, batched varlen (the prefill's KV writes)
 *
 * Error convention (pool.py:31-47, kv.py:34-43): functions return fc_status;
 * FC_ERR_CAPACITY fills (requested, available) out-params; fc_last_error()
 * returns a thread-local message for the last failing call.
 */
#ifndef FASTCACHE_H_
#define FASTCACHE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FC_ABI_VERSION 1

#if defined(__GNUC__)
#define FC_API __attribute__((visibility("default")))
#else
#define FC_API
#endif

typedef enum fc_status {
  FC_OK = 0,
  FC_ERR_CAPACITY = 1,      /* kvservesim.pool.CapacityExceeded  pool.py:31-39 */
  FC_ERR_INVALID_STATE = 2, /* kvservesim.pool.InvalidState      pool.py:42-43 */
  FC_ERR_DOUBLE_FREE = 3,   /* kvservesim.pool.DoubleFree        pool.py:46-47 */
  FC_ERR_INVALID_ARG = 4,   /* ValueError                                      */
  FC_ERR_CUDA = 5,          /* CUDA runtime error                              */
  FC_ERR_DEVICE = 6,        /* a kernel raised the pool's device error word    */
  FC_ERR_UNSUPPORTED = 7,   /* shape/dtype without a compiled kernel           */
  FC_ERR_ALREADY_COMPRESSED = 8, /* kvservesim.kv.AlreadyCompressed kv.py:34-35 */
  FC_ERR_EMPTY_INPUT = 9    /* kvservesim.kv.EmptyInput kv.py:38-39            */
} fc_status;

typedef enum fc_dtype { FC_F16 = 0, FC_BF16 = 1, FC_F32 = 2, FC_U8 = 3, FC_F64 = 4 } fc_dtype;

typedef enum fc_pool_mode { FC_POOLED = 0, FC_LEGACY_ZOMBIE = 1 } fc_pool_mode; /* pool.py:26-28 */

typedef enum fc_press_kind {
  FC_PRESS_KNORM = 0,
  FC_PRESS_SNAPKV = 1,
  FC_PRESS_EXPECTED_ATTENTION = 2,
  FC_PRESS_MEANPOOL = 3,     /* MapKind.MEAN_POOL     kv.py:227-231 */
  FC_PRESS_SEEDEDLINEAR = 4  /* MapKind.SEEDED_LINEAR kv.py:232-239 */
} fc_press_kind;

typedef enum fc_synth_dist { FC_SYNTH_SCALED = 0, FC_SYNTH_PLAIN = 1 } fc_synth_dist;

/* ModelConfig (kv.py:51-76) + the element type the kernels interpret. */
typedef struct fc_model_config {
  int32_t num_layers;
  int32_t num_kv_heads;
  int32_t head_dim;
  int32_t bytes_per_element; /* 1, 2 or 4 */
  int32_t dtype;             /* fc_dtype; must agree with bytes_per_element */
} fc_model_config;

typedef struct fc_pool_options {
  int32_t block_size;            /* tokens per block (all layers/heads/K|V), default 16 */
  int32_t max_handles;           /* live handles the device block tables hold           */
  int32_t max_blocks_per_handle; /* block-table row length                              */
  int32_t mode;                  /* fc_pool_mode                                        */
  int64_t num_blocks;            /* 0 = capacity/block_bytes + max_handles              */
  void* arena;                   /* optional caller-owned device arena (NULL = cudaMalloc) */
  uint64_t arena_bytes;          /* size of `arena` when given                          */
  int32_t device;                /* CUDA device ordinal                                 */
  int32_t reserved;
} fc_pool_options;

/* Press configuration (CompressorSpec kv.py:134-144, extended). */
typedef struct fc_press_config {
  int32_t kind;        /* fc_press_kind                                   */
  int32_t factor;      /* k >= 1; K_r = sum_seg ceil(n_seg / k) (kv.py:188) */
  int32_t window;      /* SnapKV observation window w                     */
  int32_t pool_kernel; /* SnapKV avg-pool kernel (odd)                    */
  int32_t n_sink;      /* ExpectedAttention sinks                         */
  int32_t num_q_heads; /* Hq = g * Hkv (SnapKV / EA query heads)          */
  int32_t per_segment; /* 1: top-ceil(n_seg/k) per modality segment       */
  int32_t reserved;
  const double* chunk_weights; /* SEEDEDLINEAR: `factor` host weights (kv.py:197-208) */
} fc_press_config;

/* Device-resident per-request press inputs, row-major, request order = batch order. */
typedef struct fc_press_inputs {
  const void* q_window; /* SnapKV: [n][L][Hq][w][D] in the pool dtype            */
  const float* mean_q;  /* EA:     [n][L][Hq][D] fp32                              */
  const float* cov_q;   /* EA:     [n][L][Hq][D][D] fp32                           */
} fc_press_inputs;

/* Optional device outputs of fc_pool_compress_batch (NULL to skip). Request r's
 * region starts at the prefix sum over earlier requests, laid out [L][Hkv][...]. */
typedef struct fc_press_outputs {
  int32_t* kept_idx; /* [sum_r K_r * L * Hkv]: kept source positions, ascending */
  float* scores;     /* [sum_r T_r * L * Hkv]: press scores (+inf = forced keep) */
} fc_press_outputs;

typedef struct fc_pool_stats {
  uint64_t current_bytes;          /* PoolStats pool.py:63-70 */
  uint64_t peak_bytes;
  uint64_t capacity_bytes;
  int64_t live_handles;
  uint64_t zombie_bytes_reclaimed;
  int64_t allocation_count;
  int64_t num_blocks;              /* device arena */
  int64_t free_blocks;
  int64_t used_blocks;
  uint64_t block_bytes;
  uint64_t live_token_bytes;       /* sum over live handles of kv_bytes(tokens) */
  double fragmentation;            /* 1 - live_token_bytes / (used_blocks * block_bytes) */
  int32_t device_error;            /* device error word (0 = clean) */
  int32_t reserved;
} fc_pool_stats;

typedef struct fc_pool fc_pool;

/* --- library --------------------------------------------------------------- */
FC_API int32_t fc_abi_version(void);
FC_API const char* fc_last_error(void);
/* Number of kernel launches this thread issued through the library so far. */
FC_API int64_t fc_launch_count(void);

/* --- pool lifecycle ---------------------------------------------------------- */
FC_API fc_status fc_pool_create(const fc_model_config* cfg, uint64_t capacity_bytes,
                         const fc_pool_options* opts, fc_pool** out);
FC_API fc_status fc_pool_destroy(fc_pool* pool);
FC_API fc_status fc_pool_arena(fc_pool* pool, void** dev_ptr, uint64_t* bytes, int64_t* num_blocks,
                        uint64_t* block_bytes);

/* --- pool operations --------------------------------------------------------- */
/* Admit n raw caches (strict: each needs kv_bytes(tokens) <= available at its
 * turn, pool.py:147-165). Pops ceil(tokens/bs) blocks per request from the
 * device free stack in batch order. On FC_ERR_CAPACITY the first failing
 * request's (requested, available) are written and nothing is admitted. */
FC_API fc_status fc_pool_alloc_batch(fc_pool* pool, int32_t n, const int64_t* request_ids,
                              const int64_t* tokens, int64_t* handle_ids_out,
                              uint64_t* requested_out, uint64_t* available_out, void* stream);

/* Compress n RAW handles in one batched pass and transition them to
 * COMPRESSED in batch order (pool.py:167-192). seg_tokens[2*i + s] = the raw
 * token count of modality segment s (image, text; 0 = absent) of request i,
 * which must sum to the handle's tokens. K_r = sum_s ceil(seg/k). Pooled
 * mode compacts in place and frees tail blocks in the same stream step;
 * legacy mode writes into freshly popped blocks and retains the raw ones. */
FC_API fc_status fc_pool_compress_batch(fc_pool* pool, int32_t n, const int64_t* handle_ids,
                                 const int64_t* seg_tokens, const fc_press_config* press,
                                 const fc_press_inputs* inputs, const fc_press_outputs* outputs,
                                 uint64_t* requested_out, uint64_t* available_out, void* stream);

/* fc_pool_compress_batch for raw KV that is still in pinned host memory:
 * host_kv[i] is request i's dense [L][2][Hkv][T_i][D] buffer in the pool
 * dtype (cudaHostAlloc / torch pin_memory; it must stay valid until the
 * stream reaches this call's work). Pooled Knorm / SnapKV move only the K
 * planes (DMA, double-buffered through pool-owned staging) and, after
 * selection, the kept V rows (zero-copy gather): 0.5 R + 0.5 C bytes over
 * PCIe instead of R. Other presses and legacy mode copy all of K and V. The
 * handles' raw blocks receive the payload; the result equals
 * fc_pool_store_tokens of every request followed by fc_pool_compress_batch. */
FC_API fc_status fc_pool_compress_host_batch(fc_pool* pool, int32_t n, const int64_t* handle_ids,
                                      const int64_t* seg_tokens, const fc_press_config* press,
                                      const fc_press_inputs* inputs,
                                      const fc_press_outputs* outputs, const void* const* host_kv,
                                      uint64_t* requested_out, uint64_t* available_out,
                                      void* stream);

/* Grow n COMPRESSED handles by tokens[i] decode tokens (pool.py:194-211). */
FC_API fc_status fc_pool_append(fc_pool* pool, int32_t n, const int64_t* handle_ids,
                         const int64_t* tokens, uint64_t* requested_out, uint64_t* available_out,
                         void* stream);

/* P.Store: one layer of the prefill's K and V for n handles in
 * the varlen layout k, v = [cu_seqlens[n]][Hkv][D] (pool dtype, device):
 * rows cu_seqlens[i] .. cu_seqlens[i+1]-1 (host array, cu_seqlens[0] = 0) go
 * to tokens tok_begin[i] + j of handle i (tok_begin NULL = 0). Chunked
 * prefill calls it once per chunk with the chunk's token offsets. */
FC_API fc_status fc_pool_write_prefill_kv(fc_pool* pool, int32_t layer, int32_t n,
                                   const int64_t* handle_ids, const int64_t* cu_seqlens,
                                   const int64_t* tok_begin, const void* k, const void* v,
                                   void* stream);

/* Decode over the compacted blocks, one layer at a time. fc_pool_write_kv
 * writes one token's K and V per handle (k, v: [n][Hkv][D], pool dtype) at
 * positions[i] (NULL: the handle's last token, i.e. the slot fc_pool_append
 * just added). fc_pool_decode_attention computes, for each handle i and query
 * head j, softmax(scale * q_ij . K^T) V over the handle's live tokens in
 * layer `layer` (q, out: [n][num_q_heads][D], pool dtype; scale <= 0 means
 * 1/sqrt(D); fp32 accumulation). */
FC_API fc_status fc_pool_write_kv(fc_pool* pool, int32_t layer, int32_t n, const int64_t* handle_ids,
                           const int64_t* positions, const void* k, const void* v, void* stream);
FC_API fc_status fc_pool_decode_attention(fc_pool* pool, int32_t layer, int32_t n,
                                   const int64_t* handle_ids, int32_t num_q_heads, float scale,
                                   const void* q, void* out, void* stream);

/* Release n handles, pushing their blocks (request order, ascending logical
 * block) onto the device free stack (pool.py:213-224). */
FC_API fc_status fc_pool_release_batch(fc_pool* pool, int32_t n, const int64_t* handle_ids,
                                void* stream);

/* Synchronising: waits for the pool's device work and reads the error word. */
FC_API fc_status fc_pool_get_stats(fc_pool* pool, fc_pool_stats* out);
FC_API fc_status fc_pool_synchronize(fc_pool* pool);

/* Kernel timing (CUDA events recorded on the launch stream around the press
 * kernels and the tail-free step of each fc_pool_compress_batch call). */
typedef struct fc_profile {
  double press_ms;       /* press kernel(s): score + top-k + compaction          */
  double free_ms;        /* tail-block push kernel                               */
  double total_ms;       /* whole device span of the call                        */
  int64_t press_launches;
  int64_t total_launches;
} fc_profile;
FC_API fc_status fc_pool_set_profiling(fc_pool* pool, int32_t enable);
/* Synchronising: timings of the most recent compress call. */
FC_API fc_status fc_pool_last_profile(fc_pool* pool, fc_profile* out);

/* Press launches of the most recent compress call per implementation:
 * out[0] tensor-core (tcgen05/TMA/TMEM) kernels, out[1] SIMT press kernels,
 * out[2] chunk-fold (MEAN_POOL / SEEDED_LINEAR) kernels. Not synchronising. */
FC_API fc_status fc_pool_last_paths(fc_pool* pool, int64_t out[3]);

/* Kernel of the most recent fc_pool_write_prefill call: *tma = 1 the TMA ingest
 * (head-group tiles, whole-chunk bulk stores), 0 the register-copy kernel (chunks above
 * the 16-KB tile), -1 no prefill written yet. Not synchronising. */
FC_API fc_status fc_pool_last_prefill_path(fc_pool* pool, int32_t* tma);

/* Device pointer of a handle's block-table row and its live block count. */
FC_API fc_status fc_pool_block_table(fc_pool* pool, int64_t handle_id, const int32_t** dev_row,
                              int32_t* n_blocks, int64_t* n_tokens);

/* --- payload movement -------------------------------------------------------- */
/* Copy tokens [tok_begin, tok_begin + n_tok) of a handle between a dense device
 * buffer laid out [L][2][Hkv][n_tok][D] and the handle's blocks. */
FC_API fc_status fc_pool_store_tokens(fc_pool* pool, int64_t handle_id, int64_t tok_begin,
                               int64_t n_tok, const void* src, void* stream);
FC_API fc_status fc_pool_load_tokens(fc_pool* pool, int64_t handle_id, int64_t tok_begin,
                              int64_t n_tok, void* dst, void* stream);

/* Deterministic counter-based KV generator (K8) writing every token of n
 * handles. keys[i] is request i's generator key (the oracle regenerates any
 * element from (seed, key, layer, kv, head, pos, dim)). */
FC_API fc_status fc_synth_fill(fc_pool* pool, int32_t n, const int64_t* handle_ids, const int64_t* keys,
                        uint64_t seed, int32_t dist, void* stream);

/* Reference compress_tensor (kv.py:211-239) on a dense device (n, d) matrix:
 * MEANPOOL writes ceil(n/k) rows in the input dtype; SEEDEDLINEAR writes fp64. */
FC_API fc_status fc_compress_tensor(const void* src, int64_t n, int64_t d, int32_t dtype,
                             const fc_press_config* press, void* dst, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FASTCACHE_H_ */
