/* hisa_cuda.h — C ABI of the B200 (sm_100a) hierarchical-indexer library.
 *
 * This is the drop-in boundary for the reference's indexer hot path (reference tree: proj/core, headers
 * only).  The reference has no FFI of its own; each entry point below names the reference C++ interface
 * it replaces, batched over all query rows because a per-row device call is meaningless:
 *
 *   hisa_cuda_upload_keys / _pool_build / _pool_append / _pool_read / _pool_set
 *        <- hisa::build_block_summaries, BlockSummaryCache::append / pooled / count
 *           (proj/core/include/hisa/block_summary.hpp:23-59)
 *   hisa_cuda_score_blocks       <- hisa::score_blocks      (hisa/hisa.hpp:16-21)
 *   hisa_cuda_select_blocks      <- hisa::select_blocks     (hisa/hisa.hpp:23-28)
 *   hisa_cuda_score_tokens       <- hisa::score_tokens      (hisa/dsa.hpp:13-20)
 *   hisa_cuda_top_k              <- hisa::top_k_tokens      (hisa/dsa.hpp:22-27)
 *   hisa_cuda_hisa_select        <- hisa::hisa_select       (hisa/hisa.hpp:35-45) incl. candidate_union (:30-33)
 *   hisa_cuda_dsa_select         <- hisa::dsa_select        (hisa/dsa.hpp:29-32)
 *   hisa_cuda_block_sparse_select<- hisa::block_sparse_select (hisa/block_sparse.hpp:12-19)
 *   hisa_cuda_attn_set_latents   <- hisa::AttentionInputs   (hisa/attention.hpp:16-46), latent_states part
 *   hisa_cuda_sparse_attend      <- hisa::sparse_attend     (hisa/attention.hpp:48-56), the step after the path
 *   hisa_cuda_dense_attend       <- hisa::dense_attend      (hisa/attention.hpp:58-59)
 *   hisa_cuda_config             <- hisa::HisaConfig        (hisa/config.hpp:26-67), POD mirror
 *   status codes                 <- the exception leaves of hisa/errors.hpp:10-28
 *
 * Conventions
 *   - plain pointers and sizes only; no C++ or torch types cross this boundary.
 *   - data pointers may be HOST or DEVICE memory (detected with cudaPointerGetAttributes); host buffers
 *     are copied inside the call (pinned memory from hisa_cuda_host_alloc makes those copies asynchronous).
 *   - nothing throws: every function returns a hisa_status; hisa_cuda_last_error gives the message.
 *   - there is NO CPU fallback: without a usable sm_100 device hisa_cuda_create fails with
 *     HISA_ERR_NO_DEVICE and nothing else can be called.
 *   - a context is bound to one device and one stream and is not thread-safe; use one per GPU.
 *   - selection output is a fixed int32 [Q, token_budget] matrix: the first out_count[row] entries of a
 *     row are the selected token positions in ascending order, the rest is padded with -1.
 */
#ifndef HISA_CUDA_H_
#define HISA_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HISA_CUDA_ABI_VERSION 1

typedef struct hisa_cuda_ctx hisa_cuda_ctx;

typedef enum hisa_status {
  HISA_OK = 0,
  HISA_ERR_INFEASIBLE_CONFIG = 1,  /* hisa::InfeasibleConfig */
  HISA_ERR_CAUSAL_VIOLATION = 2,   /* hisa::CausalViolation */
  HISA_ERR_EMPTY_SEQUENCE = 3,     /* hisa::EmptySequence */
  HISA_ERR_DIMENSION_MISMATCH = 4, /* hisa::DimensionMismatch */
  HISA_ERR_NON_FINITE = 5,         /* hisa::NonFiniteValue */
  HISA_ERR_SHAPE_MISMATCH = 6,     /* hisa::ShapeMismatch */
  HISA_ERR_EMPTY_SELECTION = 7,    /* hisa::EmptySelection */
  HISA_ERR_INVALID_ARGUMENT = 8,
  HISA_ERR_UNSUPPORTED = 9,        /* shape outside what the sm_100a kernels cover (H > 64, d > 128, ...) */
  HISA_ERR_NO_DEVICE = 10,         /* no CUDA device / not sm_100: there is no CPU fallback */
  HISA_ERR_CUDA = 11,              /* a CUDA runtime/driver call failed; message has the detail */
  HISA_ERR_OUT_OF_MEMORY = 12
} hisa_status;

typedef enum hisa_dtype {
  HISA_DTYPE_F32 = 0,  /* float32 storage; scored with exact 3-way bf16 splits (fp32-grade products) */
  HISA_DTYPE_BF16 = 1, /* bfloat16 storage, the production format */
  /* e4m3 bytes for queries and keys (DeepSeek-V3.2 indexer format), num_heads = 64 and dim = 128 only.
   * A key is float(k8[s, :]) * key_scale[s] (hisa_cuda_upload_keys_scaled / _pool_append_scaled; scale > 0).
   * The per-(query, head) scale of q is folded into `gates` by the caller: gate[t, j] = w[t, j] * q_scale[t, j],
   * which is exact because a positive scale commutes with the ReLU of Eq.1 (hisa/dsa.hpp:13-20).
   * Token scores are computed by the e4m3 tensor-core path (tcgen05 kind::f8f6f4, fp32 accumulate); block scores
   * multiply a bf16 copy of q (exact) with the bf16 hi|lo split of the pooled means. */
  HISA_DTYPE_FP8_E4M3 = 2
} hisa_dtype;

typedef enum hisa_tie_break { HISA_TIE_SMALLEST_INDEX = 0, HISA_TIE_LARGEST_INDEX = 1 } hisa_tie_break;
typedef enum hisa_pool_mode { HISA_POOL_MEAN = 0, HISA_POOL_MAX = 1 } hisa_pool_mode;

/* scorer implementation: the tcgen05/TMA kernel is the product path; the SIMT kernel is a slow
 * device-side cross-check used by the tests (still CUDA, never the CPU). */
typedef enum hisa_scorer { HISA_SCORER_TENSOR = 0, HISA_SCORER_SIMT = 1 } hisa_scorer;

/* POD mirror of hisa::HisaConfig (hisa/config.hpp:47-66) plus the storage dtype of q and k. */
typedef struct hisa_cuda_config {
  uint32_t block_size;    /* B */
  uint32_t block_budget;  /* m */
  uint32_t token_budget;  /* k */
  uint32_t num_heads;     /* H_I  (<= 64) */
  uint32_t dim;           /* d    (<= 128) */
  uint8_t force_first_last; /* default 1 */
  uint8_t forced_in_budget; /* default 0 */
  uint8_t tie_break;        /* hisa_tie_break */
  uint8_t pool_mode;        /* hisa_pool_mode */
  uint32_t dtype;           /* hisa_dtype of queries and keys */
  uint32_t scorer;          /* hisa_scorer */
  uint32_t reserved[4];     /* must be zero */
} hisa_cuda_config;

/* fills the defaults of hisa::HisaConfig for the given sizes */
void hisa_cuda_config_init(hisa_cuda_config* cfg, uint32_t block_size, uint32_t block_budget,
                           uint32_t token_budget, uint32_t num_heads, uint32_t dim, uint32_t dtype);

/* same rule as the HisaConfig constructor (config.hpp:34-44): all fields > 0 and m*B >= k */
int hisa_cuda_config_validate(const hisa_cuda_config* cfg);

int hisa_cuda_abi_version(void);
const char* hisa_cuda_status_name(int status);
/* message of the last failure on this context; ctx == NULL reads the calling thread's global slot
 * (used by hisa_cuda_create failures). The pointer stays valid until the next call on that ctx/thread. */
const char* hisa_cuda_last_error(const hisa_cuda_ctx* ctx);

int hisa_cuda_device_count(int* count);
int hisa_cuda_create(int device, const hisa_cuda_config* cfg, hisa_cuda_ctx** out);
int hisa_cuda_destroy(hisa_cuda_ctx* ctx);
int hisa_cuda_synchronize(hisa_cuda_ctx* ctx);
/* the CUDA stream (cudaStream_t) all work of this context is enqueued on */
void* hisa_cuda_stream(hisa_cuda_ctx* ctx);

/* pinned host memory for asynchronous host<->device copies */
int hisa_cuda_host_alloc(void** ptr, size_t bytes);
int hisa_cuda_host_free(void* ptr);
/* plain device memory helpers so non-CUDA hosts (ctypes, cgo, JNI) can stage data themselves */
int hisa_cuda_device_alloc(hisa_cuda_ctx* ctx, void** ptr, size_t bytes);
int hisa_cuda_device_free(hisa_cuda_ctx* ctx, void* ptr);
int hisa_cuda_memcpy(hisa_cuda_ctx* ctx, void* dst, const void* src, size_t bytes);

/* ---- keys and block summaries ------------------------------------------------------------------ */
/* Replaces the sequence with `seq_len` keys [seq_len, dim] of the context dtype. EmptySequence if 0.
 * check_finite != 0 additionally scans for NaN/Inf (IndexerInputs ingestion rule, inputs.hpp:15-16). */
int hisa_cuda_upload_keys(hisa_cuda_ctx* ctx, const void* keys, uint64_t seq_len, int check_finite);
/* fp8 storage: same as hisa_cuda_upload_keys with per-key dequantisation scales [seq_len] (host or device; NULL = 1). */
int hisa_cuda_upload_keys_scaled(hisa_cuda_ctx* ctx, const void* keys, const float* key_scales, uint64_t seq_len,
                                 int check_finite);
/* (Re)builds all block summaries of the current sequence: build_block_summaries. */
int hisa_cuda_pool_build(hisa_cuda_ctx* ctx);
/* Installs caller-provided block summaries instead of pooling the uploaded keys: the contents of a
 * hisa::BlockSummaryCache (hisa/block_summary.hpp:16-18: per-block f64 sums [num_blocks, dim] and counts [num_blocks])
 * that covers the first num_tokens positions. The snapshot may be SHORTER than the key sequence (the decode contract,
 * block_summary.hpp:27-30: append, then select): a query's eligible blocks are [0, floor(t/B)] clipped to num_blocks
 * (hisa/hisa.hpp:16-21), its forced local block is the last eligible one. Host or device pointers.
 * hisa_cuda_upload_keys / _pool_build / _pool_append go back to summaries computed from the context's keys. */
int hisa_cuda_pool_set(hisa_cuda_ctx* ctx, const double* sums, const uint32_t* counts, uint64_t num_blocks,
                       uint64_t num_tokens);
/* Appends n keys [n, key_dim] at positions seq_len.. and updates only the touched tail blocks
 * (BlockSummaryCache::append, n times, in position order). DimensionMismatch if key_dim != dim. */
int hisa_cuda_pool_append(hisa_cuda_ctx* ctx, const void* keys, uint64_t n, uint32_t key_dim);
/* fp8 storage: same as hisa_cuda_pool_append with per-key dequantisation scales [n] (NULL = 1). */
int hisa_cuda_pool_append_scaled(hisa_cuda_ctx* ctx, const void* keys, const float* key_scales, uint64_t n,
                                 uint32_t key_dim);
/* Reads summaries back: sums [num_blocks, dim] (double), counts [num_blocks], pooled [num_blocks, dim]
 * (double, = sum/count for Mean). Any output may be NULL. */
int hisa_cuda_pool_read(hisa_cuda_ctx* ctx, double* sums, uint32_t* counts, double* pooled);
int hisa_cuda_seq_len(const hisa_cuda_ctx* ctx, uint64_t* seq_len, uint64_t* num_blocks);

/* ---- batched selection ------------------------------------------------------------------------- */
/* queries [Q, H, d] (ctx dtype), gates [Q, H] float32, positions [Q] uint32 (each <= seq_len).
 * out_idx     int32  [Q, token_budget]      ascending, -1 padded            (required)
 * out_count   uint32 [Q]                    = min(k, candidate_size)        (optional)
 * out_blocks  int32  [Q, block_budget + 2]  selected blocks ascending, -1 padded (optional; hisa only)
 * out_nblocks uint32 [Q]                                                     (optional)
 * out_cand    uint32 [Q]                    candidate_size = |Omega_t| (hisa) or t+1 (dsa) (optional)
 * check_finite != 0 scans queries/gates for NaN/Inf first (costs one extra pass). */
int hisa_cuda_hisa_select(hisa_cuda_ctx* ctx, const void* queries, const float* gates,
                          const uint32_t* positions, uint64_t num_queries, int check_finite,
                          int32_t* out_idx, uint32_t* out_count, int32_t* out_blocks,
                          uint32_t* out_nblocks, uint32_t* out_cand);
int hisa_cuda_dsa_select(hisa_cuda_ctx* ctx, const void* queries, const float* gates,
                         const uint32_t* positions, uint64_t num_queries, int check_finite,
                         int32_t* out_idx, uint32_t* out_count, uint32_t* out_cand);
/* Stage 1 only: out_idx is int32 [Q, (block_budget+2)*block_size], all causally valid tokens of the
 * selected blocks, ascending, -1 padded. */
int hisa_cuda_block_sparse_select(hisa_cuda_ctx* ctx, const void* queries, const float* gates,
                                  const uint32_t* positions, uint64_t num_queries, int check_finite,
                                  int32_t* out_idx, uint32_t* out_count, int32_t* out_blocks,
                                  uint32_t* out_nblocks);

/* Output placement for row-sharded runs (one context per GPU, each selecting a subset of the rows of one logical
 * [Q_total, token_budget] result; "callers may fan out queries across workers").
 * While set, hisa_cuda_hisa_select / _dsa_select treat out_idx / out_count / out_cand as the FULL arrays: the result
 * of the call's i-th query is stored at row out_rows[i] (device array of at least num_queries entries; NULL = row i).
 * Every result row is ALSO stored, by the selection kernel itself, at the same row of num_replicas (<= 7) replica
 * arrays replica_idx[r] / replica_count[r] (may be NULL) — device memory that may live on OTHER GPUs with peer access
 * enabled, so that on an NVLink/NVSwitch box the top-k kernel performs the all-gather of the indices with its own
 * stores and no collective, staging copy or permutation follows it. All pointers must be device memory.
 * out_rows == NULL && num_replicas == 0 switches placement off. */
int hisa_cuda_set_output_placement(hisa_cuda_ctx* ctx, const uint32_t* out_rows, int num_replicas,
                                   int32_t* const* replica_idx, uint32_t* const* replica_count);

/* ---- single stages (for per-operation parity tests and callers that compose stages) ------------- */
/* J[row, b] for b in [0, floor(t/B)] (eligible blocks); out_scores float32 [Q, num_blocks], entries of
 * non-eligible blocks are unspecified; out_neligible uint32 [Q]. */
int hisa_cuda_score_blocks(hisa_cuda_ctx* ctx, const void* queries, const float* gates,
                           const uint32_t* positions, uint64_t num_queries, float* out_scores,
                           uint32_t* out_neligible);
/* select_blocks on caller-provided block scores: scores float32 [Q, score_stride], the first
 * neligible[row] entries of a row are the eligible blocks 0..E-1. out_blocks int32 [Q, m+2]. */
int hisa_cuda_select_blocks(hisa_cuda_ctx* ctx, const float* scores, uint64_t score_stride,
                            const uint32_t* neligible, uint64_t num_queries, int32_t* out_blocks,
                            uint32_t* out_nblocks);
/* score_tokens for the whole causal prefix of each row: out_scores float32 [Q, out_stride] with
 * out_stride >= round_up(seq_len, 128); entries beyond t are unspecified. CausalViolation cannot
 * occur by construction (the prefix is generated, not passed in). */
int hisa_cuda_score_tokens(hisa_cuda_ctx* ctx, const void* queries, const float* gates,
                           const uint32_t* positions, uint64_t num_queries, float* out_scores,
                           uint64_t out_stride);
/* top_k_tokens on caller-provided scores: row r holds n[r] candidates at positions 0..n[r]-1.
 * out_idx int32 [Q, k]. */
int hisa_cuda_top_k(hisa_cuda_ctx* ctx, const float* scores, uint64_t score_stride, const uint32_t* n,
                    uint64_t num_rows, uint32_t k, int32_t* out_idx, uint32_t* out_count);

/* ---- downstream consumer: attention over the selected tokens (hisa/attention.hpp:13-59, Eq.3) ----- */
/* Stores latent_states [seq_len, d_model] (HISA_DTYPE_F32 or HISA_DTYPE_BF16; one latent per token acts as key and
 * value). d_model <= 512. Independent of the indexer keys of the context. check_finite != 0 scans for NaN/Inf. */
int hisa_cuda_attn_set_latents(hisa_cuda_ctx* ctx, const void* latent_states, uint64_t seq_len, uint32_t d_model,
                               uint32_t dtype, int check_finite);
/* u_t = sum_{s in T_t} softmax_s(scale * h_t . c_s) * c_s with the softmax normalised over T_t only.
 * query_states [Q, d_model] of q_dtype (F32 or BF16), positions [Q] (each < seq_len),
 * selected int32 [Q, sel_stride]: exactly the out_idx matrix of hisa_cuda_*_select (negative entries are padding),
 * counts [Q] entries to read per row (NULL: all sel_stride entries, padding skipped),
 * scale <= 0 selects 1/sqrt(d_model).  out float32 [Q, d_model]; weights float32 [Q, sel_stride] (optional,
 * selection order, sum to 1, zero on padding).
 * HISA_ERR_EMPTY_SELECTION if a row selects nothing, HISA_ERR_CAUSAL_VIOLATION if an index exceeds the row's position. */
int hisa_cuda_sparse_attend(hisa_cuda_ctx* ctx, const void* query_states, uint32_t q_dtype, const uint32_t* positions,
                            uint64_t num_queries, const int32_t* selected, uint64_t sel_stride, const uint32_t* counts,
                            double scale, float* out, float* weights);
/* Causal softmax attention over the whole prefix [0, t] of every row (the sparse = dense identity oracle). */
int hisa_cuda_dense_attend(hisa_cuda_ctx* ctx, const void* query_states, uint32_t q_dtype, const uint32_t* positions,
                           uint64_t num_queries, double scale, float* out);
/* device time of the attention kernel of the last sparse/dense attend call (CUDA events on the context's stream) */
int hisa_cuda_attn_last_ms(hisa_cuda_ctx* ctx, float* ms);

/* ---- multi-GPU: query rows sharded over the GPUs of one box (csrc/dist.cu) -----------------------------
 * The reference fans rows out over worker threads (hisa/parallel.hpp:15-19; every query row is
 * independent, the key sequence is shared and read-only). Here the workers are GPUs: keys are replicated by
 * ncclBroadcast over NVLink, block summaries are recomputed on every GPU, rows are dealt in 512-row tiles zig-zag over
 * the ranks (causal work grows with the row), and every GPU ends up with the whole [total_rows, token_budget] index
 * matrix in global row order, bit-identical to a single-GPU run. */
typedef struct hisa_cuda_dist hisa_cuda_dist;
#define HISA_DIST_TILE_ROWS 512u
enum { HISA_DIST_DSA = 0, HISA_DIST_HISA = 1 };
/* how "every GPU holds every index row" is achieved:
 *   PEER  the top-k kernel stores each finished row into every GPU's matrix itself (peer stores over NVLink: compute
 *         and all-gather are one kernel). Needs all ranks in one process and peer access between every pair.
 *   NCCL  per-tile ncclBroadcast from the tile's owner, in place, grouped per slice on a second stream so that the
 *         gather of slice i overlaps the kernels of slice i+1.
 *   AUTO  PEER when possible, else NCCL. */
enum { HISA_DIST_GATHER_AUTO = 0, HISA_DIST_GATHER_NCCL = 1, HISA_DIST_GATHER_PEER = 2 };

/* Pure index arithmetic, no device needed: the rows rank `rank` of `world` owns among num_rows rows, ascending
 * (rows_out may be NULL to query only the count). */
int hisa_cuda_dist_plan(uint64_t num_rows, int world, int rank, uint64_t* count, uint32_t* rows_out);
/* One process drives num_devices GPUs (ncclCommInitAll, one host thread + context + stream per GPU). flags: gather mode.
 * A device may be listed several times (logical ranks on one GPU; PEER gather only): used by this library's tests. */
int hisa_cuda_dist_create(const int* devices, int num_devices, const hisa_cuda_config* cfg, uint32_t flags,
                          hisa_cuda_dist** out);
/* One rank of a multi-process job (torchrun / MPI style): rank 0 makes an id (128 bytes) with _unique_id and hands it to
 * the other ranks by any out-of-band channel; every rank then calls _create_rank (ncclCommInitRank). NCCL gather. */
int hisa_cuda_dist_unique_id(void* id, size_t bytes);
int hisa_cuda_dist_create_rank(const void* id, int world, int rank, int device, const hisa_cuda_config* cfg, uint32_t flags,
                               hisa_cuda_dist** out);
int hisa_cuda_dist_destroy(hisa_cuda_dist* d);
/* d == NULL: the calling thread's slot (failures of the create functions and of _plan) */
const char* hisa_cuda_dist_last_error(const hisa_cuda_dist* d);
/* world size, ranks living in this process, the first of them, the gather mode in use (any output may be NULL) */
int hisa_cuda_dist_info(const hisa_cuda_dist* d, int* world, int* num_local, int* first_rank, int* gather);
/* the single-GPU context of local rank `local` (for pool reads, stage timings, launch counts) */
hisa_cuda_ctx* hisa_cuda_dist_ctx(hisa_cuda_dist* d, int local);
/* Replicates the key sequence from rank `root` to every rank and builds the block summaries on each. `keys` (and
 * key_scales for fp8) are read by the process that owns `root` only: host memory or memory of the root's GPU. */
int hisa_cuda_dist_upload_keys(hisa_cuda_dist* d, const void* keys, const float* key_scales, uint64_t seq_len, int root);
/* Sharded selection of total_rows rows. For every LOCAL rank l (index into this process' ranks): queries[l] / gates[l] /
 * positions[l] hold that rank's rows in hisa_cuda_dist_plan order (device memory of that rank's GPU, or host memory).
 * num_slices >= 1: a rank's rows run in that many slices of whole tiles (NCCL gather overlaps slice by slice).
 * Asynchronous: returns when everything is enqueued; results are read with _result after _synchronize (or _fetch). */
int hisa_cuda_dist_select(hisa_cuda_dist* d, int strategy, const void* const* queries, const float* const* gates,
                          const uint32_t* const* positions, uint64_t total_rows, int num_slices);
int hisa_cuda_dist_synchronize(hisa_cuda_dist* d);
/* device pointers of local rank l's copy of the full result: int32 [total_rows, token_budget] and uint32 [total_rows] */
int hisa_cuda_dist_result(hisa_cuda_dist* d, int local, int32_t** idx, uint32_t** count);
/* synchronises and copies local rank l's copy of the result to host memory (either output may be NULL) */
int hisa_cuda_dist_fetch(hisa_cuda_dist* d, int local, int32_t* host_idx, uint32_t* host_count);
/* device time of the last _select: first kernel to "this GPU holds every row", maximum over the local ranks */
int hisa_cuda_dist_last_ms(hisa_cuda_dist* d, float* ms);

/* ---- instrumentation --------------------------------------------------------------------------- */
typedef struct hisa_cuda_stage_times {
  float prepare_ms;      /* dtype conversion / padding of q and w */
  float score_blocks_ms; /* stage 1 scorer (tcgen05)  */
  float select_blocks_ms;/* top-m + forced blocks     */
  float invert_ms;       /* per-block query lists     */
  float score_tokens_ms; /* stage 2 / flat scorer (tcgen05) */
  float top_k_ms;        /* final top-k               */
  float total_ms;        /* first kernel to last kernel of the call */
  uint64_t launches;     /* kernels launched by the call */
  uint64_t work_items_stage1, work_items_stage2; /* scorer work-item capacity (tile x query-list units) */
  uint64_t calls;        /* API calls accumulated in this record */
} hisa_cuda_stage_times;
/* enable != 0: record CUDA events around every stage of subsequent calls (adds a few us).
 * enable & 2: additionally launch the instrumented instantiation of the tensor-core scorer, which keeps the role-level
 * stall counters read by hisa_cuda_scorer_stall_cycles (its clock reads slow the kernel down by a few percent). */
int hisa_cuda_set_profiling(hisa_cuda_ctx* ctx, int enable);
/* Sums over all calls since the previous read (then resets); synchronizes the context's stream. */
int hisa_cuda_last_stage_times(hisa_cuda_ctx* ctx, hisa_cuda_stage_times* out);
/* Role-level stall accounting of the tensor-core scorer, collected while profiling is enabled: 16 counters
 * per stage (cycles summed over all CTAs since the previous read; then reset). Index meaning:
 * 0 CTA lifetime, 1 producer<-scheduler, 2 producer<-tile buffer, 3 producer<-query stage, 4 MMA<-query data,
 * 5 MMA<-tile data, 6 MMA<-epilogue, 7 epilogue<-gates, 8 epilogue<-MMA, 9 epilogue busy, 10 groups. */
int hisa_cuda_scorer_stall_cycles(hisa_cuda_ctx* ctx, uint64_t* stage1, uint64_t* stage2);
/* total kernels launched on this context since creation */
int hisa_cuda_launch_count(const hisa_cuda_ctx* ctx, uint64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* HISA_CUDA_H_ */
