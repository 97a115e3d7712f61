// Internal device-side contracts shared by the kernels and the context (not part of the C ABI).
//
// Operand layout in HBM:
//   key operand   bf16 [L_cap,  nseg_k * 128]   row s = key s, split into nseg_k bf16 segments, d padded to 128
//   pooled operand bf16 [M_cap, nseg_p * 128]   row b = pooled key of block b (hi | lo [| lo2] split of the f32 mean)
//   query operand bf16 [Q * 64, nseg_q * 128]   row t*64+j = head j of query t (heads padded to 64 with zeros)
//   gates         f32  [Q, 64]                  padded with zeros and PERMUTED: head j is stored at gate_slot(j),
//                                               so that the 16 gates an epilogue lane needs are contiguous
// A "tile" is 128 consecutive operand rows (the tcgen05 M extent); a "group" is 4 queries x 64 heads
// (the tcgen05 N extent, 256 columns of TMEM).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hisa_dev {

constexpr int kTileRows = 128;  // operand rows per tile (UMMA M)
constexpr int kHeads = 64;      // heads per query in the operand (padded)
constexpr int kDim = 128;       // elements per operand segment (padded d)
constexpr int kGroupQ = 4;      // queries per MMA group (UMMA N = 256)
constexpr int kMaxSeg = 3;       // bf16 segments per operand row
constexpr int kPool8Seg = 4;     // e4m3 terms of a pooled key (fp8 storage): 4 x 4 significant bits
constexpr int kMaxReplicas = 7;  // peer copies of the selection output (8-GPU box: 7 peers)

// position of head j inside a query's 64-float gate row. tcgen05.ld.16x128b hands the columns (heads) {4i + c : i = 0..15}
// to the lanes with (lane % 4) == c; such a lane reads its 16 gates as four 16-byte pieces h = 0..3 (heads 4(4h + u) + c,
// u = 0..3). Piece (h, c) lives at float offset h * 16 + c * 4: for one h the four lane classes read 64 CONTIGUOUS bytes,
// so an LDS.128 of a quarter warp touches every bank once. (Round 1 stored piece (c, h) at c * 16 + h * 4: lane classes
// 0/2 and 1/3 then hit the same banks — a 2-way conflict on every gate load, 475 M conflict wavefronts per C3 launch.)
__host__ __device__ constexpr uint32_t gate_slot(uint32_t j) { return ((j / 4) / 4) * 16 + (j % 4) * 4 + (j / 4) % 4; }

// One unit of scorer work: one operand tile against `count` queries.
//   dense mode: queries are rows first .. first+count-1, results go to out[row, tile*128 + lane]
//   list  mode: queries are pairs[first + i] = {row, col}, results go to out[row, col + (tile % spb)*128 + lane]
struct WorkItem {
  uint32_t tile;
  uint32_t first;
  uint32_t count;
  uint32_t reserved;
};

struct ScoreArgs {
  const WorkItem* work;
  const uint32_t* work_count;  // device scalar: number of valid items in `work`
  uint32_t* work_cursor;       // device scalar, zeroed before launch: dynamic scheduler
  const uint2* pairs;          // list mode
  const float* gates;          // [Q, 64]
  float* out;
  uint64_t out_stride;         // floats per output row
  uint32_t list_mode;
  uint32_t segs_per_block;     // list mode: tiles per key block = ceil(B / 128); dense: 1
  uint32_t block_rows;         // list mode: B; dense: 128
  uint32_t nseg_a, nseg_b;     // operand segments of the tile (A) and query (B) operands (fp8: nseg_a is 1, or 4 for pooled keys)
  uint32_t terms[kMaxSeg];     // terms[ib] = bit mask of A segments multiplied with B segment ib
  uint32_t a_rows;             // rows that exist in the A operand (rows beyond read as zero)
  uint32_t fp8;                // operands are e4m3 bytes [rows, nseg * 128] (kind::f8f6f4); nseg_b = 1
  const float* a_scale;        // fp8: per-row dequantisation scale of the A operand (may be null = 1)
  uint32_t a_tmem;             // bf16, one segment each: multiply the tile from tensor memory (groups of 3 queries)
  uint32_t producers;          // TMA producer warps that take part (1..3)
  uint32_t epi_sleep_ns;       // nanosleep between polls of the epilogue warps' accumulator barrier (0 = spin)
  unsigned long long* stats;   // optional [kScoreStats] role-level stall cycles, summed over CTAs (may be null)
};

// indices into ScoreArgs::stats (cycles, summed over all CTAs of a launch)
enum ScoreStat : int {
  kStatCta = 0,          // CTA lifetime
  kStatProdUnit,         // producer waiting for the scheduler
  kStatProdAEmpty,       // producer waiting for a free tile buffer
  kStatProdBEmpty,       // producer waiting for a free query stage
  kStatMmaBFull,         // MMA issuer waiting for query data (TMA latency / bandwidth)
  kStatMmaAFull,         // MMA issuer waiting for tile data
  kStatMmaTEmpty,        // MMA issuer waiting for the epilogue to drain an accumulator
  kStatEpiWFull,         // MMA issuer waiting for the gates of a group (they ride with its first query chunk)
  kStatCtaMax,           // longest CTA lifetime (max, not a sum)
  kStatEpiBusy,          // epilogue (warp 0) cycles between t_full and t_empty arrive
  kStatGroups,           // groups processed
  kScoreStats
};

// tile -> first operand row and number of meaningful rows
__host__ __device__ inline uint32_t tile_row0(const ScoreArgs& a, uint32_t tile) {
  return (tile / a.segs_per_block) * a.block_rows + (tile % a.segs_per_block) * kTileRows;
}
__host__ __device__ inline uint32_t tile_valid_rows(const ScoreArgs& a, uint32_t tile) {
  const uint32_t off = (tile % a.segs_per_block) * kTileRows;
  const uint32_t left = a.block_rows - off;
  return left < (uint32_t)kTileRows ? left : (uint32_t)kTileRows;
}

enum SelectMode : uint32_t {
  kSelFlat = 0,       // n = t_eff + 1 candidates at positions 0..n-1                  (dsa top-k)
  kSelBlocks = 1,     // n = t_eff / B + 1 block scores, forced first/last, output = block ids (select_blocks)
  kSelCand = 2,       // candidates are the tokens of the row's selected blocks        (hisa top-k)
  kSelGeneric = 3,    // n = n_in[row] candidates at positions 0..n-1                  (top_k_tokens)
  kSelBlocksGeneric = 4  // like kSelBlocks with n = n_in[row]                         (select_blocks)
};

struct SelectArgs {
  const float* scores;
  uint64_t stride;
  const uint32_t* pos;   // [rows] query positions (modes 0,1,2)
  const uint32_t* n_in;  // [rows] candidate counts (modes 3,4)
  uint32_t seq_len, num_blocks, block_size, keep;  // keep = k (tokens) or m (blocks)
  const uint32_t* dyn_len;  // non-null: seq_len (and num_blocks = ceil(seq_len / block_size)) are read from this device word
  uint32_t mode;
  const int32_t* sel;  // mode 2: [rows, sel_stride] selected blocks ascending
  const uint32_t* nsel;
  uint32_t sel_stride;      // entries per row of `sel` (launch_select turns it into the smem word count)
  uint32_t sel_row_stride;  // filled by launch_select: row stride of `sel` in global memory
  uint32_t vec_ok;          // filled by launch_select: score rows are 16-byte aligned
  uint32_t vec_out;         // filled by launch_select: output rows are 16-byte aligned
  uint32_t block_shift;     // filled by launch_select: log2(block_size) or 32
  uint32_t tie_break, force_first_last, forced_in_budget;
  int32_t* out_idx;  // [rows, out_stride], -1 padded
  uint64_t out_stride;
  uint32_t out_width;  // entries to write per row (k, or m+2 for block modes)
  uint32_t* out_count;
  uint32_t* out_cand;
  // output placement (multi-GPU row sharding): result row `row` of this launch is stored at row out_rows[row] of the
  // output arrays (null = identity), and additionally at the same row of n_rep peer replicas of out_idx / out_count
  // (device pointers, usually on OTHER GPUs with peer access enabled: the stores travel over NVLink)
  const uint32_t* out_rows;
  uint32_t n_rep;
  int32_t* rep_out[kMaxReplicas];
  uint32_t* rep_count[kMaxReplicas];
};

// sparse_attend / dense_attend (attention.hpp:48-59): one warp per query row
struct AttendArgs {
  const void* latents;    // [seq_len, dm_pad] f32 or bf16 (zero padded beyond d_model)
  const float* queries;   // [num_rows, dm_pad] f32 query states (zero padded)
  const uint32_t* pos;    // [num_rows] query positions, each < seq_len
  const int32_t* idx;     // [num_rows, idx_stride] selected tokens (negative = padding); null = whole prefix [0, t]
  const uint32_t* count;  // [num_rows] entries of idx to read per row; null = idx_stride
  uint64_t idx_stride;
  uint32_t num_rows, seq_len, d_model, dm_pad;
  uint32_t latents_bf16;
  float scale;
  float* out;             // [num_rows, d_model]
  float* weights;         // optional [num_rows, weights_stride], selection order, zero beyond the row's count
  uint64_t weights_stride;
  uint32_t* flag;         // device word, OR of: 1 empty selection, 2 causal violation, 4 position >= seq_len
  uint32_t force_simt;    // HISA_ATTEND_SIMT: keep bf16 latents on the SIMT kernel (cross-check of the MMA kernel)
};

// Opts `func` into `bytes` of dynamic shared memory on the CURRENT device. The attribute belongs to the device's
// context, not to the process, so the "already done" memo is keyed by (device, function): a process that drives one
// hisa_cuda_ctx per GPU opts every kernel in on every device. Thread-safe. Returns false when the device refuses.
bool smem_opt_in(const void* func, size_t bytes);

// ---- launchers (each returns the number of kernels it launched; a negative value is a launch the device cannot
// take, e.g. more shared memory than an SM has) -----------------------------------------------------------------
// padded model dimension the attention kernel works on (32 * 2^i, at most 512); 0 = unsupported
uint32_t attend_padded_dim(uint32_t d_model, bool bf16);
int launch_sparse_attend(const AttendArgs& args, cudaStream_t stream);
int launch_pad_rows(const void* src, bool src_bf16, uint64_t rows, uint32_t dim, uint32_t dim_pad, void* dst,
                    bool dst_bf16, cudaStream_t stream);

int launch_score_tc(const ScoreArgs& args, const CUtensorMap& map_a, const CUtensorMap& map_b, int num_sms,
                    cudaStream_t stream);
int launch_score_simt(const ScoreArgs& args, const __nv_bfloat16* a_op, const __nv_bfloat16* q_op,
                      uint32_t max_items, cudaStream_t stream);

int launch_select(const SelectArgs& args, uint32_t rows, uint32_t n_cap, cudaStream_t stream);


// dense work list: chunk-major list of (tile, chunk) items for rows [0, nq) in chunks of `chunk` queries;
// tile needed iff tile*128 <= min(max position in chunk, seq_len-1) / unit_div.
// dyn_len (may be null): device word holding the sequence length (graph replay); zero_a / zero_b (may be null): two more
// device counters the kernel clears (the stage-2 work list's, saving that list builder a launch)
int launch_build_dense_work(const uint32_t* pos, uint32_t nq, uint32_t chunk, uint32_t seq_len, uint32_t unit_div,
                            uint32_t ntiles, WorkItem* work, uint32_t* work_count, uint32_t* work_cursor,
                            const uint32_t* dyn_len, uint32_t* zero_a, uint32_t* zero_b, cudaStream_t stream);
// list work: per chunk of queries, the per-block lists of (row, slot*B) pairs and one item per (block, seg)
// `split`: most queries one work item may carry (0 = unlimited); longer per-block lists become several items
int launch_invert_selection(const int32_t* sel, const uint32_t* nsel, uint32_t sel_stride, uint32_t nq,
                            uint32_t chunk, uint32_t num_blocks, uint32_t block_size, uint32_t segs_per_block,
                            uint32_t split, WorkItem* work, uint32_t* work_count, uint32_t* work_cursor, uint2* pairs,
                            uint32_t* global_counters, bool counters_zeroed, cudaStream_t stream);
// words of global scratch launch_invert_selection needs for its per-block counters (0: they fit in shared memory)
size_t invert_global_words(uint32_t nq, uint32_t chunk, uint32_t num_blocks);
size_t invert_smem_limit();
// block-sparse output: tokens of the selected blocks clipped to <= t_eff
int launch_expand_blocks(const int32_t* sel, const uint32_t* nsel, uint32_t sel_stride, const uint32_t* pos,
                         uint32_t nq, uint32_t seq_len, uint32_t block_size, int32_t* out_idx, uint64_t out_stride,
                         uint32_t out_width, uint32_t* out_count, cudaStream_t stream);

// operand preparation
// src_type: 0 = f32, 1 = bf16, 2 = e4m3 bytes
int launch_convert_rows(const void* src, uint32_t src_type, uint64_t rows, uint32_t src_heads_or_1,
                        uint32_t src_dim, uint32_t nseg, __nv_bfloat16* dst, uint32_t dst_heads_or_1,
                        cudaStream_t stream);
int launch_permute_gates(const float* src, uint64_t rows, uint32_t heads, float* dst, cudaStream_t stream);
int launch_check_finite(const void* src, uint32_t src_type, uint64_t n, uint32_t* flag, cudaStream_t stream);
int launch_check_positions(const uint32_t* pos, uint64_t n, uint32_t seq_len, uint32_t* flag, cudaStream_t stream);
// block summaries over tokens [first, first+n): double sums, counts, pooled operand (nseg_p segments)
// len_out (may be null): device word that receives first + n, the sequence length after the update
// pool_scale (may be null): non-null selects the e4m3 form of the pooled operand: row b = kPool8Seg x 128 e4m3 bytes
// t0 | t1 | t2 | t3 with pooled key = (t0 + t1 + t2 + t3) * pool_scale[b], pool_scale[b] a power of two (same bytes per row
// as the bf16 hi | lo form, so the two share one buffer); the block scorer then runs in kind::f8f6f4 on the e4m3 queries
int launch_pool_update(const __nv_bfloat16* key_op, uint32_t nseg_k, uint64_t first, uint64_t n, uint32_t block_size,
                       uint32_t dim, uint32_t pool_max, double* sums, uint32_t* counts, __nv_bfloat16* pooled_op,
                       uint32_t nseg_p, uint32_t* len_out, cudaStream_t stream);
int launch_pool_update_fp8(const uint8_t* key8, const float* key_scale, uint64_t first, uint64_t n, uint32_t block_size,
                           uint32_t pool_max, double* sums, uint32_t* counts, __nv_bfloat16* pooled_op, uint32_t nseg_p,
                           float* pool_scale, uint32_t* len_out, cudaStream_t stream);
// installs caller-provided summaries: src_sums f64 [num_blocks, dim], src_counts [num_blocks] (device pointers)
int launch_pool_import(const double* src_sums, const uint32_t* src_counts, uint32_t num_blocks, uint32_t dim,
                       uint32_t pool_max, double* sums, uint32_t* counts, __nv_bfloat16* pooled_op, uint32_t nseg_p,
                       float* pool_scale, cudaStream_t stream);
int launch_fill_f32(float* dst, uint64_t n, float v, cudaStream_t stream);
int launch_pool_export(const double* sums, const uint32_t* counts, uint32_t num_blocks, uint32_t dim,
                       uint32_t pool_max, double* out_sums, double* out_pooled, cudaStream_t stream);

}  // namespace hisa_dev
