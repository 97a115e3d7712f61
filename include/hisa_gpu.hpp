// hisa_gpu.hpp — what this library ADDS to the reference's C++ surface: batched device entry points.
//
// Everything else a caller needs (hisa::HisaConfig, IndexerInputs, BlockSummaryCache, score_tokens, top_k_tokens,
// dsa_select, score_blocks, select_blocks, candidate_union, hisa_select, block_sparse_select, sparse_attend, ...) is
// declared by the reference's own headers, proj/core/include/hisa/*.hpp, and implemented by libhisa_dropin.so; this
// file includes those headers by their reference names and declares nothing they declare.
//
// A per-row device call is meaningless at scale, so the per-row functions of the reference are thin views over the
// batched calls below (one launch sequence for all rows of an IndexerInputs).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include <hisa/attention.hpp>
#include <hisa/bench.hpp>
#include <hisa/block_summary.hpp>
#include <hisa/config.hpp>
#include <hisa/inputs.hpp>
#include <hisa/types.hpp>

namespace hisa::gpu {

// How q / k are stored on the device (hisa_dtype of hisa_cuda.h). FP8: e4m3 bytes, one f32 scale per key and one per
// (query, head), computed on upload (amax / 448) — the scales of q are folded into the gates (hisa_cuda.h).
enum class Storage { F32 = 0, BF16 = 1, FP8 = 2 };

// RAII handle on one hisa_cuda_ctx: one GPU, one stream. Not thread-safe (one per host thread / GPU).
class Indexer {
 public:
  Indexer(const HisaConfig& cfg, Storage storage = Storage::F32, int device = 0);
  ~Indexer();
  Indexer(const Indexer&) = delete;
  Indexer& operator=(const Indexer&) = delete;

  // keys [L, dim] float32 on the host (rounded to bf16 / quantised to e4m3 on upload); pools them on the device
  void set_keys(std::span<const float> keys);
  void append_keys(std::span<const float> keys);  // decode: incremental tail-block update
  // use the contents of `cache` (which may cover fewer tokens than the keys, block_summary.hpp:27-30) instead of the
  // summaries of the uploaded keys: eligible blocks are clipped to cache.num_blocks() (hisa.hpp:16-21)
  void set_summaries(const BlockSummaryCache& cache);
  uint32_t seq_len() const;
  uint32_t num_blocks() const;
  void read_summaries(std::vector<double>& sums, std::vector<uint32_t>& counts) const;
  float last_pool_build_ms() const { return pool_build_ms_; }  // device time of the pooling kernel in set_keys

  // all rows of `inputs` in one device call each; results in row order
  std::vector<SelectionResult> hisa_select_batch(const IndexerInputs& inputs, OpCounter* counter = nullptr);
  std::vector<SelectionResult> dsa_select_batch(const IndexerInputs& inputs, OpCounter* counter = nullptr);
  std::vector<SelectionResult> block_sparse_select_batch(const IndexerInputs& inputs, OpCounter* counter = nullptr);
  // stage outputs for all rows
  std::vector<ScoreVector> score_blocks_batch(const IndexerInputs& inputs);
  std::vector<ScoreVector> score_prefix_batch(const IndexerInputs& inputs);  // score_tokens over [0, t]

  // device time (ms) of the last batched call, by stage; see hisa_cuda_stage_times
  struct Times { float score_blocks_ms, select_blocks_ms, invert_ms, score_tokens_ms, top_k_ms, total_ms; };
  void enable_timing(bool on);
  Times last_times();

  void* raw() const { return ctx_; }  // the underlying hisa_cuda_ctx*

 private:
  void* ctx_ = nullptr;
  HisaConfig cfg_;
  Storage storage_;
  uint32_t summary_blocks_ = 0;  // > 0: summaries installed by set_summaries cover this many blocks
  float pool_build_ms_ = 0.f;
};

// Batched consumer: latents live on the device; one call attends all rows of `attn` over their selections.
class Attention {
 public:
  explicit Attention(const AttentionInputs& attn, Storage storage = Storage::F32, int device = 0);
  ~Attention();
  Attention(const Attention&) = delete;
  Attention& operator=(const Attention&) = delete;
  // out [Q, d_model] row-major; selections[r] belongs to query row r. weights (optional): per row, selection order.
  std::vector<float> sparse_attend_batch(const std::vector<SelectionResult>& selections,
                                         std::vector<std::vector<double>>* weights_out = nullptr);
  std::vector<float> sparse_attend_rows(std::span<const uint32_t> rows, const std::vector<std::span<const uint32_t>>& selected,
                                        std::vector<std::vector<double>>* weights_out = nullptr);
  std::vector<float> dense_attend_batch();
  std::vector<float> dense_attend_rows(std::span<const uint32_t> rows);
  float last_kernel_ms();
  // reads query states / positions from `attn` from now on; its latent table must equal the uploaded one
  void rebind(const AttentionInputs& attn) { attn_ = &attn; }

 private:
  void* ctx_ = nullptr;
  const AttentionInputs* attn_;
  Storage storage_;
};

// Query rows sharded over several GPUs of one box (hisa_cuda_dist_* of hisa_cuda.h; the reference's fan-out over rows,
// hisa/parallel.hpp:15-19, with GPUs as the workers). Keys are replicated by ncclBroadcast, rows are dealt in 512-row
// tiles zig-zag over the GPUs, every GPU ends up with the whole index matrix; results equal the single-GPU ones bit for
// bit. One process drives all GPUs (one host thread per GPU inside the library).
class MultiIndexer {
 public:
  enum class Gather { Auto = 0, Nccl = 1, Peer = 2 };  // how the index rows reach every GPU (hisa_cuda.h)
  MultiIndexer(const HisaConfig& cfg, Storage storage, std::vector<int> devices, Gather gather = Gather::Auto);
  ~MultiIndexer();
  MultiIndexer(const MultiIndexer&) = delete;
  MultiIndexer& operator=(const MultiIndexer&) = delete;

  int world() const { return world_; }
  Gather gather() const { return gather_; }
  void set_keys(std::span<const float> keys);
  // all rows of `inputs`, sharded; token_indices in row order (read back from the first GPU's copy of the gathered
  // matrix). selected_blocks / candidate_size stay on the GPU that computed them and are left empty / 0.
  std::vector<SelectionResult> hisa_select_batch(const IndexerInputs& inputs, int num_slices = 4);
  std::vector<SelectionResult> dsa_select_batch(const IndexerInputs& inputs, int num_slices = 4);
  float last_ms();  // device time of the last batch call, maximum over the GPUs
  // the rows GPU `rank` of `world` owns among num_rows rows, ascending (pure index arithmetic)
  static std::vector<uint32_t> rank_rows(uint64_t num_rows, int world, int rank);
  void* raw() const { return dist_; }  // the underlying hisa_cuda_dist*

 private:
  std::vector<SelectionResult> run(int strategy, const IndexerInputs& inputs, int num_slices);
  void* dist_ = nullptr;
  HisaConfig cfg_;
  Storage storage_;
  int world_ = 1;
  Gather gather_ = Gather::Auto;
};

// The two panels of the paper's Fig. 2 (SPEC.md `bench --mode fixed-budget | ratio`): one BenchRecord per
// (strategy, length). FixedBudget keeps cfg.block_budget; Ratio recomputes m per length so that M : m = ratio : 1
// (m = ceil(ceil(L/B) / ratio), raised to keep m*B >= k).
enum class SweepMode { FixedBudget, Ratio };
// storage: how keys and queries are held on the device (F32 = what hisa::run_bench uses: the reference stores f32).
// time_base: what wall_ns_* measure. Call = the whole batched call, host containers in, host results out (the copies of
// the f32 IndexerInputs over PCIe dominate calls of ~1000 rows); Kernels = the device time of the indexer's kernels only
// (operands resident, as the paper times its kernels).
enum class TimeBase { Call, Kernels };
std::vector<BenchRecord> run_bench_sweep(const HisaConfig& cfg, std::span<const uint32_t> lengths, uint32_t num_queries,
                                         uint64_t seed, std::span<const Strategy> strategies, SweepMode mode,
                                         uint32_t ratio = 4, const BenchOptions& options = {},
                                         Storage storage = Storage::F32, TimeBase time_base = TimeBase::Call);
// hisa::run_bench (hisa/bench.hpp:53) with the device storage and the time base chosen by the caller
BenchRecord run_bench(const HisaConfig& cfg, uint32_t seq_len, uint32_t num_queries, uint64_t seed, Strategy strategy,
                      const BenchOptions& options, Storage storage, TimeBase time_base = TimeBase::Call);

}  // namespace hisa::gpu
