// hisa/api.hpp — stand-in for the reference's proj/core/include/hisa/*.hpp where that tree is not installed.
//
// The library is built AGAINST THE REFERENCE'S OWN HEADERS when they are present (cpp/Makefile puts
// $(REF)/include ahead of this directory; tests/test_reference_headers.py checks that every translation unit
// then compiles with no header of this directory except hisa_gpu.hpp / hisa_cuda.h). This file restates the
// same declarations (namespace hisa, same names, argument meaning and error behaviour, each citing the
// reference header it mirrors) so that the drop-in also builds on a machine that only has this repository,
// e.g. the GPU box; the per-file names of the reference (hisa/dsa.hpp, hisa/hisa.hpp, ...) forward here.
//
// What runs where: every function that scores or selects runs on the GPU through the C ABI in
// hisa_cuda.h (there is no CPU implementation of the hot path in this library). Plain containers,
// validation, the RNG, synthetic inputs and file I/O are host code.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <filesystem>
#include <functional>
#include <iosfwd>
#include <optional>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace hisa {

// ---------------------------------------------------------------------------------------------------
// errors — reference: hisa/errors.hpp:10-28
// ---------------------------------------------------------------------------------------------------
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
struct BadMagic : Error { using Error::Error; };
struct VersionMismatch : Error { using Error::Error; };
struct ShapeMismatch : Error { using Error::Error; };
struct NonFiniteValue : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct CausalViolation : Error { using Error::Error; };
struct EmptySequence : Error { using Error::Error; };
struct DimensionMismatch : Error { using Error::Error; };
struct EmptySelection : Error { using Error::Error; };
struct InfeasibleConfig : Error { using Error::Error; };
struct BothEmpty : Error { using Error::Error; };

// ---------------------------------------------------------------------------------------------------
// configuration — reference: hisa/config.hpp:12-67
// ---------------------------------------------------------------------------------------------------
enum class TieBreak { SmallestIndex, LargestIndex };
enum class PoolMode { Mean, Max };

struct HisaConfig {
  // Rejects zero fields and m*B < k, like the reference constructor (config.hpp:27-45).
  HisaConfig(uint32_t block_size_, uint32_t block_budget_, uint32_t token_budget_, uint32_t num_heads_,
             uint32_t dim_)
      : block_size(block_size_), block_budget(block_budget_), token_budget(token_budget_),
        num_heads(num_heads_), dim(dim_) {
    if (!block_size || !block_budget || !token_budget || !num_heads || !dim)
      throw InfeasibleConfig("config: all integer fields must be strictly positive");
    const uint64_t pool = uint64_t(block_budget) * block_size;
    if (pool < token_budget)
      throw InfeasibleConfig("infeasible config: block budget times block size must satisfy mB >= k (got " +
                             std::to_string(block_budget) + "*" + std::to_string(block_size) + "=" +
                             std::to_string(pool) + " < " + std::to_string(token_budget) + ")");
  }
  uint32_t block_size, block_budget, token_budget, num_heads, dim;
  bool force_first_last = true;
  bool forced_in_budget = false;
  TieBreak tie_break = TieBreak::SmallestIndex;
  PoolMode pool_mode = PoolMode::Mean;
};

// ---------------------------------------------------------------------------------------------------
// value types — reference: hisa/types.hpp:12-45
// ---------------------------------------------------------------------------------------------------
enum class Strategy { Dsa, Hisa, BlockSparse };
std::string_view to_string(Strategy s);
Strategy strategy_from_string(std::string_view name);

struct ScoreVector {
  std::vector<double> scores;
  std::vector<uint32_t> positions;
};

struct SelectionResult {
  std::vector<uint32_t> token_indices;
  std::vector<uint32_t> selected_blocks;
  uint64_t candidate_size = 0;
};

struct OpCounter {
  uint64_t dot_products = 0, comparisons = 0, pool_updates = 0;
  void reset() { *this = OpCounter{}; }
  OpCounter& operator+=(const OpCounter& o) {
    dot_products += o.dot_products;
    comparisons += o.comparisons;
    pool_updates += o.pool_updates;
    return *this;
  }
};

// ---------------------------------------------------------------------------------------------------
// inputs — reference: hisa/inputs.hpp:20-56
// ---------------------------------------------------------------------------------------------------
class IndexerInputs {
 public:
  // Validates shapes, rejects NaN/Inf (NonFiniteValue) and positions > L (ShapeMismatch).
  IndexerInputs(std::vector<float> queries, std::vector<float> gates, std::vector<float> keys,
                std::vector<uint32_t> query_positions, uint32_t num_heads, uint32_t dim);

  uint32_t num_queries() const { return static_cast<uint32_t>(query_positions_.size()); }
  uint32_t seq_len() const { return seq_len_; }
  uint32_t num_heads() const { return num_heads_; }
  uint32_t dim() const { return dim_; }
  std::span<const float> query(uint32_t row, uint32_t head) const {
    return {&queries_[(std::size_t(row) * num_heads_ + head) * dim_], dim_};
  }
  float gate(uint32_t row, uint32_t head) const { return gates_[std::size_t(row) * num_heads_ + head]; }
  std::span<const float> key(uint32_t pos) const { return {&keys_[std::size_t(pos) * dim_], dim_}; }
  uint32_t position(uint32_t row) const { return query_positions_[row]; }
  const std::vector<float>& queries_raw() const { return queries_; }
  const std::vector<float>& gates_raw() const { return gates_; }
  const std::vector<float>& keys_raw() const { return keys_; }
  const std::vector<uint32_t>& positions_raw() const { return query_positions_; }

 private:
  std::vector<float> queries_, gates_, keys_;
  std::vector<uint32_t> query_positions_;
  uint32_t num_heads_ = 0, dim_ = 0, seq_len_ = 0;
};

// ---------------------------------------------------------------------------------------------------
// block summaries — reference: hisa/block_summary.hpp:23-59
// ---------------------------------------------------------------------------------------------------
class BlockSummaryCache {
 public:
  BlockSummaryCache(uint32_t block_size, uint32_t dim, PoolMode mode = PoolMode::Mean);
  void append(std::span<const float> key, OpCounter* counter = nullptr);
  uint32_t num_blocks() const { return static_cast<uint32_t>(counts_.size()); }
  uint32_t num_tokens() const { return num_tokens_; }
  uint32_t block_size() const { return block_size_; }
  uint32_t dim() const { return dim_; }
  PoolMode pool_mode() const { return mode_; }
  uint32_t count(uint32_t block) const { return counts_[block]; }
  void pooled(uint32_t block, std::span<double> out) const;
  std::vector<double> pooled(uint32_t block) const;

 private:
  uint32_t block_size_, dim_;
  PoolMode mode_;
  uint32_t num_tokens_ = 0;
  std::vector<double> summary_;  // [num_blocks, dim]: sums (Mean) or running max (Max)
  std::vector<uint32_t> counts_;
};
BlockSummaryCache build_block_summaries(std::span<const float> keys, uint32_t dim, uint32_t block_size,
                                        PoolMode mode = PoolMode::Mean, OpCounter* counter = nullptr);

// ---------------------------------------------------------------------------------------------------
// the flat indexer — reference: hisa/dsa.hpp:13-32
// ---------------------------------------------------------------------------------------------------
ScoreVector score_tokens(const IndexerInputs& inputs, uint32_t query_row, std::span<const uint32_t> candidates,
                         OpCounter* counter = nullptr);
SelectionResult top_k_tokens(const ScoreVector& scores, uint32_t k, TieBreak tie_break,
                             OpCounter* counter = nullptr);
SelectionResult dsa_select(const IndexerInputs& inputs, const HisaConfig& cfg, uint32_t query_row,
                           OpCounter* counter = nullptr);

// ---------------------------------------------------------------------------------------------------
// the hierarchical indexer — reference: hisa/hisa.hpp:16-45, hisa/block_sparse.hpp:12-19
// ---------------------------------------------------------------------------------------------------
ScoreVector score_blocks(const IndexerInputs& inputs, const BlockSummaryCache& cache, uint32_t query_row,
                         OpCounter* counter = nullptr);
std::vector<uint32_t> select_blocks(const ScoreVector& block_scores, const HisaConfig& cfg,
                                    uint32_t query_position, OpCounter* counter = nullptr);
std::vector<uint32_t> candidate_union(std::span<const uint32_t> blocks, uint32_t block_size,
                                      uint32_t query_position, uint32_t seq_len);
SelectionResult hisa_select(const IndexerInputs& inputs, const BlockSummaryCache& cache, const HisaConfig& cfg,
                            uint32_t query_row, OpCounter* counter = nullptr);
SelectionResult block_sparse_select(const IndexerInputs& inputs, const BlockSummaryCache& cache,
                                    const HisaConfig& cfg, uint32_t query_row, OpCounter* counter = nullptr);

// ---------------------------------------------------------------------------------------------------
// hisa-rng-v1 — reference: hisa/rng.hpp:15-67 (the stream is fixed by mt19937_64 + the formulas below)
// ---------------------------------------------------------------------------------------------------
class Rng {
 public:
  explicit Rng(uint64_t seed) : gen_(seed) {}
  uint64_t next_u64() { return gen_(); }
  uint64_t below(uint64_t n) { return uint64_t((static_cast<unsigned __int128>(next_u64()) * n) >> 64); }
  double uniform() { return double(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 2.0 * 3.14159265358979323846 * u2;
    spare_ = radius * std::sin(angle);
    have_spare_ = true;
    return radius * std::cos(angle);
  }

 private:
  std::mt19937_64 gen_;
  bool have_spare_ = false;
  double spare_ = 0.0;
};
inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline uint64_t mix_seed(uint64_t a, uint64_t b, uint64_t c = 0, uint64_t d = 0) {
  return splitmix64(splitmix64(splitmix64(splitmix64(a) ^ b) ^ c) ^ d);
}

// ---------------------------------------------------------------------------------------------------
// synthetic inputs — reference: hisa/synth.hpp:13-39
// ---------------------------------------------------------------------------------------------------
enum class QueryPlacement { Final, Spread };
IndexerInputs make_random_inputs(Rng& rng, uint32_t seq_len, uint32_t num_queries, uint32_t num_heads, uint32_t dim,
                                 QueryPlacement placement = QueryPlacement::Final);
IndexerInputs make_random_inputs(Rng& rng, uint32_t seq_len, std::vector<uint32_t> positions, uint32_t num_heads,
                                 uint32_t dim);
IndexerInputs make_lattice_inputs(Rng& rng, uint32_t seq_len, std::vector<uint32_t> positions, uint32_t num_heads,
                                  uint32_t dim);
IndexerInputs make_clustered_inputs(Rng& rng, uint32_t seq_len, uint32_t num_queries, uint32_t num_heads,
                                    uint32_t dim, uint32_t num_spans = 12, uint32_t span_len = 96,
                                    double span_boost = 3.0);

// ---------------------------------------------------------------------------------------------------
// HSB tensor files — reference: hisa/tensor_io.hpp:11-24
//   "HSB1", u32 version = 1, u32 H, d, L, Q, then keys, queries, gates (f32) and positions (u32), LE.
// ---------------------------------------------------------------------------------------------------
inline constexpr char kHsbMagic[4] = {'H', 'S', 'B', '1'};
inline constexpr uint32_t kHsbVersion = 1;
IndexerInputs load_tensor_file(const std::filesystem::path& path);
void save_tensor_file(const IndexerInputs& inputs, const std::filesystem::path& path);

// ---------------------------------------------------------------------------------------------------
// fan-out helpers — reference: hisa/parallel.hpp:11-19
// ---------------------------------------------------------------------------------------------------
uint32_t worker_count();
void parallel_for(std::size_t n, uint32_t threads, const std::function<void(std::size_t)>& fn);

// ---------------------------------------------------------------------------------------------------
// benchmark harness — reference: hisa/bench.hpp:16-58 (timing is CUDA-event time of the batched device call)
// ---------------------------------------------------------------------------------------------------
struct BenchRecord {
  Strategy strategy = Strategy::Dsa;
  uint32_t seq_len = 0, block_size = 0, block_budget = 0, token_budget = 0, num_heads = 0, dim = 0, queries = 0;
  uint64_t wall_ns_median = 0, wall_ns_p10 = 0, wall_ns_p90 = 0;
  uint64_t pool_build_ns = 0;
  uint64_t dot_products = 0;
  uint64_t analytic_bound = 0;
};
struct BenchOptions {
  uint32_t repetitions = 5;
  uint32_t warmup = 1;
  bool timing = true;
  QueryPlacement placement = QueryPlacement::Final;
};
uint64_t analytic_cost(const HisaConfig& cfg, uint64_t prefix_len, Strategy strategy);
BenchRecord run_bench(const HisaConfig& cfg, uint32_t seq_len, uint32_t num_queries, uint64_t seed,
                      Strategy strategy, const BenchOptions& options = {});
void write_bench_csv(std::ostream& os, const std::vector<BenchRecord>& records);

// ---------------------------------------------------------------------------------------------------
// downstream consumer — reference: hisa/attention.hpp:13-59 (softmax attention over the selected tokens; one latent
// per token acts as key and value). sparse_attend / dense_attend run on the device (hisa_cuda_sparse_attend).
// ---------------------------------------------------------------------------------------------------
class AttentionInputs {
 public:
  // query_states [Q, d_model], latent_states [L, d_model], query_positions [Q] with every position < L;
  // scale <= 0 selects 1/sqrt(d_model). Rejects NaN/Inf (NonFiniteValue) and inconsistent shapes (ShapeMismatch).
  AttentionInputs(std::vector<float> query_states, std::vector<float> latent_states,
                  std::vector<uint32_t> query_positions, uint32_t d_model, double scale = 0.0);

  uint32_t num_queries() const { return static_cast<uint32_t>(query_positions_.size()); }
  uint32_t seq_len() const { return seq_len_; }
  uint32_t d_model() const { return d_model_; }
  double scale() const { return scale_; }
  std::span<const float> query_state(uint32_t row) const { return {&query_states_[std::size_t(row) * d_model_], d_model_}; }
  std::span<const float> latent(uint32_t pos) const { return {&latent_states_[std::size_t(pos) * d_model_], d_model_}; }
  uint32_t position(uint32_t row) const { return query_positions_[row]; }

 private:
  std::vector<float> query_states_, latent_states_;
  std::vector<uint32_t> query_positions_;
  uint32_t d_model_ = 0, seq_len_ = 0;
  double scale_ = 0.0;
};

std::vector<float> sparse_attend(const AttentionInputs& attn, std::span<const uint32_t> selected, uint32_t query_row,
                                 std::vector<double>* weights_out = nullptr);
std::vector<float> sparse_attend(const AttentionInputs& attn, const SelectionResult& selection, uint32_t query_row,
                                 std::vector<double>* weights_out = nullptr);
std::vector<float> dense_attend(const AttentionInputs& attn, uint32_t query_row);

// ---------------------------------------------------------------------------------------------------
// self-checking audits — reference: hisa/audit.hpp:14-80. Every strategy call inside is a batched device call.
// ---------------------------------------------------------------------------------------------------
struct AuditFailure {
  uint64_t instance_seed = 0;
  uint32_t query_row = 0;
  std::string detail;
};
struct AuditReport {
  uint32_t instances_run = 0;
  uint32_t queries_checked = 0;
  std::optional<AuditFailure> failure;
  bool passed() const { return !failure.has_value(); }
};
struct AuditOptions {
  uint64_t base_seed = 1;
  uint32_t min_queries = 1000;  // instances are generated until this many query checks ran
  uint32_t threads = 0;         // unused on the device path (kept for source compatibility)
  bool inject_tie_mismatch = false;  // fault injection: opposite tie-break on a tie-saturated instance
};
AuditReport run_regime_equivalence_audit(const AuditOptions& options);
AuditReport run_dense_regime_audit(const AuditOptions& options);
AuditReport run_subset_chain_audit(const AuditOptions& options);

struct AblationConfig {
  uint32_t block_size = 0;
  uint32_t block_budget = 0;
  bool token_refinement = true;  // false: block-sparse baseline
};
struct AblationRow {
  AblationConfig config;
  double mean_overlap = 0.0;
  double min_overlap = 0.0;
};
struct AblationOptions {
  std::vector<AblationConfig> configs = {{64, 128, true}, {128, 64, true}, {256, 32, true}, {128, 16, false}};
  uint32_t seq_len = 16384;
  uint32_t token_budget = 2048;
  uint32_t num_heads = 4;
  uint32_t dim = 64;
  uint32_t seeds = 20;
  uint64_t base_seed = 7;
  uint32_t threads = 0;
};
std::vector<AblationRow> run_overlap_ablation(const AblationOptions& options);

// ---------------------------------------------------------------------------------------------------
// needle-in-a-haystack harness — reference: hisa/niah.hpp:14-86 (a caller of the path: every selection inside is a
// device call; the haystack scores that place the needle "strictly above every haystack score" also come from the
// device scorer)
// ---------------------------------------------------------------------------------------------------
struct NiahInstance {
  IndexerInputs inputs;
  std::vector<uint32_t> needle_positions;
  uint64_t haystack_seed = 0;
};
NiahInstance generate_niah(uint32_t seq_len, double depth_fraction, uint64_t seed, const HisaConfig& cfg,
                           double needle_sigmas = 6.0);
double selection_overlap(const SelectionResult& a, const SelectionResult& b);  // IoU; BothEmpty if both are empty
double needle_recall(const NiahInstance& instance, const SelectionResult& selection);
struct NiahRecord {
  Strategy strategy = Strategy::Dsa;
  uint32_t seq_len = 0;
  double depth = 0.0;
  uint32_t seed_index = 0;
  double recall = 0.0;
  double overlap_vs_dsa = 0.0;
};
struct NiahGridParams {
  std::vector<uint32_t> lengths = {1024, 2048, 4096, 8192, 16384, 32768};
  std::vector<double> depths = {0.0, 0.25, 0.5, 0.75, 1.0};
  uint32_t seeds = 100;
  uint64_t base_seed = 42;
  uint32_t block_size = 128;
  uint32_t token_budget = 2048;
  uint32_t num_heads = 4;
  uint32_t dim = 16;
  uint32_t ratio = 4;
  double needle_sigmas = 6.0;
  uint32_t threads = 0;  // accepted for source compatibility; the device batches instead
  std::vector<Strategy> strategies = {Strategy::Dsa, Strategy::Hisa, Strategy::BlockSparse};
};
std::vector<NiahRecord> run_niah_grid(const NiahGridParams& params);
void write_niah_csv(std::ostream& os, const std::vector<NiahRecord>& records);
void write_niah_grid_dat(std::ostream& os, const std::vector<NiahRecord>& records, Strategy strategy);

}  // namespace hisa

// batched device entry points (namespace hisa::gpu): this library's own additions, see hisa_gpu.hpp
#include "hisa_gpu.hpp"
