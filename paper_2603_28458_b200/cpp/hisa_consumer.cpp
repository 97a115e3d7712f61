// C++ host layer, part 2: the downstream consumer (hisa/attention.hpp:13-59) and the self-checking audits
// (hisa/audit.hpp:14-80), over the C ABI. As in hisa_gpu.cpp there is no CUDA header here and no CPU
// implementation of scoring, selection or attention: the audits compare device results with each other and with
// pure index arithmetic.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <set>

#include "hisa/attention.hpp"
#include "hisa/audit.hpp"
#include "hisa/bench.hpp"
#include "hisa/config.hpp"
#include "hisa/errors.hpp"
#include "hisa/hisa.hpp"
#include "hisa/inputs.hpp"
#include "hisa/rng.hpp"
#include "hisa/synth.hpp"
#include "hisa/types.hpp"
#include "hisa_cuda.h"
#include "hisa_gpu.hpp"
#include "host_util.hpp"

namespace hisa {

namespace {

[[noreturn]] void raise_status(int status, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (status) {
    case HISA_ERR_CAUSAL_VIOLATION: throw CausalViolation(m);
    case HISA_ERR_EMPTY_SEQUENCE: throw EmptySequence(m);
    case HISA_ERR_DIMENSION_MISMATCH: throw DimensionMismatch(m);
    case HISA_ERR_NON_FINITE: throw NonFiniteValue(m);
    case HISA_ERR_SHAPE_MISMATCH: throw ShapeMismatch(m);
    case HISA_ERR_EMPTY_SELECTION: throw EmptySelection(m);
    case HISA_ERR_INFEASIBLE_CONFIG: throw InfeasibleConfig(m);
    default: throw Error(std::string(hisa_cuda_status_name(status)) + ": " + m);
  }
}
hisa_cuda_ctx* C(void* p) { return static_cast<hisa_cuda_ctx*>(p); }
void check(void* ctx, int status) {
  if (status != HISA_OK) raise_status(status, hisa_cuda_last_error(C(ctx)));
}
using detail::to_bf16;
// the whole latent table / all query states as one span (the reference exposes rows only, attention.hpp:31-36)
std::span<const float> all_latents(const AttentionInputs& a) {
  return a.seq_len() ? std::span<const float>(a.latent(0).data(), size_t(a.seq_len()) * a.d_model()) : std::span<const float>();
}

}  // namespace

// ==================================================================================================
// AttentionInputs (attention.hpp:16-46)
// ==================================================================================================
AttentionInputs::AttentionInputs(std::vector<float> query_states, std::vector<float> latent_states,
                                 std::vector<uint32_t> query_positions, uint32_t d_model, double scale)
    : query_states_(std::move(query_states)), latent_states_(std::move(latent_states)),
      query_positions_(std::move(query_positions)), d_model_(d_model) {
  if (d_model_ == 0) throw DimensionMismatch("attention inputs: d_model must be positive");
  if (latent_states_.size() % d_model_ != 0) throw ShapeMismatch("attention inputs: latent_states size is not a multiple of d_model");
  seq_len_ = uint32_t(latent_states_.size() / d_model_);
  if (query_states_.size() != query_positions_.size() * size_t(d_model_))
    throw ShapeMismatch("attention inputs: query_states size does not match [Q, d_model]");
  auto finite = [](const std::vector<float>& v, const char* what) {
    for (size_t i = 0; i < v.size(); ++i)
      if (!std::isfinite(v[i]))
        throw NonFiniteValue(std::string("attention inputs: non-finite value in ") + what + " at flat index " + std::to_string(i));
  };
  finite(query_states_, "query_states");
  finite(latent_states_, "latent_states");
  for (size_t i = 0; i < query_positions_.size(); ++i)
    if (query_positions_[i] >= seq_len_)
      throw ShapeMismatch("attention inputs: query position " + std::to_string(query_positions_[i]) + " of row " +
                          std::to_string(i) + " is not below the sequence length " + std::to_string(seq_len_));
  scale_ = scale > 0.0 ? scale : 1.0 / std::sqrt(double(d_model_));
}

// ==================================================================================================
// gpu::Attention — batched consumer
// ==================================================================================================
namespace gpu {

Attention::Attention(const AttentionInputs& attn, Storage storage, int device) : attn_(&attn), storage_(storage) {
  // the consumer does not use the indexer configuration; any feasible one creates the context
  hisa_cuda_config c;
  hisa_cuda_config_init(&c, 128, 16, 2048, 64, 128, HISA_DTYPE_BF16);
  hisa_cuda_ctx* ctx = nullptr;
  const int rc = hisa_cuda_create(device, &c, &ctx);
  if (rc != HISA_OK) raise_status(rc, hisa_cuda_last_error(nullptr));
  ctx_ = ctx;
  if (attn.seq_len() == 0) return;  // attending then reports EmptySequence
  int st;
  if (storage == Storage::FP8) {
    hisa_cuda_destroy(ctx);
    ctx_ = nullptr;
    throw Error("attention: latent states are stored as float32 or bfloat16");
  }
  if (storage == Storage::BF16) {
    const auto b = to_bf16(all_latents(attn));
    st = hisa_cuda_attn_set_latents(ctx, b.data(), attn.seq_len(), attn.d_model(), HISA_DTYPE_BF16, 0);
  } else {
    st = hisa_cuda_attn_set_latents(ctx, all_latents(attn).data(), attn.seq_len(), attn.d_model(), HISA_DTYPE_F32, 0);
  }
  if (st != HISA_OK) {
    const std::string msg = hisa_cuda_last_error(ctx);
    hisa_cuda_destroy(ctx);
    ctx_ = nullptr;
    raise_status(st, msg.c_str());
  }
}
Attention::~Attention() {
  if (ctx_) hisa_cuda_destroy(C(ctx_));
}

std::vector<float> Attention::sparse_attend_rows(std::span<const uint32_t> rows,
                                                 const std::vector<std::span<const uint32_t>>& selected,
                                                 std::vector<std::vector<double>>* weights_out) {
  const AttentionInputs& a = *attn_;
  const size_t n = rows.size(), dm = a.d_model();
  if (selected.size() != n) throw ShapeMismatch("sparse_attend: one selection per row expected");
  size_t stride = 1;
  for (size_t i = 0; i < n; ++i) {
    if (rows[i] >= a.num_queries()) throw Error("sparse_attend: query row " + std::to_string(rows[i]) + " out of range");
    if (selected[i].empty()) throw EmptySelection("sparse_attend: empty selection for query row " + std::to_string(rows[i]));
    stride = std::max(stride, selected[i].size());
  }
  std::vector<float> q(n * dm);
  std::vector<uint32_t> pos(n), cnt(n);
  std::vector<int32_t> idx(n * stride, -1);
  for (size_t i = 0; i < n; ++i) {
    std::copy_n(a.query_state(rows[i]).data(), dm, q.data() + i * dm);
    pos[i] = a.position(rows[i]);
    cnt[i] = uint32_t(selected[i].size());
    for (size_t j = 0; j < selected[i].size(); ++j) {
      if (selected[i][j] > 0x7FFFFFFFu || selected[i][j] > pos[i])  // attention.hpp:52
        throw CausalViolation("sparse_attend: index " + std::to_string(selected[i][j]) + " exceeds query position " +
                              std::to_string(pos[i]));
      idx[i * stride + j] = int32_t(selected[i][j]);
    }
  }
  std::vector<float> out(n * dm), w;
  if (weights_out) w.resize(n * stride);
  const void* qp = q.data();
  std::vector<uint16_t> qb;
  if (storage_ == Storage::BF16) {
    qb = to_bf16(q);
    qp = qb.data();
  }
  check(ctx_, hisa_cuda_sparse_attend(C(ctx_), qp, storage_ == Storage::BF16 ? HISA_DTYPE_BF16 : HISA_DTYPE_F32, pos.data(), n,
                                      idx.data(), stride, cnt.data(), a.scale(), out.data(), weights_out ? w.data() : nullptr));
  if (weights_out) {
    weights_out->assign(n, {});
    for (size_t i = 0; i < n; ++i) (*weights_out)[i].assign(w.begin() + i * stride, w.begin() + i * stride + cnt[i]);
  }
  return out;
}

std::vector<float> Attention::sparse_attend_batch(const std::vector<SelectionResult>& selections,
                                                  std::vector<std::vector<double>>* weights_out) {
  std::vector<uint32_t> rows(selections.size());
  std::iota(rows.begin(), rows.end(), 0u);
  std::vector<std::span<const uint32_t>> sel;
  sel.reserve(selections.size());
  for (const SelectionResult& s : selections) sel.emplace_back(s.token_indices);
  return sparse_attend_rows(rows, sel, weights_out);
}

std::vector<float> Attention::dense_attend_rows(std::span<const uint32_t> rows) {
  const AttentionInputs& a = *attn_;
  const size_t n = rows.size(), dm = a.d_model();
  std::vector<float> q(n * dm), out(n * dm);
  std::vector<uint32_t> pos(n);
  for (size_t i = 0; i < n; ++i) {
    if (rows[i] >= a.num_queries()) throw Error("dense_attend: query row " + std::to_string(rows[i]) + " out of range");
    std::copy_n(a.query_state(rows[i]).data(), dm, q.data() + i * dm);
    pos[i] = a.position(rows[i]);
  }
  const void* qp = q.data();
  std::vector<uint16_t> qb;
  if (storage_ == Storage::BF16) {
    qb = to_bf16(q);
    qp = qb.data();
  }
  check(ctx_, hisa_cuda_dense_attend(C(ctx_), qp, storage_ == Storage::BF16 ? HISA_DTYPE_BF16 : HISA_DTYPE_F32, pos.data(), n,
                                     a.scale(), out.data()));
  return out;
}

std::vector<float> Attention::dense_attend_batch() {
  std::vector<uint32_t> rows(attn_->num_queries());
  std::iota(rows.begin(), rows.end(), 0u);
  return dense_attend_rows(rows);
}

float Attention::last_kernel_ms() {
  float ms = 0.f;
  check(ctx_, hisa_cuda_attn_last_ms(C(ctx_), &ms));
  return ms;
}

}  // namespace gpu

// ==================================================================================================
// the reference's per-row consumer calls: one-row device launches on a cached context per AttentionInputs
// ==================================================================================================
namespace {
std::mutex g_attn_mu;
uint64_t g_attn_hash = 0;
uint32_t g_attn_len = 0, g_attn_dm = 0;
std::unique_ptr<gpu::Attention> g_attn_ctx;

// The latent table is uploaded once per latent CONTENT: the key is a hash of the whole table, never the object's
// address (a new AttentionInputs built where a destroyed one lived must not be served the old table). O(table) per
// call; bulk callers use gpu::Attention.
gpu::Attention& attention_for(const AttentionInputs& a) {
  const uint64_t h = detail::hash_span(all_latents(a), 3);
  if (!g_attn_ctx || g_attn_hash != h || g_attn_len != a.seq_len() || g_attn_dm != a.d_model()) {
    g_attn_ctx.reset();
    g_attn_ctx = std::make_unique<gpu::Attention>(a, gpu::Storage::F32);
    g_attn_hash = h;
    g_attn_len = a.seq_len();
    g_attn_dm = a.d_model();
  }
  g_attn_ctx->rebind(a);  // rows and positions are read from the caller's object of THIS call
  return *g_attn_ctx;
}
}  // namespace

std::vector<float> sparse_attend(const AttentionInputs& attn, std::span<const uint32_t> selected, uint32_t row,
                                 std::vector<double>* weights_out) {
  if (selected.empty()) throw EmptySelection("sparse_attend: empty selection");  // attention.hpp:51
  std::lock_guard<std::mutex> g(g_attn_mu);
  const uint32_t rows[1] = {row};
  std::vector<std::vector<double>> w;
  std::vector<float> out = attention_for(attn).sparse_attend_rows(rows, {selected}, weights_out ? &w : nullptr);
  if (weights_out) *weights_out = std::move(w[0]);
  return out;
}

std::vector<float> sparse_attend(const AttentionInputs& attn, const SelectionResult& selection, uint32_t row,
                                 std::vector<double>* weights_out) {
  return sparse_attend(attn, std::span<const uint32_t>(selection.token_indices), row, weights_out);
}

std::vector<float> dense_attend(const AttentionInputs& attn, uint32_t row) {
  std::lock_guard<std::mutex> g(g_attn_mu);
  const uint32_t rows[1] = {row};
  return attention_for(attn).dense_attend_rows(rows);
}

// ==================================================================================================
// audits (audit.hpp:37-80)
// ==================================================================================================
namespace {

struct Instance {
  uint64_t seed;
  HisaConfig cfg;
  uint32_t L;
  std::vector<uint32_t> positions;
};

// Random feasible instance (the reference leaves the distribution open; this one is ours): B in {8..64}, m in
// [2, 8], k in [1, mB], H in [1, 8], d in {8, 16, 32}, L up to 8 mB. `max_t` caps the query positions (regimes).
enum class Regime { Unrestricted, FlatEquivalent, Dense };
Instance draw_instance(uint64_t seed, Regime regime, uint32_t num_queries) {
  Rng rng(seed);
  const uint32_t B = 8u << rng.below(4);
  const uint32_t m = 2 + uint32_t(rng.below(7));
  const uint32_t k = 1 + uint32_t(rng.below(uint64_t(m) * B));
  const uint32_t H = 1 + uint32_t(rng.below(8));
  const uint32_t d = 8u << rng.below(3);
  const uint32_t L = 1 + uint32_t(rng.below(uint64_t(8) * m * B));
  uint32_t max_t = L - 1;
  if (regime == Regime::FlatEquivalent) max_t = std::min(max_t, m * B - 1);  // t + 1 <= mB
  if (regime == Regime::Dense) max_t = std::min(max_t, k - 1);               // t + 1 <= k
  Instance inst{seed, HisaConfig(B, m, k, H, d), L, {}};
  for (uint32_t i = 0; i < num_queries; ++i) inst.positions.push_back(uint32_t(rng.below(uint64_t(max_t) + 1)));
  std::sort(inst.positions.begin(), inst.positions.end());
  return inst;
}

std::string list_head(const std::vector<uint32_t>& v) {
  std::string s = "[";
  for (size_t i = 0; i < std::min<size_t>(v.size(), 8); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s + (v.size() > 8 ? ",...]" : "]");
}

void fail_report(AuditReport& rep, uint64_t seed, uint32_t row, std::string detail) {
  if (rep.failure) return;
  rep.failure = AuditFailure{seed, row, std::move(detail)};
}

constexpr uint32_t kAuditQueries = 64;

}  // namespace

AuditReport run_regime_equivalence_audit(const AuditOptions& opt) {
  AuditReport rep;
  for (uint32_t i = 0; rep.queries_checked < opt.min_queries && rep.passed(); ++i) {
    const uint64_t seed = mix_seed(opt.base_seed, i, 0x5245u);
    Instance inst = draw_instance(seed, Regime::FlatEquivalent, kAuditQueries);
    Rng rng(mix_seed(seed, 1));
    // fault injection runs on the integer lattice (saturated with exact ties) with the opposite tie-break in the
    // hierarchical arm: any row with more than k candidates must then disagree
    const bool inject = opt.inject_tie_mismatch;
    if (inject) {
      inst.cfg = HisaConfig(inst.cfg.block_size, inst.cfg.block_budget, std::min(inst.cfg.token_budget, 4u), 1, inst.cfg.dim);
      inst.L = std::max(inst.L, 4 * inst.cfg.token_budget + 8);
      for (auto& p : inst.positions) p = std::min(inst.L - 1, inst.cfg.block_budget * inst.cfg.block_size - 1);
    }
    const IndexerInputs in = inject ? make_lattice_inputs(rng, inst.L, inst.positions, inst.cfg.num_heads, inst.cfg.dim)
                                    : make_random_inputs(rng, inst.L, inst.positions, inst.cfg.num_heads, inst.cfg.dim);
    gpu::Indexer flat(inst.cfg, gpu::Storage::F32);
    flat.set_keys(in.keys_raw());
    HisaConfig hcfg = inst.cfg;
    if (inject) hcfg.tie_break = inst.cfg.tie_break == TieBreak::SmallestIndex ? TieBreak::LargestIndex : TieBreak::SmallestIndex;
    gpu::Indexer hier(hcfg, gpu::Storage::F32);
    hier.set_keys(in.keys_raw());
    const auto a = hier.hisa_select_batch(in);
    const auto b = flat.dsa_select_batch(in);
    ++rep.instances_run;
    for (uint32_t r = 0; r < in.num_queries() && rep.passed(); ++r) {
      ++rep.queries_checked;
      if (a[r].token_indices != b[r].token_indices)
        fail_report(rep, seed, r, "t=" + std::to_string(in.position(r)) + " <= mB-1 but hisa " + list_head(a[r].token_indices) +
                                      " != dsa " + list_head(b[r].token_indices));
    }
  }
  return rep;
}

AuditReport run_dense_regime_audit(const AuditOptions& opt) {
  AuditReport rep;
  for (uint32_t i = 0; rep.queries_checked < opt.min_queries && rep.passed(); ++i) {
    const uint64_t seed = mix_seed(opt.base_seed, i, 0x4445u);
    const Instance inst = draw_instance(seed, Regime::Dense, kAuditQueries);
    Rng rng(mix_seed(seed, 1));
    const IndexerInputs in = make_random_inputs(rng, inst.L, inst.positions, inst.cfg.num_heads, inst.cfg.dim);
    gpu::Indexer ix(inst.cfg, gpu::Storage::F32);
    ix.set_keys(in.keys_raw());
    const std::vector<SelectionResult> res[3] = {ix.dsa_select_batch(in), ix.hisa_select_batch(in), ix.block_sparse_select_batch(in)};
    ++rep.instances_run;
    for (uint32_t r = 0; r < in.num_queries() && rep.passed(); ++r) {
      ++rep.queries_checked;
      std::vector<uint32_t> prefix(in.position(r) + 1);
      std::iota(prefix.begin(), prefix.end(), 0u);
      for (int s = 0; s < 3; ++s)
        if (res[s][r].token_indices != prefix)
          fail_report(rep, seed, r, std::string(to_string(Strategy(s))) + ": t=" + std::to_string(in.position(r)) +
                                        " < k but selection " + list_head(res[s][r].token_indices) + " is not the full prefix");
    }
  }
  return rep;
}

AuditReport run_subset_chain_audit(const AuditOptions& opt) {
  AuditReport rep;
  for (uint32_t i = 0; rep.queries_checked < opt.min_queries && rep.passed(); ++i) {
    const uint64_t seed = mix_seed(opt.base_seed, i, 0x5343u);
    const Instance inst = draw_instance(seed, Regime::Unrestricted, kAuditQueries);
    Rng rng(mix_seed(seed, 1));
    const IndexerInputs in = make_random_inputs(rng, inst.L, inst.positions, inst.cfg.num_heads, inst.cfg.dim);
    const HisaConfig& cfg = inst.cfg;
    gpu::Indexer ix(cfg, gpu::Storage::F32);
    ix.set_keys(in.keys_raw());
    OpCounter ops;
    const auto first = ix.hisa_select_batch(in, &ops);
    const auto again = ix.hisa_select_batch(in);
    ++rep.instances_run;
    uint64_t bound = 0;
    for (uint32_t r = 0; r < in.num_queries() && rep.passed(); ++r) {
      ++rep.queries_checked;
      const SelectionResult& s = first[r];
      const uint32_t t = in.position(r), B = cfg.block_size;
      bound += analytic_cost(cfg, uint64_t(t) + 1, Strategy::Hisa);
      auto bad = [&](const std::string& what) { fail_report(rep, seed, r, "t=" + std::to_string(t) + ": " + what); };
      // candidate pool = tokens of the selected blocks clipped to the prefix (hisa.hpp:30-33)
      const std::vector<uint32_t> omega = candidate_union(s.selected_blocks, B, t, in.seq_len());
      if (omega.size() != s.candidate_size) bad("candidate_size " + std::to_string(s.candidate_size) + " != |Omega| " + std::to_string(omega.size()));
      if (!omega.empty() && omega.back() > t) bad("candidate pool leaves the causal prefix");
      if (s.token_indices.size() != std::min<size_t>(cfg.token_budget, omega.size())) bad("|T| != min(k, |Omega|)");
      if (!std::is_sorted(s.token_indices.begin(), s.token_indices.end()) ||
          std::adjacent_find(s.token_indices.begin(), s.token_indices.end()) != s.token_indices.end())
        bad("selection is not strictly ascending");
      if (!std::includes(omega.begin(), omega.end(), s.token_indices.begin(), s.token_indices.end())) bad("T is not a subset of Omega");
      const uint32_t limit = cfg.block_budget + (cfg.force_first_last && !cfg.forced_in_budget ? 2u : 0u);
      if (s.selected_blocks.size() > limit) bad("more than m (+2 forced) blocks selected");
      if (cfg.force_first_last && (s.selected_blocks.empty() || s.selected_blocks.front() != 0 || s.selected_blocks.back() != t / B))
        bad("forced first/last block missing");
      if (again[r].token_indices != s.token_indices || again[r].selected_blocks != s.selected_blocks) bad("second run differs (determinism)");
    }
    if (rep.passed() && ops.dot_products > bound)
      fail_report(rep, seed, 0, "dot products " + std::to_string(ops.dot_products) + " exceed the analytic bound " + std::to_string(bound));
  }
  return rep;
}

std::vector<AblationRow> run_overlap_ablation(const AblationOptions& opt) {
  std::vector<AblationRow> rows;
  for (const AblationConfig& ac : opt.configs) rows.push_back(AblationRow{ac, 0.0, 1.0});
  std::vector<double> sum(opt.configs.size(), 0.0);
  uint64_t count = 0;
  constexpr uint32_t kQueries = 16;
  for (uint32_t sidx = 0; sidx < opt.seeds; ++sidx) {
    Rng rng(mix_seed(opt.base_seed, sidx));
    const IndexerInputs in = make_clustered_inputs(rng, opt.seq_len, kQueries, opt.num_heads, opt.dim);
    // the flat indexer is the reference selection; any feasible (B, m) gives the same dsa result
    const HisaConfig flat_cfg(opt.configs.empty() ? 128 : opt.configs[0].block_size,
                              opt.configs.empty() ? (opt.token_budget + 127) / 128 : opt.configs[0].block_budget, opt.token_budget,
                              opt.num_heads, opt.dim);
    gpu::Indexer flat(flat_cfg, gpu::Storage::F32);
    flat.set_keys(in.keys_raw());
    const auto ref = flat.dsa_select_batch(in);
    for (size_t c = 0; c < opt.configs.size(); ++c) {
      const AblationConfig& ac = opt.configs[c];
      // the block-sparse baseline keeps whole blocks, so its budget need not reach k (SPEC: "Stage 1 only")
      const uint32_t k_cfg = ac.token_refinement ? opt.token_budget : std::min<uint32_t>(opt.token_budget, ac.block_budget * ac.block_size);
      const HisaConfig cfg(ac.block_size, ac.block_budget, k_cfg, opt.num_heads, opt.dim);
      gpu::Indexer ix(cfg, gpu::Storage::F32);
      ix.set_keys(in.keys_raw());
      const auto got = ac.token_refinement ? ix.hisa_select_batch(in) : ix.block_sparse_select_batch(in);
      for (uint32_t r = 0; r < in.num_queries(); ++r) {
        std::vector<uint32_t> inter, uni;
        std::set_intersection(got[r].token_indices.begin(), got[r].token_indices.end(), ref[r].token_indices.begin(),
                              ref[r].token_indices.end(), std::back_inserter(inter));
        std::set_union(got[r].token_indices.begin(), got[r].token_indices.end(), ref[r].token_indices.begin(),
                       ref[r].token_indices.end(), std::back_inserter(uni));
        const double iou = uni.empty() ? 1.0 : double(inter.size()) / double(uni.size());
        sum[c] += iou;
        rows[c].min_overlap = std::min(rows[c].min_overlap, iou);
      }
    }
    count += in.num_queries();
  }
  for (size_t c = 0; c < rows.size(); ++c) rows[c].mean_overlap = count ? sum[c] / double(count) : 0.0;
  return rows;
}

}  // namespace hisa
