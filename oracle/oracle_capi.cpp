// ORACLE — TEST INFRASTRUCTURE ONLY. Plain-C surface over hisa_oracle.cpp so tests/ and bench.py's
// cpu_baseline leg can drive the CPU restatement through ctypes. Not part of the product.
#include <atomic>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "hisa_oracle.hpp"

using namespace hisa_oracle;

namespace {
thread_local std::string g_err;

struct Problem {  // mirrored by oracle/pyoracle.py::Problem
  const float* queries;
  const float* gates;
  const float* keys;
  const uint32_t* positions;
  uint32_t Q, L, H, d;
  uint32_t block_size, block_budget, token_budget;
  uint8_t force_first_last, forced_in_budget, tie_break, pool_mode;
  uint32_t pool_tokens;  // the BlockSummaryCache covers the first pool_tokens keys (0 = the whole sequence)
};

// the cache a caller would hold: a snapshot of the first pool_tokens positions (block_summary.hpp:27-30)
PoolCache cache_of(const Problem& p, const Inputs& in, const Config& cfg) {
  const uint32_t n = p.pool_tokens ? std::min(p.pool_tokens, in.L) : in.L;
  return build_block_summaries(in.keys, n, in.d, cfg.block_size, cfg.pool_mode);
}

Inputs inputs_of(const Problem& p) {
  Inputs in;
  in.queries = p.queries; in.gates = p.gates; in.keys = p.keys; in.positions = p.positions;
  in.Q = p.Q; in.L = p.L; in.H = p.H; in.d = p.d;
  return in;
}
Config config_of(const Problem& p) {
  Config c;
  c.block_size = p.block_size; c.block_budget = p.block_budget; c.token_budget = p.token_budget;
  c.num_heads = p.H; c.dim = p.d;
  c.force_first_last = p.force_first_last != 0;
  c.forced_in_budget = p.forced_in_budget != 0;
  c.tie_break = p.tie_break ? TieBreak::LargestIndex : TieBreak::SmallestIndex;
  c.pool_mode = p.pool_mode ? PoolMode::Max : PoolMode::Mean;
  return c;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const OracleError& e) {
    g_err = e.what();
    return int(e.code);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

// parallel.hpp:15-19 semantics: independent items, first exception rethrown on the caller.
template <class F>
void parallel_rows(size_t n, uint32_t threads, F&& fn) {
  threads = std::max<uint32_t>(1, std::min<uint32_t>(threads, uint32_t(std::max<size_t>(n, 1))));
  if (threads == 1) {
    for (size_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<size_t> next{0};
  std::exception_ptr first;
  std::mutex mu;
  std::vector<std::thread> pool;
  for (uint32_t w = 0; w < threads; ++w)
    pool.emplace_back([&] {
      try {
        for (size_t i; (i = next.fetch_add(1)) < n;) fn(i);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!first) first = std::current_exception();
        next.store(n);
      }
    });
  for (auto& t : pool) t.join();
  if (first) std::rethrow_exception(first);
}
}  // namespace

extern "C" {

const char* horacle_last_error() { return g_err.c_str(); }
uint32_t horacle_hardware_threads() { return std::max(1u, std::thread::hardware_concurrency()); }

// ---- rng ----
void* horacle_rng_new(uint64_t seed) { return new Rng(seed); }
void horacle_rng_free(void* r) { delete static_cast<Rng*>(r); }
uint64_t horacle_rng_next_u64(void* r) { return static_cast<Rng*>(r)->next_u64(); }
uint64_t horacle_rng_below(void* r, uint64_t n) { return static_cast<Rng*>(r)->below(n); }
double horacle_rng_uniform(void* r) { return static_cast<Rng*>(r)->uniform(); }
double horacle_rng_normal(void* r) { return static_cast<Rng*>(r)->normal(); }
uint64_t horacle_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t horacle_mix_seed(uint64_t a, uint64_t b, uint64_t c, uint64_t d) { return mix_seed(a, b, c, d); }

// ---- synth: kind 0 random, 1 lattice, 2 clustered (positions ignored -> Final placement) ----
int horacle_make_inputs(int kind, uint64_t seed, uint32_t L, const uint32_t* positions, uint32_t Q, uint32_t H,
                        uint32_t d, float* keys, float* queries, float* gates, uint32_t* positions_out) {
  return guarded([&] {
    Rng rng(seed);
    std::vector<uint32_t> pos(positions, positions + (positions ? Q : 0));
    OwnedInputs o = kind == 0   ? make_random_inputs(rng, L, pos, H, d)
                    : kind == 1 ? make_lattice_inputs(rng, L, pos, H, d)
                                : make_clustered_inputs(rng, L, Q, H, d);
    std::memcpy(keys, o.keys.data(), o.keys.size() * sizeof(float));
    std::memcpy(queries, o.queries.data(), o.queries.size() * sizeof(float));
    std::memcpy(gates, o.gates.data(), o.gates.size() * sizeof(float));
    if (positions_out) std::memcpy(positions_out, o.positions.data(), o.positions.size() * sizeof(uint32_t));
  });
}
int horacle_make_positions(uint32_t L, uint32_t Q, int placement, uint32_t* out) {
  return guarded([&] {
    auto p = make_positions(L, Q, placement ? Placement::Spread : Placement::Final);
    std::memcpy(out, p.data(), p.size() * sizeof(uint32_t));
  });
}

int horacle_config_validate(uint32_t B, uint32_t m, uint32_t k, uint32_t H, uint32_t d) {
  return guarded([&] {
    Config c;
    c.block_size = B; c.block_budget = m; c.token_budget = k; c.num_heads = H; c.dim = d;
    c.validate();
  });
}
int horacle_inputs_validate(const Problem* p) {
  return guarded([&] { inputs_of(*p).validate(); });
}
uint64_t horacle_analytic_cost(const Problem* p, uint64_t prefix_len, int strategy) {
  return analytic_cost(config_of(*p), prefix_len, strategy);
}

// ---- block summaries. incremental != 0 streams tokens through append(); both must agree. ----
int horacle_pool_build(const float* keys, uint64_t L, uint32_t d, uint32_t B, int mode, int incremental,
                       double* sums_out, uint32_t* counts_out, double* pooled_out, uint32_t* num_blocks_out) {
  return guarded([&] {
    const PoolMode pm = mode ? PoolMode::Max : PoolMode::Mean;
    PoolCache cache(B, d, pm);
    if (incremental) {
      for (uint64_t s = 0; s < L; ++s) cache.append(keys + s * d, d);
      if (L == 0) throw OracleError(Err::EmptySequence, "empty sequence");
    } else {
      cache = build_block_summaries(keys, L, d, B, pm);
    }
    if (num_blocks_out) *num_blocks_out = cache.num_blocks();
    if (sums_out) std::memcpy(sums_out, cache.raw_summary().data(), cache.raw_summary().size() * sizeof(double));
    if (counts_out) std::memcpy(counts_out, cache.raw_counts().data(), cache.raw_counts().size() * sizeof(uint32_t));
    if (pooled_out)
      for (uint32_t b = 0; b < cache.num_blocks(); ++b) cache.pooled(b, pooled_out + size_t(b) * d);
  });
}
int horacle_pool_append_dim_check(uint32_t cache_dim, uint32_t key_dim) {
  return guarded([&] {
    PoolCache cache(4, cache_dim);
    std::vector<float> key(key_dim, 1.0f);
    cache.append(key.data(), key_dim);
  });
}
int horacle_pool_pooled_check(uint32_t block) {  // pooling an unknown block is an error
  return guarded([&] {
    PoolCache cache(4, 2);
    float key[2] = {1, 2};
    cache.append(key, 2);
    double out[2];
    cache.pooled(block, out);
  });
}

// ---- single operations ----
int horacle_score_tokens(const Problem* p, uint32_t row, const uint32_t* cand, uint64_t n, double* out,
                         uint64_t* dots) {
  return guarded([&] {
    OpCounter c;
    ScoreVector sv = score_tokens(inputs_of(*p), row, cand, n, &c);
    std::memcpy(out, sv.scores.data(), n * sizeof(double));
    if (dots) *dots = c.dot_products;
  });
}
int horacle_top_k(const double* scores, const uint32_t* pos, uint64_t n, uint32_t k, int tie_break,
                  uint32_t* out, uint32_t* out_n, uint64_t* cand_size) {
  return guarded([&] {
    ScoreVector sv;
    sv.scores.assign(scores, scores + n);
    sv.positions.assign(pos, pos + n);
    Selection s = top_k_tokens(sv, k, tie_break ? TieBreak::LargestIndex : TieBreak::SmallestIndex);
    std::memcpy(out, s.token_indices.data(), s.token_indices.size() * sizeof(uint32_t));
    *out_n = uint32_t(s.token_indices.size());
    if (cand_size) *cand_size = s.candidate_size;
  });
}
int horacle_score_blocks(const Problem* p, uint32_t row, double* out, uint32_t* n_out, uint64_t* dots) {
  return guarded([&] {
    Inputs in = inputs_of(*p);
    Config cfg = config_of(*p);
    PoolCache cache = cache_of(*p, in, cfg);
    OpCounter c;
    ScoreVector sv = score_blocks(in, cache, row, &c);
    std::memcpy(out, sv.scores.data(), sv.scores.size() * sizeof(double));
    *n_out = uint32_t(sv.scores.size());
    if (dots) *dots = c.dot_products;
  });
}
// scores against caller-provided pooled keys ("pooled keys {b0=[4,0], b1=[-2,0]}"), built
// by appending each pooled key as a one-token block.
int horacle_score_pooled(const Problem* p, uint32_t row, const float* pooled, uint32_t nb, double* out,
                         uint32_t* n_out) {
  return guarded([&] {
    Inputs in = inputs_of(*p);
    PoolCache cache(p->block_size, in.d);
    // each pooled key repeated block_size times gives exactly that mean
    for (uint32_t b = 0; b < nb; ++b)
      for (uint32_t r = 0; r < p->block_size; ++r) cache.append(pooled + size_t(b) * in.d, in.d);
    ScoreVector sv = score_blocks(in, cache, row);
    std::memcpy(out, sv.scores.data(), sv.scores.size() * sizeof(double));
    *n_out = uint32_t(sv.scores.size());
  });
}
int horacle_select_blocks(const double* scores, const uint32_t* pos, uint32_t n, const Problem* p, uint32_t t,
                          uint32_t* out, uint32_t* n_out) {
  return guarded([&] {
    ScoreVector sv;
    sv.scores.assign(scores, scores + n);
    sv.positions.assign(pos, pos + n);
    Config cfg = config_of(*p);
    auto blocks = select_blocks(sv, cfg, t);
    std::memcpy(out, blocks.data(), blocks.size() * sizeof(uint32_t));
    *n_out = uint32_t(blocks.size());
  });
}
int horacle_candidate_union(const uint32_t* blocks, uint32_t nb, uint32_t B, uint32_t t, uint32_t L,
                            uint32_t* out, uint64_t* n_out) {
  return guarded([&] {
    auto v = candidate_union(blocks, nb, B, t, L);
    if (out) std::memcpy(out, v.data(), v.size() * sizeof(uint32_t));
    *n_out = v.size();
  });
}

// ---- batched selection over a list of rows. strategy: 0 dsa, 1 hisa, 2 block-sparse.
// out_idx [nrows, idx_stride] padded with -1; out_blocks [nrows, m+2] padded with -1.
int horacle_select_batch(int strategy, const Problem* p, const uint32_t* rows, uint32_t nrows, uint32_t threads,
                         int32_t* out_idx, uint32_t idx_stride, uint32_t* out_count, int32_t* out_blocks,
                         uint32_t* out_nblocks, uint64_t* out_cand, uint64_t* out_dots) {
  return guarded([&] {
    const Inputs in = inputs_of(*p);
    const Config cfg = config_of(*p);
    cfg.validate();
    if (in.L == 0) throw OracleError(Err::EmptySequence, "empty sequence");
    const uint32_t bslots = cfg.block_budget + 2;
    PoolCache cache(cfg.block_size, in.d, cfg.pool_mode);
    if (strategy != 0) cache = cache_of(*p, in, cfg);
    std::atomic<uint64_t> dots{0};
    parallel_rows(nrows, threads, [&](size_t i) {
      const uint32_t row = rows ? rows[i] : uint32_t(i);
      OpCounter c;
      Selection s = strategy == 0   ? dsa_select(in, cfg, row, &c)
                    : strategy == 1 ? hisa_select(in, cache, cfg, row, &c)
                                    : block_sparse_select(in, cache, cfg, row, &c);
      dots += c.dot_products;
      if (out_idx) {
        int32_t* dst = out_idx + size_t(i) * idx_stride;
        const size_t n = std::min<size_t>(s.token_indices.size(), idx_stride);
        for (size_t j = 0; j < n; ++j) dst[j] = int32_t(s.token_indices[j]);
        for (size_t j = n; j < idx_stride; ++j) dst[j] = -1;
      }
      if (out_count) out_count[i] = uint32_t(s.token_indices.size());
      if (out_blocks) {
        int32_t* dst = out_blocks + size_t(i) * bslots;
        for (size_t j = 0; j < bslots; ++j)
          dst[j] = j < s.selected_blocks.size() ? int32_t(s.selected_blocks[j]) : -1;
      }
      if (out_nblocks) out_nblocks[i] = uint32_t(s.selected_blocks.size());
      if (out_cand) out_cand[i] = s.candidate_size;
    });
    if (out_dots) *out_dots = dots.load();
  });
}

// ---- per-row trace used by the near-tie analysis in the parity tests: block scores J, the selected
// blocks, the candidate pool and its token scores. Buffers sized by the caller: J [num_blocks],
// blocks [m+2], omega/omega_scores [(m+2)*B] (hisa) or [L] (dsa: strategy 0 fills omega with the prefix).
int horacle_trace_row(int strategy, const Problem* p, uint32_t row, double* J, uint32_t* nJ, uint32_t* blocks,
                      uint32_t* nblocks, uint32_t* omega, double* omega_scores, uint64_t* n_omega) {
  return guarded([&] {
    const Inputs in = inputs_of(*p);
    const Config cfg = config_of(*p);
    cfg.validate();
    if (in.L == 0) throw OracleError(Err::EmptySequence, "empty sequence");
    const uint32_t t = std::min(in.positions[row], in.L - 1);
    std::vector<uint32_t> cand;
    if (strategy == 0) {
      cand.resize(size_t(t) + 1);
      for (uint32_t s = 0; s <= t; ++s) cand[s] = s;
      if (nJ) *nJ = 0;
      if (nblocks) *nblocks = 0;
    } else {
      PoolCache cache = cache_of(*p, in, cfg);
      ScoreVector js = score_blocks(in, cache, row);
      auto sel = select_blocks(js, cfg, t);
      if (J) std::memcpy(J, js.scores.data(), js.scores.size() * sizeof(double));
      if (nJ) *nJ = uint32_t(js.scores.size());
      if (blocks) std::memcpy(blocks, sel.data(), sel.size() * sizeof(uint32_t));
      if (nblocks) *nblocks = uint32_t(sel.size());
      cand = candidate_union(sel.data(), sel.size(), cfg.block_size, t, in.L);
    }
    ScoreVector sv = score_tokens(in, row, cand.data(), cand.size());
    if (omega) std::memcpy(omega, cand.data(), cand.size() * sizeof(uint32_t));
    if (omega_scores) std::memcpy(omega_scores, sv.scores.data(), sv.scores.size() * sizeof(double));
    *n_omega = cand.size();
  });
}

// ---- downstream consumer (attention.hpp:48-59). selected == NULL: dense_attend over [0, t] of every row.
// selected int32 [nrows, sel_stride] (-1 padded), counts [nrows]; out float [nrows, d_model];
// weights (optional) double [nrows, sel_stride], selection order. Row r of the batch is query row rows[r] (or r).
int horacle_attend_batch(const float* query_states, const float* latent_states, const uint32_t* positions, uint32_t Q,
                         uint32_t L, uint32_t d_model, double scale, const uint32_t* rows, uint32_t nrows,
                         const int32_t* selected, uint32_t sel_stride, const uint32_t* counts, uint32_t threads,
                         float* out, double* weights) {
  return guarded([&] {
    AttnInputs a;
    a.query_states = query_states; a.latent_states = latent_states; a.positions = positions;
    a.Q = Q; a.L = L; a.d_model = d_model; a.scale = scale;
    a.validate();
    parallel_rows(nrows, threads ? threads : horacle_hardware_threads(), [&](size_t i) {
      const uint32_t row = rows ? rows[i] : uint32_t(i);
      std::vector<float> u;
      if (selected) {
        std::vector<uint32_t> sel(counts[i]);
        for (uint32_t j = 0; j < counts[i]; ++j) sel[j] = uint32_t(selected[size_t(i) * sel_stride + j]);
        std::vector<double> w;
        u = sparse_attend(a, sel.data(), sel.size(), row, weights ? &w : nullptr);
        if (weights) std::memcpy(weights + size_t(i) * sel_stride, w.data(), w.size() * sizeof(double));
      } else {
        u = dense_attend(a, row);
      }
      std::memcpy(out + size_t(i) * d_model, u.data(), d_model * sizeof(float));
    });
  });
}

}  // extern "C"
