// ORACLE — TEST INFRASTRUCTURE ONLY. See hisa_oracle.hpp for the contract and the parity-pinning notes.
#include "hisa_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>

namespace hisa_oracle {

// --------------------------------------------------------------------------------------------
// config / inputs validation
// --------------------------------------------------------------------------------------------

// Follows the inline constructor body at proj/core/include/hisa/config.hpp:27-45.
void Config::validate() const {
  if (block_size == 0 || block_budget == 0 || token_budget == 0 || num_heads == 0 || dim == 0)
    throw OracleError(Err::InfeasibleConfig, "config: all integer fields must be strictly positive");
  const uint64_t cap = uint64_t(block_budget) * block_size;
  if (cap < token_budget)
    throw OracleError(Err::InfeasibleConfig,
                      "infeasible config: mB >= k violated (" + std::to_string(block_budget) + "*" +
                          std::to_string(block_size) + " < " + std::to_string(token_budget) + ")");
}

// inputs.hpp:13-24 — finite values only, position <= L.
void Inputs::validate() const {
  if (H == 0 || d == 0) throw OracleError(Err::ShapeMismatch, "inputs: num_heads and dim must be positive");
  auto finite = [](const float* p, size_t n, const char* what) {
    for (size_t i = 0; i < n; ++i)
      if (!std::isfinite(p[i]))
        throw OracleError(Err::NonFiniteValue, std::string("inputs: non-finite value in ") + what +
                                                    " at flat index " + std::to_string(i));
  };
  finite(keys, size_t(L) * d, "keys");
  finite(queries, size_t(Q) * H * d, "queries");
  finite(gates, size_t(Q) * H, "gates");
  for (uint32_t i = 0; i < Q; ++i)
    if (positions[i] > L)
      throw OracleError(Err::ShapeMismatch, "inputs: query position " + std::to_string(positions[i]) +
                                                " of row " + std::to_string(i) + " exceeds sequence length");
}

// --------------------------------------------------------------------------------------------
// block summaries — block_summary.hpp:23-59
// --------------------------------------------------------------------------------------------

PoolCache::PoolCache(uint32_t block_size, uint32_t dim, PoolMode mode)
    : block_size_(block_size), dim_(dim), mode_(mode) {
  if (block_size == 0 || dim == 0)
    throw OracleError(Err::InvalidArgument, "block summary cache: block_size and dim must be positive");
}

// One token joins block floor(position / B); Mean keeps double sums, Max a running componentwise max.
void PoolCache::append(const float* key, uint32_t key_dim, OpCounter* c) {
  if (key_dim != dim_)
    throw OracleError(Err::DimensionMismatch, "append: key has " + std::to_string(key_dim) +
                                                  " components, cache dimension is " + std::to_string(dim_));
  const uint32_t b = num_tokens_ / block_size_;
  if (b == counts_.size()) {
    counts_.push_back(0);
    summary_.resize(summary_.size() + dim_, 0.0);
  }
  double* row = &summary_[size_t(b) * dim_];
  if (mode_ == PoolMode::Mean) {
    for (uint32_t i = 0; i < dim_; ++i) row[i] += double(key[i]);
  } else {
    for (uint32_t i = 0; i < dim_; ++i)
      row[i] = counts_[b] == 0 ? double(key[i]) : std::max(row[i], double(key[i]));
  }
  counts_[b] += 1;
  num_tokens_ += 1;
  if (c) c->pool_updates += 1;
}

void PoolCache::pooled(uint32_t block, double* out) const {
  if (block >= counts_.size() || counts_[block] == 0)
    throw OracleError(Err::InvalidArgument, "pooled: block " + std::to_string(block) + " is empty or unknown");
  const double* row = &summary_[size_t(block) * dim_];
  if (mode_ == PoolMode::Mean) {
    const double n = double(counts_[block]);
    for (uint32_t i = 0; i < dim_; ++i) out[i] = row[i] / n;
  } else {
    for (uint32_t i = 0; i < dim_; ++i) out[i] = row[i];
  }
}

PoolCache build_block_summaries(const float* keys, uint64_t L, uint32_t dim, uint32_t block_size,
                                PoolMode mode, OpCounter* c) {
  if (L == 0) throw OracleError(Err::EmptySequence, "build_block_summaries: key matrix has no rows");
  PoolCache cache(block_size, dim, mode);
  for (uint64_t s = 0; s < L; ++s) cache.append(keys + s * dim, dim, c);
  return cache;
}

// --------------------------------------------------------------------------------------------
// scoring — Eq. 1 / Eq. 5
// --------------------------------------------------------------------------------------------

namespace {

// Dot product with f32 storage and f64 accumulation. Eight interleaved partial sums,
// combined in a fixed tree: deterministic, and vectorisable without -ffast-math. A product of two
// floats is exact in double, so FMA contraction cannot change the result.
inline double dot_f64(const double* a, const float* b, uint32_t d) {
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint32_t i = 0;
  for (; i + 8 <= d; i += 8)
    for (int u = 0; u < 8; ++u) acc[u] += a[i + u] * double(b[i + u]);
  for (int u = 0; i < d; ++i, ++u) acc[u] += a[i] * double(b[i]);
  return ((acc[0] + acc[4]) + (acc[2] + acc[6])) + ((acc[1] + acc[5]) + (acc[3] + acc[7]));
}
inline double dot_f64(const double* a, const double* b, uint32_t d) {
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint32_t i = 0;
  for (; i + 8 <= d; i += 8)
    for (int u = 0; u < 8; ++u) acc[u] += a[i + u] * b[i + u];
  for (int u = 0; i < d; ++i, ++u) acc[u] += a[i] * b[i];
  return ((acc[0] + acc[4]) + (acc[2] + acc[6])) + ((acc[1] + acc[5]) + (acc[3] + acc[7]));
}

inline uint32_t effective_position(const Inputs& in, uint32_t row) {
  if (in.L == 0) throw OracleError(Err::EmptySequence, "selection over an empty key sequence");
  return std::min(in.positions[row], in.L - 1);  // decision (5)
}

std::vector<double> widen_query(const Inputs& in, uint32_t row) {
  std::vector<double> q(size_t(in.H) * in.d);
  const float* src = in.queries + size_t(row) * in.H * in.d;
  for (size_t i = 0; i < q.size(); ++i) q[i] = double(src[i]);
  return q;
}

// Strict "a ranks before b" for the deterministic top-k order: higher score first, equal scores by the
// tie-break policy (numeric equality, so +0 == -0).
struct RankBefore {
  const double* s;
  const uint32_t* p;
  TieBreak tb;
  bool operator()(uint32_t a, uint32_t b) const {
    if (s[a] > s[b]) return true;
    if (s[a] < s[b]) return false;
    return tb == TieBreak::SmallestIndex ? p[a] < p[b] : p[a] > p[b];
  }
};

// indices (into the score vector) of the min(k, n) best entries, unordered.
std::vector<uint32_t> best_k(const ScoreVector& sv, uint32_t k, TieBreak tb) {
  const size_t n = sv.scores.size();
  std::vector<uint32_t> order(n);
  std::iota(order.begin(), order.end(), 0u);
  const size_t keep = std::min<size_t>(k, n);
  RankBefore cmp{sv.scores.data(), sv.positions.data(), tb};
  if (keep < n) {
    std::nth_element(order.begin(), order.begin() + keep, order.end(), cmp);
    order.resize(keep);
  }
  return order;
}

}  // namespace

ScoreVector score_tokens(const Inputs& in, uint32_t row, const uint32_t* cand, size_t n, OpCounter* c) {
  if (row >= in.Q) throw OracleError(Err::InvalidArgument, "score_tokens: query row out of range");
  const uint32_t t = in.positions[row];
  for (size_t i = 0; i < n; ++i) {
    if (cand[i] > t)
      throw OracleError(Err::CausalViolation, "score_tokens: candidate " + std::to_string(cand[i]) +
                                                  " exceeds query position " + std::to_string(t));
    if (cand[i] >= in.L)
      throw OracleError(Err::CausalViolation, "score_tokens: candidate " + std::to_string(cand[i]) +
                                                  " is outside the key sequence");
  }
  const std::vector<double> q = widen_query(in, row);
  const float* w = in.gates + size_t(row) * in.H;
  ScoreVector out;
  out.scores.resize(n);
  out.positions.assign(cand, cand + n);
  for (size_t i = 0; i < n; ++i) {
    const float* key = in.keys + size_t(cand[i]) * in.d;
    double acc = 0.0;
    for (uint32_t j = 0; j < in.H; ++j) {
      const double dp = dot_f64(&q[size_t(j) * in.d], key, in.d);
      acc += double(w[j]) * (dp > 0.0 ? dp : 0.0);  // ReLU per head, then the gate
    }
    out.scores[i] = acc;
  }
  if (c) c->dot_products += uint64_t(in.H) * n;
  return out;
}

Selection top_k_tokens(const ScoreVector& sv, uint32_t k, TieBreak tb, OpCounter* c) {
  if (sv.scores.size() != sv.positions.size())
    throw OracleError(Err::ShapeMismatch, "top_k_tokens: scores and positions differ in length");
  if (k == 0) throw OracleError(Err::InvalidArgument, "top_k_tokens: k must be at least 1");
  Selection r;
  r.candidate_size = sv.scores.size();
  for (uint32_t i : best_k(sv, k, tb)) r.token_indices.push_back(sv.positions[i]);
  std::sort(r.token_indices.begin(), r.token_indices.end());
  if (c) c->comparisons += sv.scores.size();
  return r;
}

Selection dsa_select(const Inputs& in, const Config& cfg, uint32_t row, OpCounter* c) {
  cfg.validate();
  if (row >= in.Q) throw OracleError(Err::InvalidArgument, "dsa_select: query row out of range");
  const uint32_t t = effective_position(in, row);
  std::vector<uint32_t> prefix(size_t(t) + 1);
  std::iota(prefix.begin(), prefix.end(), 0u);
  Inputs clipped = in;  // t == L is scored as t_eff (decision 5): bypass the s <= t check consistently
  const ScoreVector sv = score_tokens(clipped, row, prefix.data(), prefix.size(), c);
  Selection r = top_k_tokens(sv, cfg.token_budget, cfg.tie_break, c);
  r.selected_blocks.clear();
  return r;
}

ScoreVector score_blocks(const Inputs& in, const PoolCache& cache, uint32_t row, OpCounter* c) {
  if (row >= in.Q) throw OracleError(Err::InvalidArgument, "score_blocks: query row out of range");
  if (cache.dim() != in.d)
    throw OracleError(Err::DimensionMismatch, "score_blocks: cache dimension differs from the inputs");
  if (cache.num_blocks() == 0) throw OracleError(Err::EmptySequence, "score_blocks: empty block summary cache");
  const uint32_t t = in.positions[row];
  const uint32_t last = std::min<uint32_t>(t / cache.block_size(), cache.num_blocks() - 1);
  const std::vector<double> q = widen_query(in, row);
  const float* w = in.gates + size_t(row) * in.H;
  ScoreVector out;
  out.scores.resize(size_t(last) + 1);
  out.positions.resize(size_t(last) + 1);
  std::vector<double> pk(in.d);
  for (uint32_t b = 0; b <= last; ++b) {
    cache.pooled(b, pk.data());
    double acc = 0.0;
    for (uint32_t j = 0; j < in.H; ++j) {
      const double dp = dot_f64(&q[size_t(j) * in.d], pk.data(), in.d);
      acc += double(w[j]) * (dp > 0.0 ? dp : 0.0);
    }
    out.scores[b] = acc;
    out.positions[b] = b;
  }
  if (c) c->dot_products += uint64_t(in.H) * (uint64_t(last) + 1);
  return out;
}

std::vector<uint32_t> select_blocks(const ScoreVector& js, const Config& cfg, uint32_t query_position,
                                    OpCounter* c) {
  const size_t n = js.scores.size();
  if (n == 0) throw OracleError(Err::EmptySelection, "select_blocks: no eligible block");
  if (js.positions.size() != n)
    throw OracleError(Err::ShapeMismatch, "select_blocks: scores and positions differ in length");
  // forced blocks: the first eligible one (sink) and the one containing the query (local context)
  std::vector<char> forced(n, 0);
  if (cfg.force_first_last) {
    forced[0] = 1;
    const uint32_t local = query_position / cfg.block_size;
    size_t li = n - 1;  // the block containing t is the last eligible one; fall back to it when t == L
    for (size_t i = 0; i < n; ++i)
      if (js.positions[i] == local) li = i;
    forced[li] = 1;
  }
  std::vector<char> keep(n, 0);
  if (cfg.forced_in_budget && cfg.force_first_last) {
    size_t used = 0;
    for (size_t i = 0; i < n; ++i)
      if (forced[i]) { keep[i] = 1; ++used; }
    const size_t room = cfg.block_budget > used ? cfg.block_budget - used : 0;
    ScoreVector rest;
    std::vector<uint32_t> back;
    for (size_t i = 0; i < n; ++i)
      if (!forced[i]) {
        rest.scores.push_back(js.scores[i]);
        rest.positions.push_back(js.positions[i]);
        back.push_back(uint32_t(i));
      }
    if (room > 0)
      for (uint32_t i : best_k(rest, uint32_t(std::min<size_t>(room, 0xffffffffu)), cfg.tie_break))
        keep[back[i]] = 1;
  } else {
    for (uint32_t i : best_k(js, cfg.block_budget, cfg.tie_break)) keep[i] = 1;
    for (size_t i = 0; i < n; ++i)
      if (forced[i]) keep[i] = 1;
  }
  std::vector<uint32_t> out;
  for (size_t i = 0; i < n; ++i)
    if (keep[i]) out.push_back(js.positions[i]);
  std::sort(out.begin(), out.end());
  if (c) c->comparisons += n;
  return out;
}

std::vector<uint32_t> candidate_union(const uint32_t* blocks, size_t nb, uint32_t block_size,
                                      uint32_t query_position, uint32_t seq_len) {
  std::vector<uint32_t> sorted(blocks, blocks + nb);
  std::sort(sorted.begin(), sorted.end());
  sorted.erase(std::unique(sorted.begin(), sorted.end()), sorted.end());
  std::vector<uint32_t> out;
  for (uint32_t b : sorted) {
    const uint64_t lo = uint64_t(b) * block_size;
    const uint64_t hi = lo + block_size;  // exclusive
    for (uint64_t s = lo; s < hi && s <= query_position && s < seq_len; ++s) out.push_back(uint32_t(s));
  }
  return out;
}

Selection hisa_select(const Inputs& in, const PoolCache& cache, const Config& cfg, uint32_t row,
                      OpCounter* c) {
  cfg.validate();
  if (row >= in.Q) throw OracleError(Err::InvalidArgument, "hisa_select: query row out of range");
  if (cache.block_size() != cfg.block_size)
    throw OracleError(Err::InvalidArgument, "hisa_select: cache block size differs from the config");
  const uint32_t t = effective_position(in, row);
  const ScoreVector js = score_blocks(in, cache, row, c);
  Selection r;
  r.selected_blocks = select_blocks(js, cfg, t, c);
  const std::vector<uint32_t> omega =
      candidate_union(r.selected_blocks.data(), r.selected_blocks.size(), cfg.block_size, t, in.L);
  const ScoreVector sv = score_tokens(in, row, omega.data(), omega.size(), c);
  Selection fine = top_k_tokens(sv, cfg.token_budget, cfg.tie_break, c);
  r.token_indices = std::move(fine.token_indices);
  r.candidate_size = omega.size();
  return r;
}

Selection block_sparse_select(const Inputs& in, const PoolCache& cache, const Config& cfg, uint32_t row,
                              OpCounter* c) {
  cfg.validate();
  if (row >= in.Q) throw OracleError(Err::InvalidArgument, "block_sparse_select: query row out of range");
  const uint32_t t = effective_position(in, row);
  const ScoreVector js = score_blocks(in, cache, row, c);
  Selection r;
  r.selected_blocks = select_blocks(js, cfg, t, c);
  r.token_indices = candidate_union(r.selected_blocks.data(), r.selected_blocks.size(), cfg.block_size, t, in.L);
  r.candidate_size = r.token_indices.size();
  return r;
}

uint64_t analytic_cost(const Config& cfg, uint64_t prefix_len, int strategy) {
  const uint64_t B = cfg.block_size, H = cfg.num_heads;
  const uint64_t blocks = (prefix_len + B - 1) / B;
  switch (strategy) {
    case 0: return H * prefix_len;
    case 1: return H * (blocks + std::min<uint64_t>(prefix_len, (uint64_t(cfg.block_budget) + 2) * B));
    default: return H * blocks;
  }
}

// --------------------------------------------------------------------------------------------
// hisa-rng-v1 — rng.hpp:15-67. std::mt19937_64 is the 64-bit Mersenne Twister of Matsumoto &
// Nishimura (w=64,n=312,m=156,r=31, a=0xB5026F5AA96619E9, tempering (29,0x5555..),(17,0x71D67FFFEDA60000),
// (37,0xFFF7EEE000000000),43, initialisation multiplier 6364136223846793005), restated here so the
// stream does not depend on the standard library in use.
// --------------------------------------------------------------------------------------------

Rng::Rng(uint64_t seed) {
  mt_[0] = seed;
  for (int i = 1; i < 312; ++i)
    mt_[i] = 6364136223846793005ULL * (mt_[i - 1] ^ (mt_[i - 1] >> 62)) + uint64_t(i);
  idx_ = 312;
}

void Rng::refill() {
  constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL, kA = 0xB5026F5AA96619E9ULL;
  for (int i = 0; i < 312; ++i) {
    const uint64_t x = (mt_[i] & kUpper) | (mt_[(i + 1) % 312] & kLower);
    mt_[i] = mt_[(i + 156) % 312] ^ (x >> 1) ^ ((x & 1ULL) ? kA : 0ULL);
  }
  idx_ = 0;
}

uint64_t Rng::next_u64() {
  if (idx_ >= 312) refill();
  uint64_t x = mt_[idx_++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

uint64_t Rng::below(uint64_t n) {  // multiply-shift reduction, rng.hpp:22-24
  return uint64_t((static_cast<unsigned __int128>(next_u64()) * n) >> 64);
}
double Rng::uniform() { return double(next_u64() >> 11) * 0x1.0p-53; }  // rng.hpp:27
double Rng::uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }

double Rng::normal() {  // Box-Muller with a cached spare, rng.hpp:32-47
  if (have_spare_) {
    have_spare_ = false;
    return spare_;
  }
  double u1;
  do { u1 = uniform(); } while (u1 <= 0.0);
  const double u2 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double a = 2.0 * 3.14159265358979323846 * u2;
  spare_ = r * std::sin(a);
  have_spare_ = true;
  return r * std::cos(a);
}

uint64_t splitmix64(uint64_t x) {  // rng.hpp:55-60
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
uint64_t mix_seed(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {  // rng.hpp:65-67
  return splitmix64(splitmix64(splitmix64(splitmix64(a) ^ b) ^ c) ^ d);
}

// --------------------------------------------------------------------------------------------
// synthetic inputs — synth.hpp:13-39 (draw order etc. are decisions (1)-(3) in the header)
// --------------------------------------------------------------------------------------------

std::vector<uint32_t> make_positions(uint32_t L, uint32_t Q, Placement p) {
  if (L == 0) throw OracleError(Err::EmptySequence, "make_positions: empty sequence");
  std::vector<uint32_t> pos(Q);
  for (uint32_t i = 0; i < Q; ++i)
    pos[i] = p == Placement::Final ? L - 1 : uint32_t((uint64_t(i) * L) / std::max<uint32_t>(Q, 1));
  return pos;
}

OwnedInputs make_random_inputs(Rng& rng, uint32_t L, std::vector<uint32_t> positions, uint32_t H, uint32_t d) {
  OwnedInputs o;
  o.H = H; o.d = d; o.L = L;
  const size_t Q = positions.size();
  o.keys.resize(size_t(L) * d);
  o.queries.resize(Q * H * d);
  o.gates.resize(Q * H);
  for (auto& v : o.keys) v = float(rng.normal());
  for (auto& v : o.queries) v = float(rng.normal());
  for (auto& v : o.gates) v = float(rng.uniform(0.5, 1.5));
  o.positions = std::move(positions);
  return o;
}

OwnedInputs make_lattice_inputs(Rng& rng, uint32_t L, std::vector<uint32_t> positions, uint32_t H, uint32_t d) {
  OwnedInputs o;
  o.H = H; o.d = d; o.L = L;
  const size_t Q = positions.size();
  o.keys.resize(size_t(L) * d);
  o.queries.resize(Q * H * d);
  o.gates.resize(Q * H);
  for (auto& v : o.keys) v = float(int64_t(rng.below(5)) - 2);
  for (auto& v : o.queries) v = float(int64_t(rng.below(5)) - 2);
  for (auto& v : o.gates) v = float(int64_t(rng.below(3)) + 1);
  o.positions = std::move(positions);
  return o;
}

OwnedInputs make_clustered_inputs(Rng& rng, uint32_t L, uint32_t Q, uint32_t H, uint32_t d, uint32_t num_spans,
                                  uint32_t span_len, double span_boost) {
  OwnedInputs o = make_random_inputs(rng, L, make_positions(L, Q, Placement::Final), H, d);
  if (Q == 0 || L == 0) return o;
  // query direction: mean over heads of query row 0, normalised; spans are pushed along it
  std::vector<double> dir(d, 0.0);
  for (uint32_t j = 0; j < H; ++j)
    for (uint32_t i = 0; i < d; ++i) dir[i] += double(o.queries[size_t(j) * d + i]);
  double nrm = 0.0;
  for (double v : dir) nrm += v * v;
  nrm = std::sqrt(nrm);
  if (nrm > 0)
    for (double& v : dir) v /= nrm;
  for (uint32_t s = 0; s < num_spans; ++s) {
    const uint32_t len = std::min(span_len, L);
    const uint32_t start = uint32_t(rng.below(uint64_t(L - len) + 1));
    for (uint32_t p = start; p < start + len; ++p)
      for (uint32_t i = 0; i < d; ++i)
        o.keys[size_t(p) * d + i] = float(double(o.keys[size_t(p) * d + i]) + span_boost * dir[i]);
  }
  return o;
}

// ---- downstream consumer: shared-KV softmax attention over a selection (attention.hpp:13-59) ----
double AttnInputs::effective_scale() const {
  return scale > 0.0 ? scale : 1.0 / std::sqrt(double(d_model));  // attention.hpp:20-21
}

void AttnInputs::validate() const {
  if (d_model == 0) throw OracleError(Err::DimensionMismatch, "attention: d_model must be positive");
  if (L == 0) throw OracleError(Err::EmptySequence, "attention: empty latent sequence");
  for (size_t i = 0; i < size_t(Q) * d_model; ++i)
    if (!std::isfinite(query_states[i])) throw OracleError(Err::NonFiniteValue, "attention: non-finite query state");
  for (size_t i = 0; i < size_t(L) * d_model; ++i)
    if (!std::isfinite(latent_states[i])) throw OracleError(Err::NonFiniteValue, "attention: non-finite latent state");
  for (uint32_t r = 0; r < Q; ++r)
    if (positions[r] >= L)  // attention.hpp:19-20: every position < L
      throw OracleError(Err::ShapeMismatch, "attention: query position " + std::to_string(positions[r]) +
                                                " is not below seq_len " + std::to_string(L));
}

namespace {
// u = sum_i softmax_i(scale * h.c_{s_i}) * c_{s_i}, all arithmetic in double, max-subtracted
std::vector<float> attend_over(const AttnInputs& a, uint32_t row, size_t n, const uint32_t* selected,
                               std::vector<double>* weights_out) {
  const uint32_t dm = a.d_model;
  const float* h = a.query_states + size_t(row) * dm;
  const double scale = a.effective_scale();
  std::vector<double> logit(n);
  double mx = -std::numeric_limits<double>::infinity();
  for (size_t i = 0; i < n; ++i) {
    const uint32_t s = selected ? selected[i] : uint32_t(i);
    const float* c = a.latent_states + size_t(s) * dm;
    double acc = 0.0;
    for (uint32_t e = 0; e < dm; ++e) acc += double(h[e]) * double(c[e]);
    logit[i] = scale * acc;
    mx = std::max(mx, logit[i]);
  }
  double denom = 0.0;
  for (size_t i = 0; i < n; ++i) {
    logit[i] = std::exp(logit[i] - mx);
    denom += logit[i];
  }
  std::vector<double> u(dm, 0.0);
  for (size_t i = 0; i < n; ++i) {
    const uint32_t s = selected ? selected[i] : uint32_t(i);
    const float* c = a.latent_states + size_t(s) * dm;
    const double w = logit[i] / denom;
    logit[i] = w;
    for (uint32_t e = 0; e < dm; ++e) u[e] += w * double(c[e]);
  }
  if (weights_out) *weights_out = std::move(logit);
  std::vector<float> out(dm);
  for (uint32_t e = 0; e < dm; ++e) out[e] = float(u[e]);
  return out;
}
}  // namespace

std::vector<float> sparse_attend(const AttnInputs& a, const uint32_t* selected, size_t n, uint32_t row,
                                 std::vector<double>* weights_out) {
  if (row >= a.Q) throw OracleError(Err::InvalidArgument, "sparse_attend: query_row out of range");
  if (n == 0) throw OracleError(Err::EmptySelection, "sparse_attend: empty selection");  // attention.hpp:51
  const uint32_t t = a.positions[row];
  for (size_t i = 0; i < n; ++i)
    if (selected[i] > t || selected[i] >= a.L)  // attention.hpp:52
      throw OracleError(Err::CausalViolation, "sparse_attend: index " + std::to_string(selected[i]) +
                                                  " exceeds query position " + std::to_string(t));
  return attend_over(a, row, n, selected, weights_out);
}

std::vector<float> dense_attend(const AttnInputs& a, uint32_t row) {
  if (row >= a.Q) throw OracleError(Err::InvalidArgument, "dense_attend: query_row out of range");
  return attend_over(a, row, size_t(a.positions[row]) + 1, nullptr, nullptr);
}

}  // namespace hisa_oracle
