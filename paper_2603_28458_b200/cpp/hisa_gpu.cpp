// C++ host layer: the reference's hisa:: entry points (proj/core/include/hisa/*.hpp — this file compiles against
// those headers themselves when the reference tree is present, see cpp/Makefile) implemented over the C ABI of
// the sm_100a library (include/hisa_cuda.h). No CUDA headers here: this file only calls hisa_cuda_*.
// Scoring and selection always run on the device; there is no CPU implementation of the hot path.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <ostream>
#include <thread>

#include "hisa/bench.hpp"
#include "hisa/block_sparse.hpp"
#include "hisa/block_summary.hpp"
#include "hisa/config.hpp"
#include "hisa/dsa.hpp"
#include "hisa/errors.hpp"
#include "hisa/hisa.hpp"
#include "hisa/inputs.hpp"
#include "hisa/parallel.hpp"
#include "hisa/rng.hpp"
#include "hisa/synth.hpp"
#include "hisa/tensor_io.hpp"
#include "hisa/types.hpp"
#include "hisa_cuda.h"
#include "hisa_gpu.hpp"
#include "host_util.hpp"

namespace hisa {

namespace {

// C status -> the matching exception leaf (hisa/errors.hpp:10-28)
[[noreturn]] void raise(int status, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (status) {
    case HISA_ERR_INFEASIBLE_CONFIG: throw InfeasibleConfig(m);
    case HISA_ERR_CAUSAL_VIOLATION: throw CausalViolation(m);
    case HISA_ERR_EMPTY_SEQUENCE: throw EmptySequence(m);
    case HISA_ERR_DIMENSION_MISMATCH: throw DimensionMismatch(m);
    case HISA_ERR_NON_FINITE: throw NonFiniteValue(m);
    case HISA_ERR_SHAPE_MISMATCH: throw ShapeMismatch(m);
    case HISA_ERR_EMPTY_SELECTION: throw EmptySelection(m);
    default: throw Error(std::string(hisa_cuda_status_name(status)) + ": " + m);
  }
}
void check(hisa_cuda_ctx* ctx, int status) {
  if (status != HISA_OK) raise(status, hisa_cuda_last_error(ctx));
}

hisa_cuda_config to_c(const HisaConfig& c, gpu::Storage st) {
  hisa_cuda_config out;
  hisa_cuda_config_init(&out, c.block_size, c.block_budget, c.token_budget, c.num_heads, c.dim,
                        st == gpu::Storage::BF16  ? HISA_DTYPE_BF16
                        : st == gpu::Storage::FP8 ? HISA_DTYPE_FP8_E4M3
                                                  : HISA_DTYPE_F32);
  out.force_first_last = c.force_first_last;
  out.forced_in_budget = c.forced_in_budget;
  out.tie_break = c.tie_break == TieBreak::LargestIndex ? HISA_TIE_LARGEST_INDEX : HISA_TIE_SMALLEST_INDEX;
  out.pool_mode = c.pool_mode == PoolMode::Max ? HISA_POOL_MAX : HISA_POOL_MEAN;
  return out;
}

using detail::to_bf16;

// float -> e4m3 (fn variant: no infinities, +-448 is the largest magnitude), round to nearest even, saturating
uint8_t e4m3_bits(float f) {
  const uint8_t sign = std::signbit(f) ? 0x80u : 0u;
  float a = std::fabs(f);
  if (!(a < 448.f)) return sign | 0x7Eu;
  if (a < 0x1p-6f) return sign | uint8_t(std::nearbyint(a * 0x1p9f));  // subnormals: multiples of 2^-9 (8 = 2^-6 itself)
  int e;
  std::frexp(a, &e);  // a = frac * 2^e, frac in [0.5, 1)
  e -= 1;             // a in [2^e, 2^(e+1))
  int m = int(std::nearbyint((std::ldexp(a, -e) - 1.f) * 8.f));
  if (m == 8) { m = 0; ++e; }
  return sign | uint8_t(((e + 7) << 3) | m);
}
// rows of `width` floats -> e4m3 bytes + one scale per row (amax / 448; 1 for an all-zero row)
void quantize_rows(std::span<const float> v, size_t width, std::vector<uint8_t>& bytes, std::vector<float>& scales) {
  const size_t rows = width ? v.size() / width : 0;
  bytes.resize(rows * width);
  scales.resize(rows);
  for (size_t r = 0; r < rows; ++r) {
    float amax = 0.f;
    for (size_t i = 0; i < width; ++i) amax = std::max(amax, std::fabs(v[r * width + i]));
    const float sc = amax > 0.f ? amax / 448.f : 1.f;
    scales[r] = sc;
    for (size_t i = 0; i < width; ++i) bytes[r * width + i] = e4m3_bits(v[r * width + i] / sc);
  }
}

hisa_cuda_ctx* C(void* p) { return static_cast<hisa_cuda_ctx*>(p); }

// BlockSummaryCache keeps its sums private (block_summary.hpp:46-52) and the reference grants no friend: the device
// builder and the device uploader reach them through the explicit-instantiation rule, which lets a member pointer of a
// private member be named as a template argument ([temp.spec]/6). Same member names in api.hpp.
template <class Tag, auto Member>
struct Expose {
  friend constexpr auto member_of(Tag) { return Member; }
};
#pragma GCC diagnostic push
#pragma GCC diagnostic ignored "-Wnon-template-friend"
struct SummaryTag { friend constexpr auto member_of(SummaryTag); };
struct CountsTag { friend constexpr auto member_of(CountsTag); };
struct TokensTag { friend constexpr auto member_of(TokensTag); };
#pragma GCC diagnostic pop
template struct Expose<SummaryTag, &BlockSummaryCache::summary_>;
template struct Expose<CountsTag, &BlockSummaryCache::counts_>;
template struct Expose<TokensTag, &BlockSummaryCache::num_tokens_>;

}  // namespace

// ==================================================================================================
// plain host code: types, inputs, summaries container, rng-driven synthesis, HSB files, fan-out
// ==================================================================================================

std::string_view to_string(Strategy s) {
  return s == Strategy::Dsa ? "dsa" : s == Strategy::Hisa ? "hisa" : s == Strategy::BlockSparse ? "block" : "unknown";
}
Strategy strategy_from_string(std::string_view name) {
  if (name == "dsa") return Strategy::Dsa;
  if (name == "hisa") return Strategy::Hisa;
  if (name == "block" || name == "block-sparse") return Strategy::BlockSparse;
  throw Error("unknown strategy '" + std::string(name) + "' (expected dsa, hisa or block)");
}

IndexerInputs::IndexerInputs(std::vector<float> queries, std::vector<float> gates, std::vector<float> keys,
                             std::vector<uint32_t> query_positions, uint32_t num_heads, uint32_t dim)
    : queries_(std::move(queries)), gates_(std::move(gates)), keys_(std::move(keys)),
      query_positions_(std::move(query_positions)), num_heads_(num_heads), dim_(dim) {
  if (num_heads_ == 0 || dim_ == 0) throw ShapeMismatch("inputs: num_heads and dim must be positive");
  if (keys_.size() % dim_ != 0) throw ShapeMismatch("inputs: keys size is not a multiple of dim");
  seq_len_ = uint32_t(keys_.size() / dim_);
  const size_t Q = query_positions_.size();
  if (queries_.size() != Q * num_heads_ * dim_) throw ShapeMismatch("inputs: queries size does not match [Q, H, d]");
  if (gates_.size() != Q * num_heads_) throw ShapeMismatch("inputs: gates size does not match [Q, H]");
  auto finite = [](const std::vector<float>& v, const char* what) {
    for (size_t i = 0; i < v.size(); ++i)
      if (!std::isfinite(v[i]))
        throw NonFiniteValue(std::string("inputs: non-finite value in ") + what + " at flat index " + std::to_string(i));
  };
  finite(keys_, "keys");
  finite(queries_, "queries");
  finite(gates_, "gates");
  for (size_t i = 0; i < Q; ++i)
    if (query_positions_[i] > seq_len_)
      throw ShapeMismatch("inputs: query position " + std::to_string(query_positions_[i]) + " of row " +
                          std::to_string(i) + " exceeds the sequence length " + std::to_string(seq_len_));
}

BlockSummaryCache::BlockSummaryCache(uint32_t block_size, uint32_t dim, PoolMode mode)
    : block_size_(block_size), dim_(dim), mode_(mode) {
  if (block_size == 0 || dim == 0) throw Error("block summary cache: block_size and dim must be positive");
}

// Single-token append is host bookkeeping on the cache object (one double add per component, the same
// arithmetic in the same order as the device kernel). Bulk work goes through build_block_summaries or
// gpu::Indexer::append_keys, which run the pooling kernel.
void BlockSummaryCache::append(std::span<const float> key, OpCounter* counter) {
  if (key.size() != dim_)
    throw DimensionMismatch("append: key has " + std::to_string(key.size()) + " components, cache dimension is " +
                            std::to_string(dim_));
  const uint32_t b = num_tokens_ / block_size_;
  if (b == counts_.size()) {
    counts_.push_back(0);
    summary_.resize(summary_.size() + dim_, 0.0);
  }
  double* row = &summary_[size_t(b) * dim_];
  for (uint32_t i = 0; i < dim_; ++i) {
    const double v = double(key[i]);
    row[i] = mode_ == PoolMode::Mean ? row[i] + v : (counts_[b] == 0 ? v : std::max(row[i], v));
  }
  ++counts_[b];
  ++num_tokens_;
  if (counter) counter->pool_updates += 1;
}

void BlockSummaryCache::pooled(uint32_t block, std::span<double> out) const {
  if (block >= counts_.size() || counts_[block] == 0)
    throw Error("pooled: block " + std::to_string(block) + " is empty or unknown");
  if (out.size() < dim_) throw DimensionMismatch("pooled: output span is smaller than the cache dimension");
  const double* row = &summary_[size_t(block) * dim_];
  const double n = double(counts_[block]);
  for (uint32_t i = 0; i < dim_; ++i) out[i] = mode_ == PoolMode::Mean ? row[i] / n : row[i];
}
std::vector<double> BlockSummaryCache::pooled(uint32_t block) const {
  std::vector<double> out(dim_);
  pooled(block, out);
  return out;
}

// Batch build = the device pooling kernel; the cache object receives the kernel's double sums.
BlockSummaryCache build_block_summaries(std::span<const float> keys, uint32_t dim, uint32_t block_size, PoolMode mode,
                                        OpCounter* counter) {
  if (dim == 0 || block_size == 0) throw Error("build_block_summaries: dim and block_size must be positive");
  if (keys.empty()) throw EmptySequence("build_block_summaries: key matrix has no rows");
  if (keys.size() % dim != 0) throw ShapeMismatch("build_block_summaries: keys size is not a multiple of dim");
  HisaConfig cfg(block_size, 1, 1, 1, dim);
  cfg.pool_mode = mode;
  gpu::Indexer ix(cfg, gpu::Storage::F32);
  ix.set_keys(keys);
  BlockSummaryCache cache(block_size, dim, mode);
  ix.read_summaries(cache.*member_of(SummaryTag{}), cache.*member_of(CountsTag{}));
  cache.*member_of(TokensTag{}) = uint32_t(keys.size() / dim);
  if (counter) counter->pool_updates += cache.num_tokens();
  return cache;
}

std::vector<uint32_t> candidate_union(std::span<const uint32_t> blocks, uint32_t block_size, uint32_t query_position,
                                      uint32_t seq_len) {
  // pure index arithmetic (hisa/hisa.hpp:30-33); on the device this never materialises (select.cu)
  std::vector<uint32_t> sorted(blocks.begin(), blocks.end());
  std::sort(sorted.begin(), sorted.end());
  sorted.erase(std::unique(sorted.begin(), sorted.end()), sorted.end());
  std::vector<uint32_t> out;
  for (uint32_t b : sorted) {
    const uint64_t lo = uint64_t(b) * block_size, hi = lo + block_size;
    for (uint64_t s = lo; s < hi && s <= query_position && s < seq_len; ++s) out.push_back(uint32_t(s));
  }
  return out;
}

namespace {
std::vector<uint32_t> placement_positions(uint32_t L, uint32_t Q, QueryPlacement p) {
  if (L == 0) throw EmptySequence("synthetic inputs: empty sequence");
  std::vector<uint32_t> pos(Q);
  for (uint32_t i = 0; i < Q; ++i) pos[i] = p == QueryPlacement::Final ? L - 1 : uint32_t(uint64_t(i) * L / std::max(Q, 1u));
  return pos;
}
}  // namespace

// Draw order: keys, queries, gates (the HSB payload order); this is a decision of this library, the
// reference does not pin it ("parity unpinned").
IndexerInputs make_random_inputs(Rng& rng, uint32_t seq_len, std::vector<uint32_t> positions, uint32_t num_heads,
                                 uint32_t dim) {
  const size_t Q = positions.size();
  std::vector<float> keys(size_t(seq_len) * dim), queries(Q * num_heads * dim), gates(Q * num_heads);
  for (auto& v : keys) v = float(rng.normal());
  for (auto& v : queries) v = float(rng.normal());
  for (auto& v : gates) v = float(rng.uniform(0.5, 1.5));
  return IndexerInputs(std::move(queries), std::move(gates), std::move(keys), std::move(positions), num_heads, dim);
}
IndexerInputs make_random_inputs(Rng& rng, uint32_t seq_len, uint32_t num_queries, uint32_t num_heads, uint32_t dim,
                                 QueryPlacement placement) {
  return make_random_inputs(rng, seq_len, placement_positions(seq_len, num_queries, placement), num_heads, dim);
}
IndexerInputs make_lattice_inputs(Rng& rng, uint32_t seq_len, std::vector<uint32_t> positions, uint32_t num_heads,
                                  uint32_t dim) {
  const size_t Q = positions.size();
  std::vector<float> keys(size_t(seq_len) * dim), queries(Q * num_heads * dim), gates(Q * num_heads);
  for (auto& v : keys) v = float(int64_t(rng.below(5)) - 2);
  for (auto& v : queries) v = float(int64_t(rng.below(5)) - 2);
  for (auto& v : gates) v = float(int64_t(rng.below(3)) + 1);
  return IndexerInputs(std::move(queries), std::move(gates), std::move(keys), std::move(positions), num_heads, dim);
}
IndexerInputs make_clustered_inputs(Rng& rng, uint32_t seq_len, uint32_t num_queries, uint32_t num_heads, uint32_t dim,
                                    uint32_t num_spans, uint32_t span_len, double span_boost) {
  IndexerInputs base = make_random_inputs(rng, seq_len, num_queries, num_heads, dim, QueryPlacement::Final);
  if (num_queries == 0) return base;
  std::vector<float> keys = base.keys_raw();
  std::vector<double> dir(dim, 0.0);
  for (uint32_t j = 0; j < num_heads; ++j)
    for (uint32_t i = 0; i < dim; ++i) dir[i] += double(base.query(0, j)[i]);
  double nrm = 0.0;
  for (double v : dir) nrm += v * v;
  nrm = std::sqrt(nrm);
  if (nrm > 0)
    for (double& v : dir) v /= nrm;
  for (uint32_t s = 0; s < num_spans; ++s) {
    const uint32_t len = std::min(span_len, seq_len);
    const uint32_t start = uint32_t(rng.below(uint64_t(seq_len - len) + 1));
    for (uint32_t p = start; p < start + len; ++p)
      for (uint32_t i = 0; i < dim; ++i) keys[size_t(p) * dim + i] = float(double(keys[size_t(p) * dim + i]) + span_boost * dir[i]);
  }
  return IndexerInputs(base.queries_raw(), base.gates_raw(), std::move(keys), base.positions_raw(), num_heads, dim);
}

// ---- HSB files (hisa/tensor_io.hpp:11-24) ----
namespace {
template <class T>
void read_exact(std::ifstream& in, T* dst, size_t n, const char* field, const std::filesystem::path& path) {
  in.read(reinterpret_cast<char*>(dst), std::streamsize(n * sizeof(T)));
  if (size_t(in.gcount()) != n * sizeof(T))
    throw ShapeMismatch("HSB file " + path.string() + ": payload truncated in field '" + field + "'");
}
}  // namespace

IndexerInputs load_tensor_file(const std::filesystem::path& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + path.string());
  char magic[4] = {0, 0, 0, 0};
  in.read(magic, 4);
  if (in.gcount() != 4 || std::memcmp(magic, kHsbMagic, 4) != 0)
    throw BadMagic("HSB file " + path.string() + ": bad magic at byte offset 0 (expected \"HSB1\")");
  uint32_t hdr[5];
  read_exact(in, hdr, 5, "header", path);
  if (hdr[0] != kHsbVersion)
    throw VersionMismatch("HSB file " + path.string() + ": version " + std::to_string(hdr[0]) + " at byte offset 4, expected 1");
  const uint32_t H = hdr[1], d = hdr[2], L = hdr[3], Q = hdr[4];
  if (H == 0 || d == 0) throw ShapeMismatch("HSB file " + path.string() + ": header field H or d is zero");
  std::vector<float> keys(size_t(L) * d), queries(size_t(Q) * H * d), gates(size_t(Q) * H);
  std::vector<uint32_t> pos(Q);
  read_exact(in, keys.data(), keys.size(), "keys", path);
  read_exact(in, queries.data(), queries.size(), "queries", path);
  read_exact(in, gates.data(), gates.size(), "gates", path);
  read_exact(in, pos.data(), pos.size(), "query_positions", path);
  char extra;
  in.read(&extra, 1);
  if (in.gcount() != 0) throw ShapeMismatch("HSB file " + path.string() + ": trailing bytes after query_positions");
  return IndexerInputs(std::move(queries), std::move(gates), std::move(keys), std::move(pos), H, d);
}

void save_tensor_file(const IndexerInputs& in, const std::filesystem::path& path) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("cannot open " + path.string() + " for writing");
  const uint32_t hdr[5] = {kHsbVersion, in.num_heads(), in.dim(), in.seq_len(), in.num_queries()};
  out.write(kHsbMagic, 4);
  out.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
  auto put = [&](const auto& v) { out.write(reinterpret_cast<const char*>(v.data()), std::streamsize(v.size() * sizeof(v[0]))); };
  put(in.keys_raw());
  put(in.queries_raw());
  put(in.gates_raw());
  put(in.positions_raw());
  out.flush();
  if (!out) throw IoError("write to " + path.string() + " failed");
}

uint32_t worker_count() {
  uint32_t n = std::max(1u, std::thread::hardware_concurrency());
  if (const char* cap = std::getenv("HISA_THREADS")) {
    const long v = std::strtol(cap, nullptr, 10);
    if (v >= 1) n = std::min<uint32_t>(n, uint32_t(v));
  }
  return std::max(1u, n);
}

void parallel_for(std::size_t n, uint32_t threads, const std::function<void(std::size_t)>& fn) {
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

uint64_t analytic_cost(const HisaConfig& cfg, uint64_t prefix_len, Strategy strategy) {
  const uint64_t B = cfg.block_size, H = cfg.num_heads, blocks = (prefix_len + B - 1) / B;
  switch (strategy) {
    case Strategy::Dsa: return H * prefix_len;
    case Strategy::Hisa: return H * (blocks + std::min<uint64_t>(prefix_len, (uint64_t(cfg.block_budget) + 2) * B));
    default: return H * blocks;
  }
}

// ==================================================================================================
// gpu::Indexer — batched device entry points
// ==================================================================================================
namespace gpu {

Indexer::Indexer(const HisaConfig& cfg, Storage storage, int device) : cfg_(cfg), storage_(storage) {
  const hisa_cuda_config c = to_c(cfg, storage);
  hisa_cuda_ctx* ctx = nullptr;
  const int rc = hisa_cuda_create(device, &c, &ctx);
  if (rc != HISA_OK) raise(rc, hisa_cuda_last_error(nullptr));
  ctx_ = ctx;
}
Indexer::~Indexer() {
  if (ctx_) hisa_cuda_destroy(C(ctx_));
}

void Indexer::set_keys(std::span<const float> keys) {
  if (keys.size() % cfg_.dim != 0) throw ShapeMismatch("set_keys: keys size is not a multiple of dim");
  const uint64_t L = keys.size() / cfg_.dim;
  if (storage_ == Storage::BF16) {
    const auto b = to_bf16(keys);
    check(C(ctx_), hisa_cuda_upload_keys(C(ctx_), b.data(), L, 0));
  } else if (storage_ == Storage::FP8) {
    std::vector<uint8_t> b;
    std::vector<float> sc;
    quantize_rows(keys, cfg_.dim, b, sc);
    check(C(ctx_), hisa_cuda_upload_keys_scaled(C(ctx_), b.data(), sc.data(), L, 0));
  } else {
    check(C(ctx_), hisa_cuda_upload_keys(C(ctx_), keys.data(), L, 0));
  }
  summary_blocks_ = 0;
  // summary build, timed on its own (hisa/bench.hpp:28: "summary build time, reported separately")
  check(C(ctx_), hisa_cuda_synchronize(C(ctx_)));
  const auto t0 = std::chrono::steady_clock::now();
  check(C(ctx_), hisa_cuda_pool_build(C(ctx_)));
  check(C(ctx_), hisa_cuda_synchronize(C(ctx_)));
  pool_build_ms_ = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
}
void Indexer::append_keys(std::span<const float> keys) {
  const uint64_t n = keys.size() / cfg_.dim;
  if (keys.size() % cfg_.dim != 0)
    check(C(ctx_), hisa_cuda_pool_append(C(ctx_), keys.data(), 1, uint32_t(keys.size())));  // -> DimensionMismatch
  summary_blocks_ = 0;
  if (storage_ == Storage::BF16) {
    const auto b = to_bf16(keys);
    check(C(ctx_), hisa_cuda_pool_append(C(ctx_), b.data(), n, cfg_.dim));
  } else if (storage_ == Storage::FP8) {
    std::vector<uint8_t> b;
    std::vector<float> sc;
    quantize_rows(keys, cfg_.dim, b, sc);
    check(C(ctx_), hisa_cuda_pool_append_scaled(C(ctx_), b.data(), sc.data(), n, cfg_.dim));
  } else {
    check(C(ctx_), hisa_cuda_pool_append(C(ctx_), keys.data(), n, cfg_.dim));
  }
}
void Indexer::set_summaries(const BlockSummaryCache& cache) {
  if (cache.dim() != cfg_.dim) throw DimensionMismatch("block summary cache dimension differs from the config");
  if (cache.block_size() != cfg_.block_size) throw Error("block summary cache block size differs from the config");
  if (cache.pool_mode() != cfg_.pool_mode) throw Error("block summary cache pool mode differs from the config");
  if (cache.num_blocks() == 0) throw EmptySequence("score_blocks: empty block summary cache");
  const std::vector<double>& sums = cache.*member_of(SummaryTag{});
  const std::vector<uint32_t>& counts = cache.*member_of(CountsTag{});
  check(C(ctx_), hisa_cuda_pool_set(C(ctx_), sums.data(), counts.data(), cache.num_blocks(), cache.num_tokens()));
  summary_blocks_ = std::min(cache.num_blocks(), (seq_len() + cfg_.block_size - 1) / cfg_.block_size);
}
uint32_t Indexer::seq_len() const {
  uint64_t L = 0, M = 0;
  hisa_cuda_seq_len(C(ctx_), &L, &M);
  return uint32_t(L);
}
uint32_t Indexer::num_blocks() const {
  if (summary_blocks_) return summary_blocks_;
  uint64_t L = 0, M = 0;
  hisa_cuda_seq_len(C(ctx_), &L, &M);
  return uint32_t(M);
}
void Indexer::read_summaries(std::vector<double>& sums, std::vector<uint32_t>& counts) const {
  const uint32_t M = num_blocks();
  sums.assign(size_t(M) * cfg_.dim, 0.0);
  counts.assign(M, 0);
  check(C(ctx_), hisa_cuda_pool_read(C(ctx_), sums.data(), counts.data(), nullptr));
}

namespace {
struct DeviceQueries {
  const void* q;
  const float* gates;
  std::vector<uint16_t> bf16;
  std::vector<uint8_t> fp8;
  std::vector<float> scaled_gates;
};
DeviceQueries queries_for(const IndexerInputs& in, Storage st) {
  DeviceQueries d{in.queries_raw().data(), in.gates_raw().data(), {}, {}, {}};
  if (st == Storage::BF16) {
    d.bf16 = to_bf16(in.queries_raw());
    d.q = d.bf16.data();
  } else if (st == Storage::FP8) {
    // one scale per (query, head), folded into the gate: exact, a positive scale commutes with the ReLU (hisa_cuda.h)
    std::vector<float> sc;
    quantize_rows(in.queries_raw(), in.dim(), d.fp8, sc);
    d.scaled_gates = in.gates_raw();
    for (size_t i = 0; i < sc.size(); ++i) d.scaled_gates[i] *= sc[i];
    d.q = d.fp8.data();
    d.gates = d.scaled_gates.data();
  }
  return d;
}
void check_shapes(const IndexerInputs& in, const HisaConfig& cfg) {
  if (in.num_heads() != cfg.num_heads || in.dim() != cfg.dim)
    throw DimensionMismatch("inputs have H=" + std::to_string(in.num_heads()) + ", d=" + std::to_string(in.dim()) +
                            " but the config says H=" + std::to_string(cfg.num_heads) + ", d=" + std::to_string(cfg.dim));
}
}  // namespace

static std::vector<SelectionResult> run_select(Indexer& ix, void* ctx, const HisaConfig& cfg, Storage st,
                                               Strategy strat, const IndexerInputs& in, OpCounter* counter) {
  check_shapes(in, cfg);
  const uint32_t Q = in.num_queries(), S = cfg.block_budget + 2;
  const uint32_t width = strat == Strategy::BlockSparse ? S * cfg.block_size : cfg.token_budget;
  std::vector<int32_t> idx(size_t(Q) * width), blocks(size_t(Q) * S, -1);
  std::vector<uint32_t> count(Q), nblocks(Q, 0), cand(Q, 0);
  const DeviceQueries dq = queries_for(in, st);
  int rc;
  if (strat == Strategy::Hisa)
    rc = hisa_cuda_hisa_select(C(ctx), dq.q, dq.gates, in.positions_raw().data(), Q, 0, idx.data(),
                               count.data(), blocks.data(), nblocks.data(), cand.data());
  else if (strat == Strategy::Dsa)
    rc = hisa_cuda_dsa_select(C(ctx), dq.q, dq.gates, in.positions_raw().data(), Q, 0, idx.data(),
                              count.data(), cand.data());
  else
    rc = hisa_cuda_block_sparse_select(C(ctx), dq.q, dq.gates, in.positions_raw().data(), Q, 0,
                                       idx.data(), count.data(), blocks.data(), nblocks.data());
  check(C(ctx), rc);
  std::vector<SelectionResult> out(Q);
  const uint64_t H = cfg.num_heads, B = cfg.block_size;
  for (uint32_t r = 0; r < Q; ++r) {
    SelectionResult& s = out[r];
    s.token_indices.assign(idx.begin() + size_t(r) * width, idx.begin() + size_t(r) * width + count[r]);
    if (strat != Strategy::Dsa) s.selected_blocks.assign(blocks.begin() + size_t(r) * S, blocks.begin() + size_t(r) * S + nblocks[r]);
    s.candidate_size = strat == Strategy::BlockSparse ? count[r] : cand[r];
    if (counter) {
      const uint64_t t = std::min(in.position(r), in.seq_len() - 1);
      const uint64_t eligible = std::min<uint64_t>(t / B, uint64_t(ix.num_blocks()) - 1) + 1;
      if (strat != Strategy::Dsa) { counter->dot_products += H * eligible; counter->comparisons += eligible; }
      if (strat != Strategy::BlockSparse) { counter->dot_products += H * s.candidate_size; counter->comparisons += s.candidate_size; }
    }
  }
  return out;
}

std::vector<SelectionResult> Indexer::hisa_select_batch(const IndexerInputs& in, OpCounter* c) {
  return run_select(*this, ctx_, cfg_, storage_, Strategy::Hisa, in, c);
}
std::vector<SelectionResult> Indexer::dsa_select_batch(const IndexerInputs& in, OpCounter* c) {
  return run_select(*this, ctx_, cfg_, storage_, Strategy::Dsa, in, c);
}
std::vector<SelectionResult> Indexer::block_sparse_select_batch(const IndexerInputs& in, OpCounter* c) {
  return run_select(*this, ctx_, cfg_, storage_, Strategy::BlockSparse, in, c);
}

std::vector<ScoreVector> Indexer::score_blocks_batch(const IndexerInputs& in) {
  check_shapes(in, cfg_);
  const uint32_t Q = in.num_queries(), M = num_blocks();
  std::vector<float> J(size_t(Q) * std::max(M, 1u));
  std::vector<uint32_t> ne(Q);
  const DeviceQueries dq = queries_for(in, storage_);
  check(C(ctx_), hisa_cuda_score_blocks(C(ctx_), dq.q, dq.gates, in.positions_raw().data(), Q, J.data(), ne.data()));
  std::vector<ScoreVector> out(Q);
  for (uint32_t r = 0; r < Q; ++r) {
    out[r].scores.assign(J.begin() + size_t(r) * M, J.begin() + size_t(r) * M + ne[r]);
    out[r].positions.resize(ne[r]);
    std::iota(out[r].positions.begin(), out[r].positions.end(), 0u);
  }
  return out;
}

std::vector<ScoreVector> Indexer::score_prefix_batch(const IndexerInputs& in) {
  check_shapes(in, cfg_);
  const uint32_t Q = in.num_queries(), L = seq_len();
  const uint64_t stride = (uint64_t(L) + 127) / 128 * 128;
  std::vector<float> S(size_t(Q) * stride);
  const DeviceQueries dq = queries_for(in, storage_);
  check(C(ctx_), hisa_cuda_score_tokens(C(ctx_), dq.q, dq.gates, in.positions_raw().data(), Q, S.data(), stride));
  std::vector<ScoreVector> out(Q);
  for (uint32_t r = 0; r < Q; ++r) {
    const uint32_t n = std::min(in.position(r), L - 1) + 1;
    out[r].scores.assign(S.begin() + size_t(r) * stride, S.begin() + size_t(r) * stride + n);
    out[r].positions.resize(n);
    std::iota(out[r].positions.begin(), out[r].positions.end(), 0u);
  }
  return out;
}

void Indexer::enable_timing(bool on) { check(C(ctx_), hisa_cuda_set_profiling(C(ctx_), on ? 1 : 0)); }
Indexer::Times Indexer::last_times() {
  hisa_cuda_stage_times t;
  check(C(ctx_), hisa_cuda_last_stage_times(C(ctx_), &t));
  return Times{t.score_blocks_ms, t.select_blocks_ms, t.invert_ms, t.score_tokens_ms, t.top_k_ms, t.total_ms};
}

}  // namespace gpu

// ==================================================================================================
// the reference's per-row entry points: thin views over batched device calls
// ==================================================================================================
namespace {

using detail::hash_bytes;
template <class T>
uint64_t hash_vec(const std::vector<T>& v, uint64_t seed) { return hash_bytes(v.data(), v.size() * sizeof(T), seed); }

// One device context + the batched results per (inputs CONTENT, cache CONTENT, config): a caller looping
// `for row: select(row)` (the reference's run_bench, audits, NIAH grid) triggers ONE batched launch, later rows are
// served from the entry. The key is a hash of the full payload, never an object address: a new IndexerInputs built at
// the address of a destroyed one (same sizes, different needle) must not be served the old results. Hashing costs
// O(payload) per call; bulk callers use gpu::Indexer directly.
struct RowCacheKey {
  uint64_t h_inputs, h_cache;
  uint32_t Q, L, H, d, B, m, k, cache_tokens;
  uint32_t ffl, fib, tb, pm;
  bool operator<(const RowCacheKey& o) const { return std::memcmp(this, &o, sizeof *this) < 0; }
};
struct RowCacheEntry {
  std::mutex mu;  // held across lookup, batched launch, insertion and copy-out: rows may be fanned out over threads
  std::unique_ptr<gpu::Indexer> ix;
  std::map<int, std::vector<SelectionResult>> results;  // by Strategy
  std::vector<ScoreVector> block_scores, prefix_scores;
};
std::mutex g_cache_mu;
std::map<RowCacheKey, std::shared_ptr<RowCacheEntry>> g_cache;
std::vector<RowCacheKey> g_cache_order;  // insertion order: the oldest entry is evicted first
constexpr size_t kMaxCached = 4;
constexpr uint64_t kMaxCachedEntries = 1ull << 27;  // beyond this many result integers, rows are launched one by one

uint64_t hash_inputs(const IndexerInputs& in) {
  uint64_t h = hash_vec(in.keys_raw(), 1);
  h = hash_vec(in.queries_raw(), h);
  h = hash_vec(in.gates_raw(), h);
  return hash_vec(in.positions_raw(), h);
}
uint64_t hash_cache(const BlockSummaryCache& cache) {
  const uint64_t h = hash_vec(cache.*member_of(SummaryTag{}), 2);
  return hash_vec(cache.*member_of(CountsTag{}), h);
}

// `cache` == nullptr: strategies that do not read block summaries (dsa_select, score_tokens)
std::shared_ptr<RowCacheEntry> entry_for(const IndexerInputs& in, const BlockSummaryCache* cache, const HisaConfig& cfg) {
  RowCacheKey key;
  std::memset(&key, 0, sizeof key);
  key.h_inputs = hash_inputs(in);
  key.h_cache = cache ? hash_cache(*cache) : 0;
  key.cache_tokens = cache ? cache->num_tokens() : 0;
  key.Q = in.num_queries(); key.L = in.seq_len(); key.H = cfg.num_heads; key.d = cfg.dim;
  key.B = cfg.block_size; key.m = cfg.block_budget; key.k = cfg.token_budget;
  key.ffl = cfg.force_first_last; key.fib = cfg.forced_in_budget;
  key.tb = uint32_t(cfg.tie_break); key.pm = uint32_t(cfg.pool_mode);
  std::lock_guard<std::mutex> g(g_cache_mu);
  auto it = g_cache.find(key);
  if (it != g_cache.end()) return it->second;
  if (in.seq_len() == 0) throw EmptySequence("selection over an empty key sequence");
  auto e = std::make_shared<RowCacheEntry>();
  e->ix = std::make_unique<gpu::Indexer>(cfg, gpu::Storage::F32);
  e->ix->set_keys(in.keys_raw());
  // the block scores come from the CALLER'S cache (its contents and its length), not from re-pooling the inputs
  if (cache) e->ix->set_summaries(*cache);
  if (g_cache.size() >= kMaxCached) {
    g_cache.erase(g_cache_order.front());
    g_cache_order.erase(g_cache_order.begin());
  }
  g_cache[key] = e;
  g_cache_order.push_back(key);
  return e;
}

IndexerInputs single_row(const IndexerInputs& in, uint32_t row) {
  const size_t hd = size_t(in.num_heads()) * in.dim();
  std::vector<float> q(in.queries_raw().begin() + row * hd, in.queries_raw().begin() + (row + 1) * hd);
  std::vector<float> w(in.gates_raw().begin() + size_t(row) * in.num_heads(),
                       in.gates_raw().begin() + size_t(row + 1) * in.num_heads());
  return IndexerInputs(std::move(q), std::move(w), in.keys_raw(), {in.position(row)}, in.num_heads(), in.dim());
}

SelectionResult select_row(Strategy strat, const IndexerInputs& in, const BlockSummaryCache* cache, const HisaConfig& cfg,
                           uint32_t row, OpCounter* counter) {
  if (row >= in.num_queries()) throw Error("query row " + std::to_string(row) + " out of range");
  if (in.num_heads() != cfg.num_heads || in.dim() != cfg.dim)
    throw DimensionMismatch("inputs and config disagree on num_heads / dim");
  auto e = entry_for(in, cache, cfg);
  const uint64_t width = strat == Strategy::BlockSparse ? uint64_t(cfg.block_budget + 2) * cfg.block_size : cfg.token_budget;
  SelectionResult r;
  uint32_t summary_blocks;
  {
    std::lock_guard<std::mutex> g(e->mu);
    summary_blocks = e->ix->num_blocks();
    if (uint64_t(in.num_queries()) * width <= kMaxCachedEntries) {
      auto it = e->results.find(int(strat));
      if (it == e->results.end()) {
        std::vector<SelectionResult> all = strat == Strategy::Hisa  ? e->ix->hisa_select_batch(in)
                                           : strat == Strategy::Dsa ? e->ix->dsa_select_batch(in)
                                                                    : e->ix->block_sparse_select_batch(in);
        it = e->results.emplace(int(strat), std::move(all)).first;
      }
      r = it->second[row];
    } else {
      const IndexerInputs one = single_row(in, row);
      r = (strat == Strategy::Hisa  ? e->ix->hisa_select_batch(one)
           : strat == Strategy::Dsa ? e->ix->dsa_select_batch(one)
                                    : e->ix->block_sparse_select_batch(one))[0];
    }
  }
  if (counter) {
    const uint64_t H = cfg.num_heads, B = cfg.block_size;
    const uint64_t t = std::min(in.position(row), in.seq_len() - 1);
    const uint64_t eligible = std::min<uint64_t>(t / B, uint64_t(summary_blocks) - 1) + 1;
    if (strat != Strategy::Dsa) { counter->dot_products += H * eligible; counter->comparisons += eligible; }
    if (strat != Strategy::BlockSparse) { counter->dot_products += H * r.candidate_size; counter->comparisons += r.candidate_size; }
  }
  return r;
}

void check_cache_matches(const IndexerInputs& in, const BlockSummaryCache& cache, const HisaConfig& cfg) {
  if (cache.dim() != in.dim()) throw DimensionMismatch("block summary cache dimension differs from the inputs");
  if (cache.block_size() != cfg.block_size) throw Error("block summary cache block size differs from the config");
  if (cache.num_blocks() == 0) throw EmptySequence("score_blocks: empty block summary cache");
}

}  // namespace

ScoreVector score_tokens(const IndexerInputs& in, uint32_t row, std::span<const uint32_t> candidates, OpCounter* counter) {
  if (row >= in.num_queries()) throw Error("score_tokens: query row out of range");
  const uint32_t t = in.position(row);
  uint32_t prev = 0;
  for (size_t i = 0; i < candidates.size(); ++i) {
    if (candidates[i] > t)
      throw CausalViolation("score_tokens: candidate " + std::to_string(candidates[i]) + " exceeds query position " + std::to_string(t));
    if (candidates[i] >= in.seq_len())
      throw CausalViolation("score_tokens: candidate " + std::to_string(candidates[i]) + " is outside the key sequence");
    if (i && candidates[i] <= prev) throw Error("score_tokens: candidates must be strictly ascending");
    prev = candidates[i];
  }
  HisaConfig cfg(1, 1, 1, in.num_heads(), in.dim());
  auto e = entry_for(in, nullptr, cfg);
  ScoreVector out;
  out.positions.assign(candidates.begin(), candidates.end());
  out.scores.resize(candidates.size());
  {
    std::lock_guard<std::mutex> g(e->mu);
    if (e->prefix_scores.empty() && uint64_t(in.num_queries()) * in.seq_len() <= kMaxCachedEntries)
      e->prefix_scores = e->ix->score_prefix_batch(in);
    if (!e->prefix_scores.empty()) {
      const ScoreVector& all = e->prefix_scores[row];
      for (size_t i = 0; i < candidates.size(); ++i) out.scores[i] = all.scores[candidates[i]];
    } else {
      const ScoreVector all = e->ix->score_prefix_batch(single_row(in, row))[0];
      for (size_t i = 0; i < candidates.size(); ++i) out.scores[i] = all.scores[candidates[i]];
    }
  }
  if (counter) counter->dot_products += uint64_t(in.num_heads()) * candidates.size();
  return out;
}

namespace {
gpu::Indexer& scratch_indexer(const HisaConfig& cfg) {
  static thread_local std::unique_ptr<gpu::Indexer> ix;
  static thread_local HisaConfig last(1, 1, 1, 1, 1);
  const bool same = last.block_size == cfg.block_size && last.block_budget == cfg.block_budget &&
                    last.token_budget == cfg.token_budget && last.num_heads == cfg.num_heads && last.dim == cfg.dim &&
                    last.force_first_last == cfg.force_first_last && last.forced_in_budget == cfg.forced_in_budget &&
                    last.tie_break == cfg.tie_break && last.pool_mode == cfg.pool_mode;
  if (!ix || !same) {
    ix = std::make_unique<gpu::Indexer>(cfg, gpu::Storage::F32);
    last = cfg;
  }
  return *ix;
}

// The `keep` best entries of `scores` under (score descending, then index ascending for SmallestIndex / descending for
// LargestIndex), as ascending indices. The device selects on fp32 keys; rounding double -> float is monotone, so every
// entry whose float key is above the smallest selected float key is selected whatever the doubles say, and only the
// entries that SHARE that boundary float key can be ordered differently by the doubles: that class is re-ranked here in
// double, which makes the result the reference's full-order contract for arbitrary double scores (dsa.hpp:22-27).
std::vector<uint32_t> device_best(std::span<const double> scores, uint32_t keep, TieBreak tie_break) {
  const uint32_t n = uint32_t(scores.size());
  std::vector<uint32_t> out;
  if (n == 0 || keep == 0) return out;
  keep = std::min(keep, n);
  HisaConfig cfg(1, keep, keep, 1, 1);
  cfg.tie_break = tie_break;
  gpu::Indexer& ix = scratch_indexer(cfg);
  std::vector<float> s(scores.begin(), scores.end());
  std::vector<int32_t> idx(keep);
  uint32_t cnt = 0;
  check(C(ix.raw()), hisa_cuda_top_k(C(ix.raw()), s.data(), n, &n, 1, keep, idx.data(), &cnt));
  out.assign(idx.begin(), idx.begin() + cnt);
  if (cnt == n) return out;
  float boundary = s[out[0]];
  for (uint32_t i : out) boundary = std::min(boundary, s[i]);
  std::vector<uint32_t> cls, sure;
  for (uint32_t i = 0; i < n; ++i)
    if (s[i] == boundary) cls.push_back(i);
  for (uint32_t i : out)
    if (s[i] != boundary) sure.push_back(i);
  const size_t need = cnt - sure.size();
  if (cls.size() == need) return out;  // the whole class is selected: nothing the doubles could reorder
  std::stable_sort(cls.begin(), cls.end(), [&](uint32_t a, uint32_t b) {
    if (scores[a] != scores[b]) return scores[a] > scores[b];
    return tie_break == TieBreak::SmallestIndex ? a < b : a > b;
  });
  sure.insert(sure.end(), cls.begin(), cls.begin() + need);
  std::sort(sure.begin(), sure.end());
  return sure;
}
}  // namespace

SelectionResult top_k_tokens(const ScoreVector& sv, uint32_t k, TieBreak tie_break, OpCounter* counter) {
  if (sv.scores.size() != sv.positions.size()) throw ShapeMismatch("top_k_tokens: scores and positions differ in length");
  if (k == 0) throw Error("top_k_tokens: k must be at least 1");
  SelectionResult r;
  r.candidate_size = sv.scores.size();
  for (uint32_t i : device_best(sv.scores, k, tie_break)) r.token_indices.push_back(sv.positions[i]);  // positions ascend
  if (counter) counter->comparisons += sv.scores.size();
  return r;
}

std::vector<uint32_t> select_blocks(const ScoreVector& js, const HisaConfig& cfg, uint32_t query_position, OpCounter* counter) {
  const uint32_t n = uint32_t(js.scores.size());
  if (n == 0) throw EmptySelection("select_blocks: no eligible block");
  if (js.positions.size() != n) throw ShapeMismatch("select_blocks: scores and positions differ in length");
  // forced blocks (hisa.hpp:23-28): the first eligible one and the one containing the query, which is the last
  // eligible one when the score vector stops short of it (a cache shorter than the inputs, or t == L)
  std::vector<char> keep(n, 0), forced(n, 0);
  if (cfg.force_first_last) {
    forced[0] = 1;
    uint32_t li = n - 1;
    const uint32_t local = query_position / cfg.block_size;
    for (uint32_t i = 0; i < n; ++i)
      if (js.positions[i] == local) li = i;
    forced[li] = 1;
  }
  if (cfg.force_first_last && cfg.forced_in_budget) {
    // forced blocks first, the rest of the budget by score among the others (config.hpp:57-63)
    std::vector<double> rest;
    std::vector<uint32_t> back;
    uint32_t used = 0;
    for (uint32_t i = 0; i < n; ++i) {
      if (forced[i]) { keep[i] = 1; ++used; }
      else { rest.push_back(js.scores[i]); back.push_back(i); }
    }
    const uint32_t room = cfg.block_budget > used ? cfg.block_budget - used : 0;
    for (uint32_t i : device_best(rest, room, cfg.tie_break)) keep[back[i]] = 1;
  } else {
    for (uint32_t i : device_best(js.scores, cfg.block_budget, cfg.tie_break)) keep[i] = 1;
    for (uint32_t i = 0; i < n; ++i)
      if (forced[i]) keep[i] = 1;
  }
  std::vector<uint32_t> out;
  for (uint32_t i = 0; i < n; ++i)
    if (keep[i]) out.push_back(js.positions[i]);
  if (counter) counter->comparisons += n;
  return out;
}

SelectionResult dsa_select(const IndexerInputs& in, const HisaConfig& cfg, uint32_t row, OpCounter* counter) {
  return select_row(Strategy::Dsa, in, nullptr, cfg, row, counter);
}

ScoreVector score_blocks(const IndexerInputs& in, const BlockSummaryCache& cache, uint32_t row, OpCounter* counter) {
  if (row >= in.num_queries()) throw Error("score_blocks: query row out of range");
  HisaConfig cfg(cache.block_size(), 1, 1, in.num_heads(), in.dim());
  cfg.pool_mode = cache.pool_mode();
  check_cache_matches(in, cache, cfg);
  auto e = entry_for(in, &cache, cfg);
  std::lock_guard<std::mutex> g(e->mu);
  if (e->block_scores.empty()) e->block_scores = e->ix->score_blocks_batch(in);
  if (counter) counter->dot_products += uint64_t(in.num_heads()) * e->block_scores[row].scores.size();
  return e->block_scores[row];
}

SelectionResult hisa_select(const IndexerInputs& in, const BlockSummaryCache& cache, const HisaConfig& cfg, uint32_t row,
                            OpCounter* counter) {
  check_cache_matches(in, cache, cfg);
  HisaConfig c2 = cfg;
  c2.pool_mode = cache.pool_mode();  // the summaries are what they are, whatever the config says
  return select_row(Strategy::Hisa, in, &cache, c2, row, counter);
}

SelectionResult block_sparse_select(const IndexerInputs& in, const BlockSummaryCache& cache, const HisaConfig& cfg,
                                    uint32_t row, OpCounter* counter) {
  check_cache_matches(in, cache, cfg);
  HisaConfig c2 = cfg;
  c2.pool_mode = cache.pool_mode();
  return select_row(Strategy::BlockSparse, in, &cache, c2, row, counter);
}

// ==================================================================================================
// bench harness (hisa/bench.hpp:47-58): same record, timing = device time of the batched call
// ==================================================================================================
BenchRecord run_bench(const HisaConfig& cfg, uint32_t seq_len, uint32_t num_queries, uint64_t seed, Strategy strategy,
                      const BenchOptions& opt) {
  return gpu::run_bench(cfg, seq_len, num_queries, seed, strategy, opt, gpu::Storage::F32);
}

BenchRecord gpu::run_bench(const HisaConfig& cfg, uint32_t seq_len, uint32_t num_queries, uint64_t seed, Strategy strategy,
                           const BenchOptions& opt, Storage storage, TimeBase time_base) {
  Rng rng(seed);
  const IndexerInputs in = make_random_inputs(rng, seq_len, num_queries, cfg.num_heads, cfg.dim, opt.placement);
  gpu::Indexer ix(cfg, storage);
  ix.enable_timing(true);
  ix.set_keys(in.keys_raw());
  BenchRecord rec;
  rec.strategy = strategy;
  rec.seq_len = seq_len; rec.block_size = cfg.block_size; rec.block_budget = cfg.block_budget;
  rec.token_budget = cfg.token_budget; rec.num_heads = cfg.num_heads; rec.dim = cfg.dim; rec.queries = num_queries;
  // summary build time, reported separately and never part of the per-query timing (bench.hpp:28, :51-52)
  rec.pool_build_ns = std::max<uint64_t>(1, uint64_t(double(ix.last_pool_build_ms()) * 1e6));
  auto once = [&](OpCounter* c) {
    if (strategy == Strategy::Dsa) ix.dsa_select_batch(in, c);
    else if (strategy == Strategy::Hisa) ix.hisa_select_batch(in, c);
    else ix.block_sparse_select_batch(in, c);
    const auto t = ix.last_times();
    if (time_base == TimeBase::Kernels)
      return t.score_blocks_ms + t.select_blocks_ms + t.invert_ms + t.score_tokens_ms + t.top_k_ms;
    return t.total_ms;
  };
  if (opt.timing) {
    for (uint32_t i = 0; i < opt.warmup; ++i) once(nullptr);
    std::vector<double> ms;
    for (uint32_t i = 0; i < std::max(1u, opt.repetitions); ++i) ms.push_back(once(nullptr));
    std::sort(ms.begin(), ms.end());
    auto pick = [&](double f) { return uint64_t(ms[size_t(f * double(ms.size() - 1) + 0.5)] * 1e6); };
    rec.wall_ns_median = std::max<uint64_t>(1, pick(0.5));
    rec.wall_ns_p10 = pick(0.1);
    rec.wall_ns_p90 = pick(0.9);
  }
  OpCounter c;
  once(&c);  // instrumented pass, untimed (hisa/bench.hpp:29)
  rec.dot_products = c.dot_products;
  for (uint32_t r = 0; r < num_queries; ++r)
    rec.analytic_bound += analytic_cost(cfg, uint64_t(std::min(in.position(r), seq_len - 1)) + 1, strategy);
  return rec;
}

void write_bench_csv(std::ostream& os, const std::vector<BenchRecord>& records) {
  os << "strategy,L,B,m,k,H,d,wall_ns_median,wall_ns_p10,wall_ns_p90,dot_products,analytic_bound\n";
  for (const BenchRecord& r : records)
    os << to_string(r.strategy) << ',' << r.seq_len << ',' << r.block_size << ',' << r.block_budget << ',' << r.token_budget
       << ',' << r.num_heads << ',' << r.dim << ',' << r.wall_ns_median << ',' << r.wall_ns_p10 << ',' << r.wall_ns_p90
       << ',' << r.dot_products << ',' << r.analytic_bound << '\n';
}

namespace gpu {
// Fig. 2's two panels (SPEC.md:462 `bench --mode fixed-budget | ratio`)
std::vector<BenchRecord> run_bench_sweep(const HisaConfig& cfg, std::span<const uint32_t> lengths, uint32_t num_queries,
                                         uint64_t seed, std::span<const Strategy> strategies, SweepMode mode, uint32_t ratio,
                                         const BenchOptions& options, Storage storage, TimeBase time_base) {
  if (mode == SweepMode::Ratio && ratio == 0) throw Error("run_bench_sweep: ratio must be at least 1");
  std::vector<BenchRecord> out;
  for (uint32_t L : lengths) {
    uint32_t m = cfg.block_budget;
    if (mode == SweepMode::Ratio) {
      const uint32_t M = (L + cfg.block_size - 1) / cfg.block_size;
      m = std::max<uint32_t>(1, (M + ratio - 1) / ratio);
      m = std::max<uint32_t>(m, (cfg.token_budget + cfg.block_size - 1) / cfg.block_size);  // keep m*B >= k
    }
    HisaConfig c(cfg.block_size, m, cfg.token_budget, cfg.num_heads, cfg.dim);
    c.force_first_last = cfg.force_first_last;
    c.forced_in_budget = cfg.forced_in_budget;
    c.tie_break = cfg.tie_break;
    c.pool_mode = cfg.pool_mode;
    for (Strategy s : strategies) out.push_back(gpu::run_bench(c, L, num_queries, seed, s, options, storage, time_base));
  }
  return out;
}
}  // namespace gpu

}  // namespace hisa
