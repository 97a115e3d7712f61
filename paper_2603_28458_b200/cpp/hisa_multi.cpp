// C++ host layer, part 4: the multi-GPU driver (rows are independent, so the reference
// fans them out over workers — hisa/parallel.hpp:15-19 — and here the workers are GPUs). Host code only: the sharding
// plan, NCCL and the peer-store gather live behind hisa_cuda_dist_* in the CUDA library.
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

#include "hisa/config.hpp"
#include "hisa/errors.hpp"
#include "hisa/inputs.hpp"
#include "hisa/types.hpp"
#include "hisa_cuda.h"
#include "hisa_gpu.hpp"
#include "host_util.hpp"

namespace hisa::gpu {

namespace {
hisa_cuda_dist* D(void* p) { return static_cast<hisa_cuda_dist*>(p); }
[[noreturn]] void raise_dist(int status, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (status) {
    case HISA_ERR_INFEASIBLE_CONFIG: throw InfeasibleConfig(m);
    case HISA_ERR_EMPTY_SEQUENCE: throw EmptySequence(m);
    case HISA_ERR_DIMENSION_MISMATCH: throw DimensionMismatch(m);
    case HISA_ERR_NON_FINITE: throw NonFiniteValue(m);
    case HISA_ERR_SHAPE_MISMATCH: throw ShapeMismatch(m);
    default: throw Error(std::string(hisa_cuda_status_name(status)) + ": " + m);
  }
}
void check(void* d, int status) {
  if (status != HISA_OK) raise_dist(status, hisa_cuda_dist_last_error(D(d)));
}
}  // namespace

std::vector<uint32_t> MultiIndexer::rank_rows(uint64_t num_rows, int world, int rank) {
  uint64_t n = 0;
  int rc = hisa_cuda_dist_plan(num_rows, world, rank, &n, nullptr);
  if (rc != HISA_OK) raise_dist(rc, hisa_cuda_dist_last_error(nullptr));
  std::vector<uint32_t> rows(n);
  rc = hisa_cuda_dist_plan(num_rows, world, rank, &n, rows.data());
  if (rc != HISA_OK) raise_dist(rc, hisa_cuda_dist_last_error(nullptr));
  return rows;
}

MultiIndexer::MultiIndexer(const HisaConfig& cfg, Storage storage, std::vector<int> devices, Gather gather)
    : cfg_(cfg), storage_(storage) {
  if (storage == Storage::FP8) throw Error("MultiIndexer: bf16 or f32 storage");
  hisa_cuda_config c;
  hisa_cuda_config_init(&c, cfg.block_size, cfg.block_budget, cfg.token_budget, cfg.num_heads, cfg.dim,
                        storage == Storage::BF16 ? HISA_DTYPE_BF16 : HISA_DTYPE_F32);
  c.force_first_last = cfg.force_first_last;
  c.forced_in_budget = cfg.forced_in_budget;
  c.tie_break = cfg.tie_break == TieBreak::LargestIndex ? HISA_TIE_LARGEST_INDEX : HISA_TIE_SMALLEST_INDEX;
  c.pool_mode = cfg.pool_mode == PoolMode::Max ? HISA_POOL_MAX : HISA_POOL_MEAN;
  hisa_cuda_dist* d = nullptr;
  const int rc = hisa_cuda_dist_create(devices.data(), int(devices.size()), &c, uint32_t(gather), &d);
  if (rc != HISA_OK) raise_dist(rc, hisa_cuda_dist_last_error(nullptr));
  dist_ = d;
  int g = 0;
  hisa_cuda_dist_info(d, &world_, nullptr, nullptr, &g);
  gather_ = Gather(g);
}

MultiIndexer::~MultiIndexer() {
  if (dist_) hisa_cuda_dist_destroy(D(dist_));
}

void MultiIndexer::set_keys(std::span<const float> keys) {
  if (keys.size() % cfg_.dim != 0) throw ShapeMismatch("set_keys: keys size is not a multiple of dim");
  const uint64_t L = keys.size() / cfg_.dim;
  if (storage_ == Storage::BF16) {
    const auto b = detail::to_bf16(keys);
    check(dist_, hisa_cuda_dist_upload_keys(D(dist_), b.data(), nullptr, L, 0));
  } else {
    check(dist_, hisa_cuda_dist_upload_keys(D(dist_), keys.data(), nullptr, L, 0));
  }
}

std::vector<SelectionResult> MultiIndexer::run(int strategy, const IndexerInputs& in, int num_slices) {
  if (in.num_heads() != cfg_.num_heads || in.dim() != cfg_.dim) throw DimensionMismatch("inputs and config disagree on num_heads / dim");
  const uint32_t Q = in.num_queries(), H = cfg_.num_heads, k = cfg_.token_budget;
  const size_t hd = size_t(H) * cfg_.dim;
  // scatter the rows to their owners (host side: the inputs live in host vectors)
  const size_t G = size_t(world_);
  std::vector<std::vector<float>> q(G), w(G);
  std::vector<std::vector<uint16_t>> qb(G);
  std::vector<std::vector<uint32_t>> pos(G);
  std::vector<const void*> qp(G);
  std::vector<const float*> wp(G);
  std::vector<const uint32_t*> pp(G);
  for (int r = 0; r < world_; ++r) {
    const std::vector<uint32_t> rows = rank_rows(Q, world_, r);
    auto& qr = q[size_t(r)];
    auto& wr = w[size_t(r)];
    auto& pr = pos[size_t(r)];
    qr.resize(rows.size() * hd);
    wr.resize(rows.size() * H);
    pr.resize(rows.size());
    for (size_t i = 0; i < rows.size(); ++i) {
      std::memcpy(&qr[i * hd], &in.queries_raw()[size_t(rows[i]) * hd], hd * sizeof(float));
      std::memcpy(&wr[i * H], &in.gates_raw()[size_t(rows[i]) * H], H * sizeof(float));
      pr[i] = in.position(rows[i]);
    }
    if (storage_ == Storage::BF16) {
      qb[size_t(r)] = detail::to_bf16(qr);
      qp[size_t(r)] = qb[size_t(r)].data();
    } else {
      qp[size_t(r)] = qr.data();
    }
    wp[size_t(r)] = wr.data();
    pp[size_t(r)] = pr.data();
  }
  check(dist_, hisa_cuda_dist_select(D(dist_), strategy, qp.data(), wp.data(), pp.data(), Q, num_slices));
  std::vector<int32_t> idx(size_t(Q) * k);
  std::vector<uint32_t> cnt(Q);
  check(dist_, hisa_cuda_dist_fetch(D(dist_), 0, idx.data(), cnt.data()));
  std::vector<SelectionResult> out(Q);
  for (uint32_t r = 0; r < Q; ++r) out[r].token_indices.assign(idx.begin() + size_t(r) * k, idx.begin() + size_t(r) * k + cnt[r]);
  return out;
}

std::vector<SelectionResult> MultiIndexer::hisa_select_batch(const IndexerInputs& in, int num_slices) {
  return run(HISA_DIST_HISA, in, num_slices);
}
std::vector<SelectionResult> MultiIndexer::dsa_select_batch(const IndexerInputs& in, int num_slices) {
  return run(HISA_DIST_DSA, in, num_slices);
}

float MultiIndexer::last_ms() {
  float ms = 0.f;
  check(dist_, hisa_cuda_dist_last_ms(D(dist_), &ms));
  return ms;
}

}  // namespace hisa::gpu
