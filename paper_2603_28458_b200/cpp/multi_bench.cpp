// hisa_multi_bench — the multi-GPU driver program (SURVEY §1 "NCCL only in the multi-GPU driver", §8e): one process,
// one host thread + context + stream per GPU (inside hisa_cuda_dist_*), keys replicated by ncclBroadcast, query rows
// dealt in zig-zag tiles, index rows gathered to every GPU. Host code only (C++ over the C ABI, no CUDA header).
//
//   hisa_multi_bench --gpus 8 [--devices 0,1,..] [--seq-len 131072] [--block-size 128] [--block-budget 64]
//                    [--token-budget 2048] [--steps 10] [--warmup 3] [--gather auto|nccl|peer] [--strategy hisa|dsa]
//                    [--slices 4] [--check]
// Prints one JSON line: whole-job queries/s (strong scaling: the workload is fixed, the GPUs share it).
// --check additionally runs the same rows on ONE GPU and requires the gathered matrix to equal it bit for bit.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "hisa_cuda.h"

namespace {

struct Args {
  int gpus = 1;
  std::vector<int> devices;
  uint64_t L = 131072;
  uint32_t B = 128, m = 64, k = 2048, H = 64, d = 128;
  int steps = 10, warmup = 3, slices = 4;
  std::string gather = "auto", strategy = "hisa";
  bool check = false;
  uint64_t seed = 1;
};

[[noreturn]] void die(const char* what, const char* detail) {
  std::fprintf(stderr, "hisa_multi_bench: %s: %s\n", what, detail ? detail : "");
  std::exit(1);
}

// xorshift64* -> bf16 bit patterns of roughly N(0,1) values (sum of four uniforms, variance-corrected)
struct Gen {
  uint64_t s;
  uint64_t next() {
    s ^= s >> 12;
    s ^= s << 25;
    s ^= s >> 27;
    return s * 0x2545F4914F6CDD1DULL;
  }
  float normalish() {
    const uint64_t r = next();
    const float u = float(r & 0xFFFF) + float((r >> 16) & 0xFFFF) + float((r >> 32) & 0xFFFF) + float(r >> 48);
    return (u * (1.0f / 65536.0f) - 2.0f) * 1.7320508f;
  }
  float uniform() { return float(next() >> 40) * (1.0f / 16777216.0f); }
};
uint16_t bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return uint16_t((u + ((u >> 16) & 1u) + 0x7FFFu) >> 16);
}

void* dev_alloc(hisa_cuda_ctx* ctx, size_t bytes) {
  void* p = nullptr;
  if (hisa_cuda_device_alloc(ctx, &p, bytes) != HISA_OK) die("device allocation", hisa_cuda_last_error(ctx));
  return p;
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  for (int i = 1; i < argc; ++i) {
    const std::string f = argv[i];
    auto val = [&]() -> const char* {
      if (i + 1 >= argc) die("missing value for", f.c_str());
      return argv[++i];
    };
    if (f == "--gpus") a.gpus = std::atoi(val());
    else if (f == "--devices") {
      std::string s = val();
      size_t p = 0;
      while (p < s.size()) {
        a.devices.push_back(std::atoi(s.c_str() + p));
        p = s.find(',', p);
        if (p == std::string::npos) break;
        ++p;
      }
    } else if (f == "--seq-len") a.L = std::strtoull(val(), nullptr, 10);
    else if (f == "--block-size") a.B = uint32_t(std::atoi(val()));
    else if (f == "--block-budget") a.m = uint32_t(std::atoi(val()));
    else if (f == "--token-budget") a.k = uint32_t(std::atoi(val()));
    else if (f == "--steps") a.steps = std::atoi(val());
    else if (f == "--warmup") a.warmup = std::atoi(val());
    else if (f == "--slices") a.slices = std::atoi(val());
    else if (f == "--gather") a.gather = val();
    else if (f == "--strategy") a.strategy = val();
    else if (f == "--seed") a.seed = std::strtoull(val(), nullptr, 10);
    else if (f == "--check") a.check = true;
    else die("unknown flag", f.c_str());
  }
  if (a.devices.empty())
    for (int i = 0; i < a.gpus; ++i) a.devices.push_back(i);
  const int G = int(a.devices.size());
  const uint32_t flags = a.gather == "nccl" ? HISA_DIST_GATHER_NCCL : a.gather == "peer" ? HISA_DIST_GATHER_PEER : HISA_DIST_GATHER_AUTO;
  const int strategy = a.strategy == "dsa" ? HISA_DIST_DSA : HISA_DIST_HISA;

  hisa_cuda_config cfg;
  hisa_cuda_config_init(&cfg, a.B, a.m, a.k, a.H, a.d, HISA_DTYPE_BF16);
  hisa_cuda_dist* dist = nullptr;
  if (hisa_cuda_dist_create(a.devices.data(), G, &cfg, flags, &dist) != HISA_OK) die("hisa_cuda_dist_create", hisa_cuda_dist_last_error(nullptr));
  int gather_used = 0;
  hisa_cuda_dist_info(dist, nullptr, nullptr, nullptr, &gather_used);

  // synthetic inputs: keys on the host (replicated by the driver), every rank's query rows generated for that rank
  const uint64_t Q = a.L;
  const size_t hd = size_t(a.H) * a.d;
  std::vector<uint16_t> keys(size_t(a.L) * a.d);
  {
    Gen g{a.seed * 0x9E3779B97F4A7C15ULL + 1};
    for (auto& v : keys) v = bf16(g.normalish());
  }
  if (hisa_cuda_dist_upload_keys(dist, keys.data(), nullptr, a.L, 0) != HISA_OK) die("upload_keys", hisa_cuda_dist_last_error(dist));

  std::vector<const void*> qp(static_cast<size_t>(G));
  std::vector<const float*> wp(static_cast<size_t>(G));
  std::vector<const uint32_t*> pp(static_cast<size_t>(G));
  std::vector<std::vector<uint32_t>> rows(static_cast<size_t>(G));
  for (int r = 0; r < G; ++r) {
    uint64_t n = 0;
    hisa_cuda_dist_plan(Q, G, r, &n, nullptr);
    rows[size_t(r)].resize(n);
    hisa_cuda_dist_plan(Q, G, r, &n, rows[size_t(r)].data());
    hisa_cuda_ctx* ctx = hisa_cuda_dist_ctx(dist, r);
    void* dq = dev_alloc(ctx, n * hd * 2);
    void* dw = dev_alloc(ctx, n * a.H * 4);
    void* dp = dev_alloc(ctx, n * 4);
    // a row's values depend on the ROW only (seeded by its global index): any sharding sees the same tensors
    const size_t chunk = 4096;
    std::vector<uint16_t> hq(chunk * hd);
    std::vector<float> hw(chunk * a.H);
    for (size_t r0 = 0; r0 < n; r0 += chunk) {
      const size_t nr = std::min(chunk, size_t(n) - r0);
      for (size_t i = 0; i < nr; ++i) {
        Gen g{(a.seed + 7) * 0xD1342543DE82EF95ULL + rows[size_t(r)][r0 + i] * 0x9E3779B97F4A7C15ULL + 1};
        for (size_t e = 0; e < hd; ++e) hq[i * hd + e] = bf16(g.normalish());
        for (size_t e = 0; e < a.H; ++e) hw[i * a.H + e] = 0.5f + g.uniform();
      }
      hisa_cuda_memcpy(ctx, static_cast<char*>(dq) + r0 * hd * 2, hq.data(), nr * hd * 2);
      hisa_cuda_memcpy(ctx, static_cast<char*>(dw) + r0 * a.H * 4, hw.data(), nr * a.H * 4);
    }
    hisa_cuda_memcpy(ctx, dp, rows[size_t(r)].data(), n * 4);  // prefill: position = row
    qp[size_t(r)] = dq;
    wp[size_t(r)] = static_cast<const float*>(dw);
    pp[size_t(r)] = static_cast<const uint32_t*>(dp);
  }

  auto step = [&] {
    if (hisa_cuda_dist_select(dist, strategy, qp.data(), wp.data(), pp.data(), Q, a.slices) != HISA_OK)
      die("hisa_cuda_dist_select", hisa_cuda_dist_last_error(dist));
  };
  for (int i = 0; i < a.warmup; ++i) step();
  hisa_cuda_dist_synchronize(dist);
  double dev_ms = 0.0;
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < a.steps; ++i) {
    step();
    float ms = 0.f;
    hisa_cuda_dist_last_ms(dist, &ms);  // synchronises: device time of this step, maximum over the GPUs
    dev_ms += ms;
  }
  const double wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();

  int bit_equal = -1;
  if (a.check) {
    std::vector<int32_t> multi(size_t(Q) * a.k), single(size_t(Q) * a.k);
    if (hisa_cuda_dist_fetch(dist, G - 1, multi.data(), nullptr) != HISA_OK) die("fetch", hisa_cuda_dist_last_error(dist));
    // the same rows on ONE context, in global row order, host buffers
    hisa_cuda_ctx* one = nullptr;
    if (hisa_cuda_create(a.devices[0], &cfg, &one) != HISA_OK) die("hisa_cuda_create", hisa_cuda_last_error(nullptr));
    hisa_cuda_upload_keys(one, keys.data(), a.L, 0);
    hisa_cuda_pool_build(one);
    const size_t chunk = 4096;
    std::vector<uint16_t> hq(chunk * hd);
    std::vector<float> hw(chunk * a.H);
    std::vector<uint32_t> hp(chunk);
    for (size_t r0 = 0; r0 < Q; r0 += chunk) {
      const size_t nr = std::min(chunk, size_t(Q) - r0);
      for (size_t i = 0; i < nr; ++i) {
        Gen g{(a.seed + 7) * 0xD1342543DE82EF95ULL + (r0 + i) * 0x9E3779B97F4A7C15ULL + 1};
        for (size_t e = 0; e < hd; ++e) hq[i * hd + e] = bf16(g.normalish());
        for (size_t e = 0; e < a.H; ++e) hw[i * a.H + e] = 0.5f + g.uniform();
        hp[i] = uint32_t(r0 + i);
      }
      const int rc = strategy == HISA_DIST_HISA
                         ? hisa_cuda_hisa_select(one, hq.data(), hw.data(), hp.data(), nr, 0, single.data() + r0 * a.k, nullptr, nullptr, nullptr, nullptr)
                         : hisa_cuda_dsa_select(one, hq.data(), hw.data(), hp.data(), nr, 0, single.data() + r0 * a.k, nullptr, nullptr);
      if (rc != HISA_OK) die("single-GPU select", hisa_cuda_last_error(one));
    }
    hisa_cuda_destroy(one);
    bit_equal = std::memcmp(multi.data(), single.data(), multi.size() * 4) == 0 ? 1 : 0;
  }

  const double ms_step = dev_ms / a.steps;
  std::printf(
      "{\"metric\": \"indexer queries/sec (HISA hierarchical top-k, full causal prefill)\", \"value\": %.1f, \"unit\": \"queries/s\", "
      "\"n_gpus\": %d, \"steps\": %d, \"warmup\": %d, \"ms_per_step\": %.4f, \"wall_ms_per_step\": %.4f, \"higher_is_better\": true, "
      "\"scaling\": \"strong\", \"dtype\": \"bf16\", \"data\": \"synthetic\", \"driver\": \"C++ (hisa_multi_bench over hisa_cuda_dist_*)\", "
      "\"config\": {\"workload\": \"prefill L=Q=%llu H=%u d=%u B=%u m=%u k=%u bf16, %s_select, rows sharded in 512-row zig-zag tiles\", "
      "\"gather\": \"%s\", \"slices\": %d}, \"bit_equal_to_one_gpu\": %s}\n",
      double(Q) / (ms_step * 1e-3), G, a.steps, a.warmup, ms_step, wall_ms / a.steps, (unsigned long long)a.L, a.H, a.d, a.B, a.m, a.k,
      a.strategy.c_str(), gather_used == HISA_DIST_GATHER_PEER ? "peer stores from the top-k kernel" : "per-tile ncclBroadcast on a second stream",
      a.slices, bit_equal < 0 ? "null" : bit_equal ? "true" : "false");
  hisa_cuda_dist_destroy(dist);
  return bit_equal == 0 ? 2 : 0;
}
