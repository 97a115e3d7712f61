// hisa_fig2_sweep — the two panels of the paper's Fig. 2 on one B200 through the reference's bench harness
// (hisa::run_bench / BenchRecord / write_bench_csv, hisa/bench.hpp:16-58; SPEC.md `bench --mode fixed-budget | ratio`):
// per sequence length one record per strategy (flat DSA, block-sparse, HISA), 1024 queries at the newest position
// (QueryPlacement::Final, the paper's shape), B = 128, k = 2048; panel (a) keeps m = 64, panel (b) keeps M : m = 4 : 1.
//   hisa_fig2_sweep [--storage bf16|f32|fp8] [--queries 1024] [--max-len 131072] > fig2.csv
// Times are the device times of the indexer's kernels (gpu::TimeBase::Kernels: operands resident, as the paper times its
// kernels; median of 5 after one warm-up, pool build excluded, bench.hpp:51-52). --call-time reports the whole batched call
// instead, i.e. with the f32 host containers of IndexerInputs crossing PCIe, which dominates 1024-row calls.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <vector>

#include "hisa/bench.hpp"
#include "hisa_gpu.hpp"

int main(int argc, char** argv) {
  using namespace hisa;
  gpu::Storage storage = gpu::Storage::BF16;
  uint32_t queries = 1024, max_len = 131072;
  gpu::TimeBase base = gpu::TimeBase::Kernels;
  for (int i = 1; i < argc; ++i) {
    auto next = [&]() -> const char* { return i + 1 < argc ? argv[++i] : ""; };
    if (!std::strcmp(argv[i], "--storage")) {
      const char* v = next();
      storage = !std::strcmp(v, "f32") ? gpu::Storage::F32 : !std::strcmp(v, "fp8") ? gpu::Storage::FP8 : gpu::Storage::BF16;
    } else if (!std::strcmp(argv[i], "--call-time")) {
      base = gpu::TimeBase::Call;
    } else if (!std::strcmp(argv[i], "--queries")) {
      queries = uint32_t(std::atoi(next()));
    } else if (!std::strcmp(argv[i], "--max-len")) {
      max_len = uint32_t(std::atoi(next()));
    } else {
      std::fprintf(stderr, "hisa_fig2_sweep: unknown flag %s\n", argv[i]);
      return 2;
    }
  }
  std::vector<uint32_t> lengths;
  for (uint32_t L = 8192; L <= max_len; L *= 2) lengths.push_back(L);
  const Strategy strategies[] = {Strategy::Dsa, Strategy::BlockSparse, Strategy::Hisa};
  const HisaConfig cfg(128, 64, 2048, 64, 128);
  try {
    for (gpu::SweepMode mode : {gpu::SweepMode::FixedBudget, gpu::SweepMode::Ratio}) {
      std::cout << "# panel " << (mode == gpu::SweepMode::FixedBudget ? "(a) fixed budget m = 64" : "(b) M : m = 4 : 1")
                << ", storage " << (storage == gpu::Storage::BF16 ? "bf16" : storage == gpu::Storage::F32 ? "f32" : "e4m3")
                << ", " << queries << " queries at the newest position, "
                << (base == gpu::TimeBase::Kernels ? "kernel time" : "whole-call time (host containers)") << "\n";
      const auto recs = gpu::run_bench_sweep(cfg, lengths, queries, 1, strategies, mode, 4, BenchOptions{}, storage, base);
      write_bench_csv(std::cout, recs);
      // speed-up of HISA over the flat indexer per length
      for (size_t i = 0; i + 2 < recs.size(); i += 3)
        std::cout << "# L=" << recs[i].seq_len << " m=" << recs[i + 2].block_budget << ": flat " << recs[i].wall_ns_median / 1e3
                  << " us, block-sparse " << recs[i + 1].wall_ns_median / 1e3 << " us, hisa " << recs[i + 2].wall_ns_median / 1e3
                  << " us -> " << double(recs[i].wall_ns_median) / double(recs[i + 2].wall_ns_median) << "x\n";
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "hisa_fig2_sweep: %s\n", e.what());
    return 1;
  }
  return 0;
}
