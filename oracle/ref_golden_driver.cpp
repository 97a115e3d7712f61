// ORACLE — TEST INFRASTRUCTURE ONLY.
// Golden-vector generator: compiled against the REFERENCE's own headers where they lie under
// /root/reference (never copied into this repo). The only parts of the reference with bodies are
// hisa/rng.hpp (fully inline), the HisaConfig constructor (hisa/config.hpp:27-45), OpCounter
// (hisa/types.hpp:33-45) and src/types.cpp — everything this driver exercises. Output: JSON on stdout,
// committed as tests/golden/ref_golden.json by oracle/Makefile's `golden` target.
#include <cinttypes>
#include <cstdio>
#include <string>

#include "hisa/config.hpp"
#include "hisa/rng.hpp"
#include "hisa/types.hpp"

static void stream_u64(const char* name, uint64_t seed, int n, bool last) {
  hisa::Rng r(seed);
  std::printf("  \"%s\": [", name);
  for (int i = 0; i < n; ++i) std::printf("%s\"%" PRIu64 "\"", i ? ", " : "", r.next_u64());
  std::printf("]%s\n", last ? "" : ",");
}

int main() {
  std::printf("{\n");
  stream_u64("u64_seed1", 1, 8, false);
  stream_u64("u64_seed42", 42, 8, false);
  stream_u64("u64_seed_max", 0xffffffffffffffffULL, 4, false);
  {  // long skip: element 100000 exercises many state refills
    hisa::Rng r(7);
    uint64_t v = 0;
    for (int i = 0; i <= 100000; ++i) v = r.next_u64();
    std::printf("  \"u64_seed7_at100000\": \"%" PRIu64 "\",\n", v);
  }
  {
    hisa::Rng r(42);
    std::printf("  \"uniform_seed42\": [");
    for (int i = 0; i < 6; ++i) std::printf("%s\"%a\"", i ? ", " : "", r.uniform());
    std::printf("],\n");
  }
  {
    hisa::Rng r(42);
    std::printf("  \"uniform_0p5_1p5_seed42\": [");
    for (int i = 0; i < 6; ++i) std::printf("%s\"%a\"", i ? ", " : "", r.uniform(0.5, 1.5));
    std::printf("],\n");
  }
  {
    hisa::Rng r(42);
    std::printf("  \"normal_seed42\": [");
    for (int i = 0; i < 9; ++i) std::printf("%s\"%a\"", i ? ", " : "", r.normal());
    std::printf("],\n");
  }
  {
    hisa::Rng r(7);
    std::printf("  \"below1000_seed7\": [");
    for (int i = 0; i < 8; ++i) std::printf("%s%" PRIu64, i ? ", " : "", r.below(1000));
    std::printf("],\n");
  }
  {
    hisa::Rng r(7);
    std::printf("  \"below5_seed7\": [");
    for (int i = 0; i < 16; ++i) std::printf("%s%" PRIu64, i ? ", " : "", r.below(5));
    std::printf("],\n");
  }
  std::printf("  \"splitmix64_0\": \"%" PRIu64 "\",\n", hisa::splitmix64(0));
  std::printf("  \"splitmix64_123456789\": \"%" PRIu64 "\",\n", hisa::splitmix64(123456789));
  std::printf("  \"mix_seed_1_2_3_4\": \"%" PRIu64 "\",\n", hisa::mix_seed(1, 2, 3, 4));
  std::printf("  \"mix_seed_1_2\": \"%" PRIu64 "\",\n", hisa::mix_seed(1, 2));
  // HisaConfig feasibility: (B, m, k, H, d) -> 1 if the reference constructor accepts, 0 if it throws
  struct Case { uint32_t B, m, k, H, d; };
  const Case cases[] = {{128, 64, 2048, 64, 128}, {128, 4, 2048, 64, 128}, {128, 16, 2048, 4, 64},
                        {128, 15, 2048, 4, 64},   {0, 1, 1, 1, 1},        {1, 0, 1, 1, 1},
                        {1, 1, 0, 1, 1},          {1, 1, 1, 0, 1},        {1, 1, 1, 1, 0},
                        {1, 1, 1, 1, 1},          {65536, 65536, 4294967295u, 1, 1}, {64, 8, 256, 4, 16}};
  std::printf("  \"config_cases\": [");
  bool first = true;
  for (const Case& c : cases) {
    int ok = 1;
    try { hisa::HisaConfig cfg(c.B, c.m, c.k, c.H, c.d); (void)cfg; } catch (const hisa::InfeasibleConfig&) { ok = 0; }
    std::printf("%s[%u, %u, %u, %u, %u, %d]", first ? "" : ", ", c.B, c.m, c.k, c.H, c.d, ok);
    first = false;
  }
  std::printf("],\n");
  {
    hisa::HisaConfig cfg(128, 64, 2048, 64, 128);
    std::printf("  \"config_defaults\": {\"force_first_last\": %d, \"forced_in_budget\": %d, \"tie_break\": %d, \"pool_mode\": %d},\n",
                int(cfg.force_first_last), int(cfg.forced_in_budget), int(cfg.tie_break), int(cfg.pool_mode));
  }
  std::printf("  \"strategy_names\": [\"%s\", \"%s\", \"%s\"]\n",
              std::string(hisa::to_string(hisa::Strategy::Dsa)).c_str(),
              std::string(hisa::to_string(hisa::Strategy::Hisa)).c_str(),
              std::string(hisa::to_string(hisa::Strategy::BlockSparse)).c_str());
  std::printf("}\n");
  return 0;
}
