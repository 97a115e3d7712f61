// Drop-in test program: the worked examples and properties SPEC.md gives for the indexer path
// (SPEC.md:118-120,128-130,138-140,178-180,188-190,198-200,208-210,218-220,228-235,427,461), written against
// the reference's own hisa:: API and run on the GPU through libhisa_dropin.so. Exit code 0 = all passed.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <numeric>
#include <sstream>

#include "hisa/attention.hpp"
#include "hisa/audit.hpp"
#include "hisa/block_sparse.hpp"
#include "hisa/bench.hpp"
#include "hisa/hisa.hpp"
#include "hisa/niah.hpp"
#include "hisa/parallel.hpp"
#include "hisa/synth.hpp"
#include "hisa/tensor_io.hpp"
#include "hisa_gpu.hpp"

using namespace hisa;

static int g_fail = 0, g_run = 0;
#define EXPECT(cond)                                                              \
  do {                                                                            \
    ++g_run;                                                                      \
    if (!(cond)) { ++g_fail; std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); } \
  } while (0)
template <class E, class F>
bool throws(F&& f) {
  try { f(); } catch (const E&) { return true; } catch (...) { return false; }
  return false;
}

static IndexerInputs tiny(std::vector<float> q, std::vector<float> w, std::vector<float> k, std::vector<uint32_t> pos,
                          uint32_t H, uint32_t d) {
  return IndexerInputs(std::move(q), std::move(w), std::move(k), std::move(pos), H, d);
}

// naive oracle for the DERIVED examples: triple loop in double
static double naive_score(const IndexerInputs& in, uint32_t row, uint32_t s) {
  double acc = 0;
  for (uint32_t j = 0; j < in.num_heads(); ++j) {
    double dp = 0;
    for (uint32_t i = 0; i < in.dim(); ++i) dp += double(in.query(row, j)[i]) * double(in.key(s)[i]);
    acc += double(in.gate(row, j)) * std::max(dp, 0.0);
  }
  return acc;
}
static std::vector<uint32_t> naive_topk(const std::vector<double>& sc, const std::vector<uint32_t>& pos, uint32_t k, TieBreak tb) {
  std::vector<uint32_t> order(sc.size());
  std::iota(order.begin(), order.end(), 0u);
  std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    if (sc[a] != sc[b]) return sc[a] > sc[b];
    return tb == TieBreak::SmallestIndex ? pos[a] < pos[b] : pos[a] > pos[b];
  });
  order.resize(std::min<size_t>(k, order.size()));
  std::vector<uint32_t> out;
  for (uint32_t i : order) out.push_back(pos[i]);
  std::sort(out.begin(), out.end());
  return out;
}

int main() {
  // ---- config ----
  EXPECT(throws<InfeasibleConfig>([] { HisaConfig c(128, 4, 2048, 64, 128); (void)c; }));
  EXPECT(!throws<InfeasibleConfig>([] { HisaConfig c(128, 16, 2048, 4, 64); (void)c; }));
  EXPECT(strategy_from_string("block-sparse") == Strategy::BlockSparse && to_string(Strategy::Hisa) == "hisa");

  // ---- score_tokens ----
  {
    auto in = tiny({1, 0}, {1}, {2, 0, -1, 3}, {1}, 1, 2);
    const uint32_t cand[] = {0, 1};
    OpCounter c;
    auto sv = score_tokens(in, 0, cand, &c);
    EXPECT(sv.scores[0] == 2.0 && sv.scores[1] == 0.0 && c.dot_products == 2);
    auto in2 = tiny({1, 0, 0, 1}, {1, -1}, {1, 1}, {0}, 2, 2);
    const uint32_t c0[] = {0};
    EXPECT(score_tokens(in2, 0, c0).scores[0] == 0.0);
    auto in3 = tiny({1, 0}, {1}, {2, 0, -1, 3}, {0}, 1, 2);
    EXPECT(throws<CausalViolation>([&] { score_tokens(in3, 0, cand); }));
    Rng rng(5);
    auto r = make_random_inputs(rng, 32, 3, 4, 16, QueryPlacement::Final);
    std::vector<uint32_t> all(32);
    std::iota(all.begin(), all.end(), 0u);
    auto got = score_tokens(r, 1, all);
    double worst = 0;
    for (uint32_t s = 0; s < 32; ++s) worst = std::max(worst, std::abs(got.scores[s] - naive_score(r, 1, s)));
    EXPECT(worst < 1e-5 * 50);  // SPEC tolerance 1e-5 on O(1) scores; these reach ~50
  }
  // ---- top_k_tokens ----
  {
    ScoreVector sv{{5, 1, 3}, {0, 1, 2}};
    EXPECT((top_k_tokens(sv, 2, TieBreak::SmallestIndex).token_indices == std::vector<uint32_t>{0, 2}));
    ScoreVector ties{{1, 1, 1}, {0, 1, 2}};
    EXPECT((top_k_tokens(ties, 2, TieBreak::SmallestIndex).token_indices == std::vector<uint32_t>{0, 1}));
    EXPECT((top_k_tokens(ties, 2, TieBreak::LargestIndex).token_indices == std::vector<uint32_t>{1, 2}));
    EXPECT(top_k_tokens(ties, 9, TieBreak::SmallestIndex).token_indices.size() == 3);
    Rng rng(9);
    for (int trial = 0; trial < 20; ++trial) {
      ScoreVector v;
      const uint32_t n = 1 + uint32_t(rng.below(1000));
      for (uint32_t i = 0; i < n; ++i) { v.scores.push_back(trial % 2 ? double(rng.below(7)) : double(float(rng.normal()))); v.positions.push_back(3 * i + 1); }
      const TieBreak tb = trial % 3 ? TieBreak::SmallestIndex : TieBreak::LargestIndex;
      EXPECT(top_k_tokens(v, 50, tb).token_indices == naive_topk(v.scores, v.positions, 50, tb));
    }
  }
  // ---- block summaries ----
  {
    const std::vector<float> k2 = {1, 2, 3, 4};
    auto c = build_block_summaries(k2, 2, 2);
    EXPECT(c.num_blocks() == 1 && c.pooled(0)[0] == 2.0 && c.pooled(0)[1] == 3.0);
    EXPECT(throws<EmptySequence>([] { build_block_summaries(std::span<const float>{}, 2, 2); }));
    BlockSummaryCache inc(4, 3);
    const std::vector<float> key = {1, 2, 3};
    inc.append(key);
    EXPECT(inc.count(0) == 1 && inc.pooled(0)[2] == 3.0);
    for (int i = 0; i < 4; ++i) inc.append(key);
    EXPECT(inc.num_blocks() == 2 && inc.count(0) == 4 && inc.count(1) == 1);
    const std::vector<float> bad = {1, 2};
    EXPECT(throws<DimensionMismatch>([&] { inc.append(bad); }));
    EXPECT(throws<Error>([&] { inc.pooled(7); }));
    Rng rng(3);
    std::vector<float> keys(1000 * 8);
    for (auto& v : keys) v = float(rng.normal());
    auto batch = build_block_summaries(keys, 8, 128);
    BlockSummaryCache stream(128, 8);
    for (int s = 0; s < 1000; ++s) stream.append(std::span<const float>(&keys[s * 8], 8));
    EXPECT(batch.num_blocks() == 8 && batch.count(7) == 104);
    double worst = 0;
    for (uint32_t b = 0; b < 8; ++b)
      for (uint32_t i = 0; i < 8; ++i) worst = std::max(worst, std::abs(batch.pooled(b)[i] - stream.pooled(b)[i]));
    EXPECT(worst <= 1e-6);  // SPEC.md:80 (device kernel and host append agree; in fact bit for bit)
    EXPECT(worst == 0.0);
  }
  // ---- score_blocks / select_blocks / candidate_union ----
  {
    auto in = tiny({1, 0}, {1}, {4, 0, -2, 0}, {1}, 1, 2);
    auto cache = build_block_summaries(in.keys_raw(), 2, 1);
    auto J = score_blocks(in, cache, 0);
    EXPECT(J.scores.size() == 2 && J.scores[0] == 4.0 && J.scores[1] == 0.0);
    HisaConfig cfg(4, 2, 8, 1, 2);
    ScoreVector js{{5, 1, 3, 2}, {0, 1, 2, 3}};
    EXPECT((select_blocks(js, cfg, 15) == std::vector<uint32_t>{0, 2, 3}));
    HisaConfig wide(4, 9, 8, 1, 2);
    EXPECT((select_blocks(js, wide, 15) == std::vector<uint32_t>{0, 1, 2, 3}));
    const uint32_t b0[] = {0}, b1[] = {1}, b023[] = {0, 2, 3};
    EXPECT((candidate_union(b0, 4, 10, 100) == std::vector<uint32_t>{0, 1, 2, 3}));
    EXPECT((candidate_union(b1, 4, 5, 100) == std::vector<uint32_t>{4, 5}));
    EXPECT(candidate_union(b023, 128, 500, 4096).size() == 373);
  }
  // ---- dsa_select / hisa_select regimes ----
  {
    Rng rng(11);
    const uint32_t L = 4096, H = 4, d = 16, B = 64, m = 8, k = 256;
    std::vector<uint32_t> pos = {0, 3, k - 1, k, m * B - 1, m * B, (m + 2) * B + 5, 2000, L - 1};
    auto in = make_random_inputs(rng, L, pos, H, d);
    HisaConfig cfg(B, m, k, H, d);
    auto cache = build_block_summaries(in.keys_raw(), d, B);
    for (uint32_t r = 0; r < pos.size(); ++r) {
      OpCounter ch, cd;
      auto h = hisa_select(in, cache, cfg, r, &ch);
      auto f = dsa_select(in, cfg, r, &cd);
      const uint32_t t = pos[r];
      EXPECT(std::is_sorted(h.token_indices.begin(), h.token_indices.end()));
      EXPECT(f.token_indices.size() == std::min(k, t + 1) && f.candidate_size == t + 1 && f.selected_blocks.empty());
      EXPECT(cd.dot_products == uint64_t(H) * (t + 1));
      if (t + 1 <= k) {
        std::vector<uint32_t> prefix(t + 1);
        std::iota(prefix.begin(), prefix.end(), 0u);
        EXPECT(h.token_indices == prefix);
      }
      if (t + 1 <= m * B) EXPECT(h.token_indices == f.token_indices);
      auto omega = candidate_union(h.selected_blocks, B, t, L);
      EXPECT(h.candidate_size == omega.size() && h.token_indices.size() == std::min<size_t>(k, omega.size()));
      EXPECT(std::includes(omega.begin(), omega.end(), h.token_indices.begin(), h.token_indices.end()));
      EXPECT(h.selected_blocks.size() <= m + 2 && h.selected_blocks.front() == 0 && h.selected_blocks.back() == t / B);
      EXPECT(ch.dot_products <= analytic_cost(cfg, t + 1, Strategy::Hisa));
      // T equals the brute-force flat selection restricted to the candidate pool
      std::vector<double> sc;
      for (uint32_t s : omega) sc.push_back(naive_score(in, r, s));
      auto want = naive_topk(sc, omega, k, cfg.tie_break);
      size_t same = 0;
      for (uint32_t v : h.token_indices) same += std::binary_search(want.begin(), want.end(), v);
      EXPECT(same + 1 >= want.size());  // identical up to one fp32-vs-f64 near-tie at the k-th score
      auto bs = block_sparse_select(in, cache, cfg, r);
      EXPECT(bs.token_indices == omega);
    }
  }
  // ---- the caller's BlockSummaryCache is what gets scored (hisa.hpp:16-21, block_summary.hpp:27-30) ----
  {
    Rng rng(31);
    const uint32_t L = 1000, H = 2, d = 8, B = 64, m = 3, k = 100;
    auto in = make_random_inputs(rng, L, std::vector<uint32_t>{10, 250, 299, 300, 640, 999}, H, d);
    HisaConfig cfg(B, m, k, H, d);
    // (a) a snapshot shorter than the inputs: 300 tokens appended = 5 blocks (the last one partial)
    BlockSummaryCache part(B, d);
    for (uint32_t s = 0; s < 300; ++s) part.append(in.key(s));
    EXPECT(part.num_blocks() == 5 && part.num_tokens() == 300);
    for (uint32_t r = 0; r < in.num_queries(); ++r) {
      const uint32_t t = in.position(r), elig = std::min(t / B, 4u) + 1;
      auto J = score_blocks(in, part, r);
      EXPECT(J.scores.size() == elig);  // eligible blocks clipped to cache.num_blocks()
      double worst = 0;
      for (uint32_t b = 0; b < elig; ++b) {
        const auto pk = part.pooled(b);
        double acc = 0;
        for (uint32_t j = 0; j < H; ++j) {
          double dp = 0;
          for (uint32_t i = 0; i < d; ++i) dp += double(in.query(r, j)[i]) * pk[i];
          acc += double(in.gate(r, j)) * std::max(dp, 0.0);
        }
        worst = std::max(worst, std::abs(acc - J.scores[b]));
      }
      EXPECT(worst < 1e-5);
      auto h = hisa_select(in, part, cfg, r);
      EXPECT(!h.selected_blocks.empty() && h.selected_blocks.front() == 0 && h.selected_blocks.back() == elig - 1);
      auto omega = candidate_union(h.selected_blocks, B, t, L);
      EXPECT(h.candidate_size == omega.size() && h.token_indices.size() == std::min<size_t>(k, omega.size()));
      EXPECT(std::includes(omega.begin(), omega.end(), h.token_indices.begin(), h.token_indices.end()));
      EXPECT(block_sparse_select(in, part, cfg, r).token_indices == omega);
    }
    // (b) a cache that was fed DIFFERENT keys: its contents decide the block scores, not the inputs' keys
    BlockSummaryCache other(B, d);
    for (uint32_t s = 0; s < L; ++s) {
      std::vector<float> kk(in.key(s).begin(), in.key(s).end());
      if (s / B == 2) for (auto& v : kk) v = -v;
      other.append(kk);
    }
    auto full = build_block_summaries(in.keys_raw(), d, B);
    auto Ja = score_blocks(in, full, 5), Jb = score_blocks(in, other, 5);
    EXPECT(Ja.scores.size() == 16 && Jb.scores.size() == 16);
    EXPECT(Ja.scores[2] != Jb.scores[2] && Ja.scores[1] == Jb.scores[1] && Ja.scores[3] == Jb.scores[3]);
    EXPECT(throws<EmptySequence>([&] { BlockSummaryCache empty(B, d); score_blocks(in, empty, 0); }));
  }
  // ---- per-row calls fanned out over threads (parallel.hpp:15-19; SPEC "callers may fan out queries") ----
  {
    Rng rng(41);
    const uint32_t L = 2048, H = 4, d = 16, B = 32, m = 4, k = 64, Q = 96;
    auto in = make_random_inputs(rng, L, Q, H, d, QueryPlacement::Spread);
    HisaConfig cfg(B, m, k, H, d);
    auto cache = build_block_summaries(in.keys_raw(), d, B);
    std::vector<SelectionResult> par(Q), par_flat(Q);
    parallel_for(Q, 8, [&](std::size_t r) {
      par[r] = hisa_select(in, cache, cfg, uint32_t(r));
      par_flat[r] = dsa_select(in, cfg, uint32_t(r));
    });
    bool same = true;
    for (uint32_t r = 0; r < Q; ++r) {
      same = same && par[r].token_indices == hisa_select(in, cache, cfg, r).token_indices;
      same = same && par_flat[r].token_indices == dsa_select(in, cfg, r).token_indices;
    }
    EXPECT(same);
  }
  // ---- results follow the CONTENT of the inputs, not their address (same sizes, one key row differs) ----
  {
    const uint32_t L = 512, H = 2, d = 8;
    HisaConfig cfg(32, 2, 16, H, d);
    std::vector<std::vector<uint32_t>> got;
    for (int variant = 0; variant < 2; ++variant) {
      Rng rng(51);  // same seed: identical tensors ...
      IndexerInputs base = make_random_inputs(rng, L, std::vector<uint32_t>{L - 1}, H, d);
      std::vector<float> keys = base.keys_raw();
      const uint32_t needle = variant ? 300u : 100u;  // ... except for one boosted key row
      for (uint32_t i = 0; i < d; ++i) keys[needle * d + i] = 40.f * base.query(0, 0)[i];
      const IndexerInputs in(base.queries_raw(), base.gates_raw(), std::move(keys), base.positions_raw(), H, d);
      got.push_back(dsa_select(in, cfg, 0).token_indices);
      EXPECT(std::binary_search(got.back().begin(), got.back().end(), needle));
    }
    EXPECT(got[0] != got[1]);
  }
  // ---- double scores that collapse to one float are still ordered by their double value (dsa.hpp:22-27) ----
  {
    ScoreVector sv{{1.0, 1.0 + 1e-12, 1.0 + 2e-12, 0.5}, {0, 1, 2, 3}};
    EXPECT((top_k_tokens(sv, 1, TieBreak::SmallestIndex).token_indices == std::vector<uint32_t>{2}));
    EXPECT((top_k_tokens(sv, 2, TieBreak::SmallestIndex).token_indices == std::vector<uint32_t>{1, 2}));
    Rng rng(61);
    for (int trial = 0; trial < 10; ++trial) {
      ScoreVector v;
      const uint32_t n = 200 + uint32_t(rng.below(800));
      for (uint32_t i = 0; i < n; ++i) { v.scores.push_back(1.0 + 1e-9 * double(rng.below(50))); v.positions.push_back(i); }
      const TieBreak tb = trial % 2 ? TieBreak::SmallestIndex : TieBreak::LargestIndex;
      EXPECT(top_k_tokens(v, 37, tb).token_indices == naive_topk(v.scores, v.positions, 37, tb));
      HisaConfig cfg(4, 9, 8, 1, 2);
      cfg.tie_break = tb;
      cfg.forced_in_budget = trial % 3 == 0;
      auto blocks = select_blocks(v, cfg, (n - 1) * 4);
      std::vector<double> rest(v.scores);
      std::vector<uint32_t> want;
      if (cfg.forced_in_budget) {
        std::vector<double> mid(v.scores.begin() + 1, v.scores.end() - 1);
        std::vector<uint32_t> mp(v.positions.begin() + 1, v.positions.end() - 1);
        want = naive_topk(mid, mp, 7, tb);
      } else {
        want = naive_topk(v.scores, v.positions, 9, tb);
      }
      want.push_back(0);
      want.push_back(n - 1);
      std::sort(want.begin(), want.end());
      want.erase(std::unique(want.begin(), want.end()), want.end());
      EXPECT(blocks == want);
    }
  }
  // ---- fp8 storage through the C++ layer, the 4:1 sweep and the separately reported pool build ----
  {
    Rng rng(71);
    const uint32_t L = 2048, H = 64, d = 128, B = 64, m = 4, k = 128;
    auto in = make_random_inputs(rng, L, std::vector<uint32_t>{100, 700, 1500, 2047}, H, d);
    HisaConfig cfg(B, m, k, H, d);
    gpu::Indexer f8(cfg, gpu::Storage::FP8), bf(cfg, gpu::Storage::BF16);
    f8.set_keys(in.keys_raw());
    bf.set_keys(in.keys_raw());
    auto a = f8.hisa_select_batch(in), b = bf.hisa_select_batch(in);
    double iou = 0;
    for (uint32_t r = 0; r < in.num_queries(); ++r) {
      EXPECT(a[r].token_indices.size() == b[r].token_indices.size() && std::is_sorted(a[r].token_indices.begin(), a[r].token_indices.end()));
      iou += selection_overlap(a[r], b[r]);
    }
    EXPECT(iou / in.num_queries() > 0.6);  // e4m3 quantisation moves the boundary, not the bulk of the selection
    HisaConfig small(32, 4, 64, 4, 16);
    const uint32_t lengths[] = {1024, 4096};
    const Strategy strategies[] = {Strategy::Dsa, Strategy::Hisa};
    auto sweep = gpu::run_bench_sweep(small, lengths, 8, 1, strategies, gpu::SweepMode::Ratio, 4);
    EXPECT(sweep.size() == 4 && sweep[0].block_budget == 8 && sweep[2].block_budget == 32 && sweep[3].strategy == Strategy::Hisa);
    EXPECT(sweep[1].pool_build_ns > 0 && sweep[3].wall_ns_median > 0);  // bench.hpp:28
  }
  // ---- analytic cost and the bench record ----
  {
    HisaConfig cfg(128, 64, 2048, 1, 16);
    EXPECT(analytic_cost(cfg, 65536, Strategy::Hisa) == 8960 && analytic_cost(cfg, 65536, Strategy::Dsa) == 65536);
    HisaConfig small(32, 4, 64, 4, 16);
    auto rec = run_bench(small, 1024, 16, 1, Strategy::Dsa);
    EXPECT(rec.dot_products == uint64_t(16) * 4 * 1024 && rec.wall_ns_median > 0);
    auto rh = run_bench(small, 1024, 16, 1, Strategy::Hisa);
    EXPECT(rh.dot_products <= rh.analytic_bound);
    std::ostringstream os;
    write_bench_csv(os, {rec, rh});
    EXPECT(os.str().rfind("strategy,L,B,m,k,H,d,wall_ns_median", 0) == 0);
  }
  // ---- HSB round trip ----
  {
    Rng rng(2);
    auto in = make_random_inputs(rng, 20, 3, 2, 4, QueryPlacement::Spread);
    const auto path = std::filesystem::temp_directory_path() / "hisa_dropin_test.hsb";
    save_tensor_file(in, path);
    auto back = load_tensor_file(path);
    EXPECT(back.keys_raw() == in.keys_raw() && back.queries_raw() == in.queries_raw() && back.gates_raw() == in.gates_raw() &&
           back.positions_raw() == in.positions_raw() && back.num_heads() == 2 && back.dim() == 4);
    {
      std::FILE* f = std::fopen(path.c_str(), "r+b");
      std::fputc('X', f);
      std::fclose(f);
    }
    EXPECT(throws<BadMagic>([&] { load_tensor_file(path); }));
    std::filesystem::remove(path);
    EXPECT(throws<IoError>([&] { load_tensor_file(path); }));
  }
  // ---- downstream consumer (attention.hpp:48-59) ----
  {
    Rng rng(21);
    const uint32_t L = 512, Q = 6, dm = 24;
    std::vector<float> lat(L * dm), hs(Q * dm);
    for (auto& v : lat) v = float(rng.normal());
    for (auto& v : hs) v = float(rng.normal());
    const AttentionInputs attn(hs, lat, {0, 100, 200, 300, 400, 511}, dm);
    EXPECT(std::abs(attn.scale() - 1.0 / std::sqrt(24.0)) < 1e-15);
    // single token -> that latent exactly; L = 1 prefix -> c_0
    const uint32_t one[] = {77};
    auto u = sparse_attend(attn, one, 2);
    EXPECT(std::equal(u.begin(), u.end(), attn.latent(77).begin()));
    auto d0 = dense_attend(attn, 0);
    EXPECT(std::equal(d0.begin(), d0.end(), attn.latent(0).begin()));
    // full prefix == dense within 1e-5; weights sum to 1 within 1e-6 (fp32 device arithmetic: 1e-5)
    std::vector<uint32_t> prefix(301);
    std::iota(prefix.begin(), prefix.end(), 0u);
    std::vector<double> w;
    auto sp = sparse_attend(attn, prefix, 3, &w);
    auto de = dense_attend(attn, 3);
    double worst = 0, wsum = 0;
    for (uint32_t i = 0; i < dm; ++i) worst = std::max(worst, double(std::abs(sp[i] - de[i])));
    for (double x : w) wsum += x;
    EXPECT(worst <= 1e-5 && w.size() == 301 && std::abs(wsum - 1.0) <= 1e-5);
    // naive double-precision check of one row
    {
      std::vector<double> logit(301), ref(dm, 0.0);
      double mx = -1e300, den = 0;
      for (uint32_t s = 0; s <= 300; ++s) {
        double acc = 0;
        for (uint32_t i = 0; i < dm; ++i) acc += double(attn.query_state(3)[i]) * double(attn.latent(s)[i]);
        logit[s] = acc * attn.scale();
        mx = std::max(mx, logit[s]);
      }
      for (auto& x : logit) { x = std::exp(x - mx); den += x; }
      for (uint32_t s = 0; s <= 300; ++s)
        for (uint32_t i = 0; i < dm; ++i) ref[i] += logit[s] / den * double(attn.latent(s)[i]);
      double err = 0;
      for (uint32_t i = 0; i < dm; ++i) err = std::max(err, std::abs(ref[i] - double(de[i])));
      EXPECT(err <= 1e-5);
    }
    EXPECT(throws<EmptySelection>([&] { sparse_attend(attn, std::span<const uint32_t>{}, 1); }));
    const uint32_t future[] = {5, 101};
    EXPECT(throws<CausalViolation>([&] { sparse_attend(attn, future, 1); }));
    EXPECT(throws<ShapeMismatch>([&] { AttentionInputs bad(hs, lat, {0, 1, 2, 3, 4, 512}, dm); (void)bad; }));
    // plug-and-play: the SelectionResult of every strategy feeds the consumer unchanged
    Rng r2(22);
    const HisaConfig cfg(32, 4, 64, 4, 16);
    auto in = make_random_inputs(r2, L, std::vector<uint32_t>{0, 100, 200, 300, 400, 511}, 4, 16);
    auto cache = build_block_summaries(in.keys_raw(), 16, 32);
    for (uint32_t row = 0; row < Q; ++row) {
      for (const SelectionResult& sel : {dsa_select(in, cfg, row), hisa_select(in, cache, cfg, row), block_sparse_select(in, cache, cfg, row)}) {
        std::vector<double> ww;
        auto out = sparse_attend(attn, sel, row, &ww);
        double s1 = 0;
        for (double x : ww) s1 += x;
        EXPECT(out.size() == dm && ww.size() == sel.token_indices.size() && std::abs(s1 - 1.0) <= 1e-5);
      }
    }
    gpu::Attention batched(attn, gpu::Storage::F32);
    std::vector<SelectionResult> sels;
    for (uint32_t row = 0; row < Q; ++row) sels.push_back(hisa_select(in, cache, cfg, row));
    auto all = batched.sparse_attend_batch(sels);
    auto row4 = sparse_attend(attn, sels[4], 4);
    EXPECT(all.size() == size_t(Q) * dm && std::equal(row4.begin(), row4.end(), all.begin() + 4 * dm));
  }
  // ---- audits (audit.hpp:37-49) ----
  {
    AuditOptions ao;
    ao.min_queries = 300;
    auto a = run_regime_equivalence_audit(ao);
    if (!a.passed()) std::printf("regime audit: seed %llu row %u %s\n", (unsigned long long)a.failure->instance_seed, a.failure->query_row, a.failure->detail.c_str());
    EXPECT(a.passed() && a.queries_checked >= 300 && a.instances_run >= 1);
    auto b = run_dense_regime_audit(ao);
    if (!b.passed()) std::printf("dense audit: seed %llu row %u %s\n", (unsigned long long)b.failure->instance_seed, b.failure->query_row, b.failure->detail.c_str());
    EXPECT(b.passed() && b.queries_checked >= 300);
    auto c = run_subset_chain_audit(ao);
    if (!c.passed()) std::printf("subset audit: seed %llu row %u %s\n", (unsigned long long)c.failure->instance_seed, c.failure->query_row, c.failure->detail.c_str());
    EXPECT(c.passed() && c.queries_checked >= 300);
    ao.inject_tie_mismatch = true;  // the failure path must fire
    auto f = run_regime_equivalence_audit(ao);
    EXPECT(!f.passed() && f.failure.has_value() && !f.failure->detail.empty());  // audit.hpp:23-24
    EXPECT(!a.failure.has_value());
    AblationOptions ab;
    ab.seq_len = 4096;
    ab.token_budget = 512;
    ab.seeds = 2;
    ab.configs = {{64, 32, true}, {128, 16, true}, {128, 4, false}};
    auto rows = run_overlap_ablation(ab);
    EXPECT(rows.size() == 3);
    for (const auto& r : rows) EXPECT(r.mean_overlap > 0.0 && r.mean_overlap <= 1.0 && r.min_overlap <= r.mean_overlap);
    EXPECT(rows[0].mean_overlap > rows[2].mean_overlap);  // token refinement beats the block-sparse baseline
    std::printf("ablation IoU vs flat: B=64,m=32 %.3f | B=128,m=16 %.3f | block-sparse B=128,m=4 %.3f\n", rows[0].mean_overlap,
                rows[1].mean_overlap, rows[2].mean_overlap);
  }
  // ---- needle-in-a-haystack harness (niah.hpp) ----
  {
    const HisaConfig cfg(128, 16, 2048, 4, 16);
    auto first = generate_niah(4096, 0.0, 11, cfg), last = generate_niah(4096, 1.0, 11, cfg), mid = generate_niah(4096, 0.5, 12, cfg);
    EXPECT(first.needle_positions == std::vector<uint32_t>{0} && last.needle_positions == std::vector<uint32_t>{4095});
    EXPECT(mid.needle_positions == std::vector<uint32_t>{2047} && mid.inputs.num_queries() == 1 && mid.inputs.position(0) == 4095);
    auto flat = dsa_select(mid.inputs, cfg, 0);
    EXPECT(needle_recall(mid, flat) == 1.0);  // the flat scan retrieves the needle by construction
    {  // the needle is the single best-scoring token
      std::vector<uint32_t> all(4096);
      std::iota(all.begin(), all.end(), 0u);
      auto sv = score_tokens(mid.inputs, 0, all);
      EXPECT(std::max_element(sv.scores.begin(), sv.scores.end()) - sv.scores.begin() == 2047);
    }
    SelectionResult a{{0, 1, 2, 3}, {}, 0}, b{{2, 3, 4, 5}, {}, 0}, c{{7, 8}, {}, 0}, e{};
    EXPECT(selection_overlap(a, a) == 1.0 && selection_overlap(a, c) == 0.0 && std::abs(selection_overlap(a, b) - 2.0 / 6.0) < 1e-15);
    EXPECT(selection_overlap(a, b) == selection_overlap(b, a) && selection_overlap(a, e) == 0.0);
    EXPECT(throws<BothEmpty>([&] { selection_overlap(e, e); }));
    NiahGridParams gp;
    gp.lengths = {1024, 8192, 16384};
    gp.seeds = 6;
    auto recs = run_niah_grid(gp);
    EXPECT(recs.size() == 3u * 5u * 6u * 3u);
    EXPECT(recs[0].strategy == Strategy::Dsa && recs[1].strategy == Strategy::Hisa && recs[2].strategy == Strategy::BlockSparse &&
           recs[0].seq_len == 1024 && recs[3].seed_index == 1 && recs.back().seq_len == 16384 && recs.back().depth == 1.0);
    double mean[3] = {0, 0, 0};
    for (const auto& r : recs) mean[int(r.strategy)] += r.recall;
    for (double& v : mean) v /= double(recs.size() / 3);
    std::printf("NIAH mean recall: dsa %.3f  hisa %.3f  block-sparse %.3f\n", mean[0], mean[1], mean[2]);
    EXPECT(mean[0] == 1.0);                       // DSA recall = 1 by construction
    EXPECT(mean[1] >= mean[2] && mean[1] >= 0.9);  // HISA >= block-sparse in aggregate
    for (const auto& r : recs) EXPECT(r.strategy != Strategy::Dsa || r.overlap_vs_dsa == 1.0);
    auto again = run_niah_grid(gp);
    bool same = again.size() == recs.size();
    for (size_t i = 0; same && i < recs.size(); ++i) same = again[i].recall == recs[i].recall && again[i].overlap_vs_dsa == recs[i].overlap_vs_dsa;
    EXPECT(same);                                 // deterministic for a given base seed
    std::ostringstream csv, dat;
    write_niah_csv(csv, recs);
    write_niah_grid_dat(dat, recs, Strategy::Hisa);
    const std::string csv_s = csv.str(), dat_s = dat.str();
    EXPECT(csv_s.rfind("strategy,L,depth,seed,recall,overlap_vs_dsa\n", 0) == 0);
    EXPECT(size_t(std::count(csv_s.begin(), csv_s.end(), '\n')) == recs.size() + 1);
    EXPECT(dat_s.rfind("depth 1024 8192 16384\n", 0) == 0 && std::count(dat_s.begin(), dat_s.end(), '\n') == 6);
  }
  std::printf("%s: %d checks, %d failed\n", g_fail ? "FAILED" : "PASSED", g_run, g_fail);
  return g_fail ? 1 : 0;
}
