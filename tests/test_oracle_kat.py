"""Known-answer tests: every worked example SPEC.md gives for the hot path (the reference ships no test
files; these examples are its golden vectors — SURVEY.md §8c), run against the CPU oracle."""
import numpy as np
import pytest


def problem(oracle, q, w, keys, pos, **cfg):
    q = np.asarray(q, np.float32)
    w = np.asarray(w, np.float32)
    keys = np.asarray(keys, np.float32)
    if q.ndim == 2:
        q = q[None]
    if w.ndim == 1:
        w = w[None]
    return oracle.Problem(q, w, keys, np.asarray(pos, np.uint32), **cfg)


# ---- score_tokens ----
def test_score_tokens_relu_zeroes_negative(oracle):
    p = problem(oracle, [[1, 0]], [1], [[2, 0], [-1, 3]], [1])
    s, dots = oracle.score_tokens(p, 0, [0, 1])
    assert s.tolist() == [2.0, 0.0] and dots == 2


def test_score_tokens_negative_gate_cancels(oracle):
    p = problem(oracle, [[1, 0], [0, 1]], [1, -1], [[1, 1]], [0])
    s, _ = oracle.score_tokens(p, 0, [0])
    assert s.tolist() == [0.0]


def test_score_tokens_vs_naive_triple_loop(oracle):
    rng = np.random.default_rng(0)
    H, d, L = 4, 16, 32
    p = problem(oracle, rng.standard_normal((1, H, d)), rng.standard_normal((1, H)), rng.standard_normal((L, d)), [L - 1])
    s, dots = oracle.score_tokens(p, 0, np.arange(L))
    ref = np.zeros(L)
    for si in range(L):
        for j in range(H):
            acc = 0.0
            for i in range(d):
                acc += float(p.queries[0, j, i]) * float(p.keys[si, i])
            ref[si] += float(p.gates[0, j]) * max(acc, 0.0)
    assert np.allclose(s, ref, rtol=0, atol=1e-5) and dots == H * L


def test_score_tokens_causal_violation(oracle):
    p = problem(oracle, [[1, 0]], [1], [[2, 0], [-1, 3]], [0])
    with pytest.raises(oracle.OracleError) as e:
        oracle.score_tokens(p, 0, [0, 1])
    assert e.value.name == "CausalViolation"


# ---- top_k_tokens ----
def test_top_k_forced_ordering(oracle):
    assert oracle.top_k([5, 1, 3], [0, 1, 2], 2).tolist() == [0, 2]


def test_top_k_tie_break(oracle):
    assert oracle.top_k([1, 1, 1], [0, 1, 2], 2, tie_break=0).tolist() == [0, 1]
    assert oracle.top_k([1, 1, 1], [0, 1, 2], 2, tie_break=1).tolist() == [1, 2]


def test_top_k_k_larger_than_n(oracle):
    assert oracle.top_k([3, 2], [4, 9], 10).tolist() == [4, 9]


@pytest.mark.parametrize("tb", [0, 1])
def test_top_k_vs_full_sort(oracle, tb):
    rng = np.random.default_rng(1)
    for trial in range(200):
        n = int(rng.integers(1, 1200))
        k = int(rng.integers(1, 80))
        scores = rng.integers(-3, 4, n).astype(np.float64) if trial % 2 else rng.standard_normal(n)
        pos = np.sort(rng.choice(5000, n, replace=False)).astype(np.uint32)
        order = sorted(range(n), key=lambda i: (-scores[i], pos[i] if tb == 0 else -int(pos[i])))
        want = sorted(int(pos[i]) for i in order[:k])
        assert oracle.top_k(scores, pos, k, tb).tolist() == want


def test_signed_zero_scores_tie(oracle):
    assert oracle.top_k([-0.0, 0.0, -1.0], [0, 1, 2], 1, tie_break=0).tolist() == [0]
    assert oracle.top_k([-0.0, 0.0, -1.0], [0, 1, 2], 1, tie_break=1).tolist() == [1]


# ---- dsa_select ----
def test_dsa_dense_regime(oracle):
    rng = np.random.default_rng(2)
    p = problem(oracle, rng.standard_normal((1, 2, 4)), [[1, 1]], rng.standard_normal((8, 4)), [3], block_size=4, block_budget=4, token_budget=10)
    r = oracle.select_batch("dsa", p)
    assert r.idx[0, :4].tolist() == [0, 1, 2, 3] and r.count[0] == 4 and r.cand[0] == 4 and r.nblocks[0] == 0


def test_dsa_single_token(oracle):
    p = problem(oracle, [[1.0]], [1], [[1.0]], [0], block_size=1, block_budget=1, token_budget=1)
    r = oracle.select_batch("dsa", p)
    assert r.idx[0].tolist() == [0]


def test_dsa_vs_brute_force(oracle):
    rng = np.random.default_rng(3)
    L, H, d, k = 256, 4, 16, 32
    p = problem(oracle, rng.standard_normal((L, H, d)), rng.uniform(0.5, 1.5, (L, H)), rng.standard_normal((L, d)),
                np.arange(L), block_size=16, block_budget=4, token_budget=k)
    r = oracle.select_batch("dsa", p)
    dots = np.einsum("thd,sd->ths", p.queries.astype(np.float64), p.keys.astype(np.float64))
    S = (np.maximum(dots, 0) * p.gates.astype(np.float64)[:, :, None]).sum(1)
    for t in range(L):
        order = sorted(range(t + 1), key=lambda s: (-S[t, s], s))[:k]
        assert r.idx[t, :r.count[t]].tolist() == sorted(order)
        assert r.count[t] == min(k, t + 1)
    assert r.dots == H * L * (L + 1) // 2


# ---- block summaries ----
def test_pool_mean_of_two(oracle):
    _, counts, pooled = oracle.pool_build(np.array([[1, 2], [3, 4]], np.float32), 2)
    assert pooled.tolist() == [[2.0, 3.0]] and counts.tolist() == [2]


def test_pool_identical_keys(oracle):
    v = np.float32([0.1, -7.25, 3.0])
    _, _, pooled = oracle.pool_build(np.tile(v, (37, 1)), 5)
    assert np.allclose(pooled, np.tile(v.astype(np.float64), (8, 1)), rtol=0, atol=1e-6)


def test_pool_partial_last_block(oracle):
    rng = np.random.default_rng(4)
    keys = rng.standard_normal((1000, 8)).astype(np.float32)
    _, counts, pooled = oracle.pool_build(keys, 128)
    assert len(counts) == 8 and counts.tolist() == [128] * 7 + [104]
    for b in range(8):
        assert np.allclose(pooled[b], keys[b * 128:(b + 1) * 128].astype(np.float64).mean(0), rtol=0, atol=1e-6)


def test_pool_append_rollover_and_batch_equivalence(oracle):
    rng = np.random.default_rng(5)
    keys = rng.standard_normal((10000, 4)).astype(np.float32)
    _, c1, _ = oracle.pool_build(keys[:1], 4, incremental=True)
    assert c1.tolist() == [1]
    _, c2, _ = oracle.pool_build(keys[:5], 4, incremental=True)
    assert c2.tolist() == [4, 1]
    _, _, inc = oracle.pool_build(keys, 128, incremental=True)
    _, _, bat = oracle.pool_build(keys, 128)
    assert np.allclose(inc, bat, rtol=0, atol=1e-6)


def test_pool_errors(oracle):
    with pytest.raises(oracle.OracleError) as e:
        oracle.pool_build(np.zeros((0, 4), np.float32), 4)
    assert e.value.name == "EmptySequence"
    assert oracle.lib().horacle_pool_append_dim_check(4, 3) == 4  # DimensionMismatch
    assert oracle.lib().horacle_pool_append_dim_check(4, 4) == 0
    assert oracle.lib().horacle_pool_pooled_check(0) == 0
    assert oracle.lib().horacle_pool_pooled_check(1) != 0


# ---- score_blocks ----
def test_score_blocks_trivial(oracle):
    p = problem(oracle, [[1, 0]], [1], np.zeros((8, 2)), [7], block_size=4)
    assert oracle.score_pooled(p, 0, [[4, 0], [-2, 0]]).tolist() == [4.0, 0.0]


def test_score_blocks_eligibility_count(oracle):
    rng = np.random.default_rng(6)
    B = 4
    p = problem(oracle, rng.standard_normal((1, 2, 3)), [[1, 1]], rng.standard_normal((5 * B, 3)), [2 * B + 1], block_size=B)
    assert len(oracle.score_blocks(p, 0)) == 3


def test_score_blocks_vs_naive(oracle):
    rng = np.random.default_rng(7)
    L, H, d, B = 300, 4, 16, 32
    p = problem(oracle, rng.standard_normal((1, H, d)), rng.standard_normal((1, H)), rng.standard_normal((L, d)), [L - 1], block_size=B)
    J = oracle.score_blocks(p, 0)
    M = (L + B - 1) // B
    ref = np.zeros(M)
    for b in range(M):
        pk = p.keys[b * B:(b + 1) * B].astype(np.float64).mean(0)
        for j in range(H):
            ref[b] += float(p.gates[0, j]) * max(float(p.queries[0, j].astype(np.float64) @ pk), 0.0)
    assert np.allclose(J, ref, rtol=0, atol=1e-5)


# ---- select_blocks ----
def cfgp(oracle, **cfg):
    return oracle.Problem(np.zeros((1, 1, 1)), np.zeros((1, 1)), np.zeros((1, 1)), np.zeros(1, np.uint32), **cfg)


def test_select_blocks_forced_union(oracle):
    p = cfgp(oracle, block_size=4, block_budget=2, token_budget=8)
    assert oracle.select_blocks([5, 1, 3, 2], [0, 1, 2, 3], p, 15).tolist() == [0, 2, 3]


def test_select_blocks_budget_covers_all(oracle):
    p = cfgp(oracle, block_size=4, block_budget=9, token_budget=8)
    assert oracle.select_blocks([5, 1, 3, 2], [0, 1, 2, 3], p, 15).tolist() == [0, 1, 2, 3]


def test_select_blocks_no_forcing_and_in_budget(oracle):
    p = cfgp(oracle, block_size=4, block_budget=2, token_budget=8, force_first_last=False)
    assert oracle.select_blocks([1, 5, 3, 2], [0, 1, 2, 3], p, 15).tolist() == [1, 2]
    p = cfgp(oracle, block_size=4, block_budget=3, token_budget=8, forced_in_budget=True)
    assert oracle.select_blocks([1, 5, 3, 2], [0, 1, 2, 3], p, 15).tolist() == [0, 1, 3]


@pytest.mark.parametrize("tb", [0, 1])
def test_select_blocks_vs_sort_oracle(oracle, tb):
    rng = np.random.default_rng(8)
    for trial in range(200):
        n = int(rng.integers(1, 80))
        m = int(rng.integers(1, 24))
        J = rng.integers(0, 5, n).astype(np.float64) if trial % 2 else rng.standard_normal(n)
        B = 4
        t = (n - 1) * B + int(rng.integers(0, B))
        p = cfgp(oracle, block_size=B, block_budget=m, token_budget=m * B, tie_break=tb)
        order = sorted(range(n), key=lambda b: (-J[b], b if tb == 0 else -b))[:m]
        want = sorted(set(order) | {0, n - 1})
        assert oracle.select_blocks(J, np.arange(n), p, t).tolist() == want


# ---- candidate_union ----
def test_candidate_union_examples(oracle):
    assert oracle.candidate_union([0], 4, 10, 100).tolist() == [0, 1, 2, 3]
    assert oracle.candidate_union([1], 4, 5, 100).tolist() == [4, 5]
    assert len(oracle.candidate_union([0, 2, 3], 128, 500, 4096)) == 373
    assert oracle.candidate_union([0, 1], 4, 9, 6).tolist() == [0, 1, 2, 3, 4, 5]  # clipped to < L


# ---- hisa_select and module invariants ----
def test_hisa_regimes_and_restricted_brute_force(oracle):
    rng = np.random.default_rng(9)
    L, H, d, B, m, k = 4096, 2, 8, 64, 8, 256
    rows = np.unique(np.concatenate([np.arange(0, 40), [k - 1, k, k + 1, m * B - 1, m * B, m * B + 1, (m + 2) * B, L - 1],
                                     rng.integers(0, L, 40)])).astype(np.uint32)
    p = problem(oracle, rng.standard_normal((L, H, d)), rng.uniform(0.5, 1.5, (L, H)), rng.standard_normal((L, d)),
                np.arange(L), block_size=B, block_budget=m, token_budget=k)
    hs = oracle.select_batch("hisa", p, rows)
    ds = oracle.select_batch("dsa", p, rows)
    for i, t in enumerate(rows):
        T = hs.idx[i, :hs.count[i]]
        if t + 1 <= k:
            assert T.tolist() == list(range(t + 1))            # dense regime
        if t + 1 <= m * B:
            assert T.tolist() == ds.idx[i, :ds.count[i]].tolist()  # flat-equivalence regime
        tr = oracle.trace_row("hisa", p, int(t))
        assert set(T.tolist()) <= set(tr["omega"].tolist()) and tr["omega"].max() <= t
        assert hs.count[i] == min(k, len(tr["omega"])) and hs.cand[i] == len(tr["omega"])
        order = sorted(range(len(tr["omega"])), key=lambda j: (-tr["omega_scores"][j], tr["omega"][j]))[:k]
        assert T.tolist() == sorted(int(tr["omega"][j]) for j in order)
        assert hs.nblocks[i] <= m + 2


def test_position_equal_to_seq_len_is_streaming_query(oracle):
    rng = np.random.default_rng(10)
    L, B = 64, 8
    p = problem(oracle, rng.standard_normal((2, 2, 4)), np.ones((2, 2)), rng.standard_normal((L, 4)), [L, L - 1],
                block_size=B, block_budget=2, token_budget=8)
    r = oracle.select_batch("hisa", p)
    assert r.idx[0].tolist() == r.idx[1].tolist() or p.queries[0].tolist() != p.queries[1].tolist()
    assert r.blocks[0, r.nblocks[0] - 1] == L // B - 1
    with pytest.raises(oracle.OracleError):
        bad = problem(oracle, p.queries, p.gates, p.keys, [L + 1, 0])
        oracle.inputs_validate(bad)


def test_analytic_cost(oracle):
    p = cfgp(oracle, block_size=128, block_budget=64, token_budget=2048)
    assert oracle.analytic_cost(p, 65536, 1) == 512 + 66 * 128 == 8960   # SPEC.md:427 (H=1)
    assert oracle.analytic_cost(p, 65536, 0) == 65536
    assert oracle.analytic_cost(p, 1000, 1) == 8 + 1000
    assert oracle.analytic_cost(p, 1000, 2) == 8


def test_block_sparse_is_union_of_selected_blocks(oracle):
    rng = np.random.default_rng(11)
    L, B, m = 512, 16, 4
    p = problem(oracle, rng.standard_normal((L, 2, 4)), np.ones((L, 2)), rng.standard_normal((L, 4)), np.arange(L),
                block_size=B, block_budget=m, token_budget=m * B)
    rows = np.array([0, 17, 200, 511], np.uint32)
    r = oracle.select_batch("block", p, rows)
    for i, t in enumerate(rows):
        want = oracle.candidate_union(r.blocks[i, :r.nblocks[i]], B, int(t), L)
        assert r.idx[i, :r.count[i]].tolist() == want.tolist()


def test_non_finite_rejected(oracle):
    p = problem(oracle, [[1, np.inf]], [1], [[2, 0]], [0])
    with pytest.raises(oracle.OracleError) as e:
        oracle.inputs_validate(p)
    assert e.value.name == "NonFiniteValue"


def test_lattice_inputs_are_small_integers_with_ties(oracle):
    pos = oracle.make_positions(256, 8, "final")
    p = oracle.make_inputs("lattice", 3, 256, pos, 4, 8, block_size=16, block_budget=4, token_budget=32)
    assert set(np.unique(p.keys)) <= {-2, -1, 0, 1, 2} and set(np.unique(p.gates)) <= {1, 2, 3}
    tr = oracle.trace_row("dsa", p, 0)
    assert len(np.unique(tr["omega_scores"])) < len(tr["omega_scores"])  # exact ties exist
