"""Known-answer and property tests for the downstream consumer in the CPU oracle: every worked example and
invariant SPEC.md:291-325 gives for sparse_attend / dense_attend (attention.hpp:48-59)."""
import numpy as np
import pytest


def _instance(seed, L, Q, dm):
    rng = np.random.default_rng(seed)
    lat = rng.standard_normal((L, dm)).astype(np.float32)
    qs = rng.standard_normal((Q, dm)).astype(np.float32)
    pos = np.sort(rng.integers(0, L, Q)).astype(np.uint32)
    return qs, lat, pos


def test_single_token_selection_returns_that_latent_exactly(oracle):
    qs, lat, pos = _instance(1, 16, 3, 8)
    pos[:] = 15
    sel = np.int32([[4], [0], [15]])
    out = oracle.attend_batch(qs, lat, pos, sel, np.uint32([1, 1, 1]))
    assert np.array_equal(out, lat[[4, 0, 15]])


def test_full_prefix_selection_equals_dense(oracle):
    qs, lat, pos = _instance(2, 300, 12, 24)
    sel = np.full((12, 300), -1, np.int32)
    cnt = pos + 1
    for r in range(12):
        sel[r, :cnt[r]] = np.arange(cnt[r])
    sparse = oracle.attend_batch(qs, lat, pos, sel, cnt)
    dense = oracle.attend_batch(qs, lat, pos)
    assert np.abs(sparse - dense).max() <= 1e-5


def test_weights_sum_to_one_and_are_nonnegative(oracle):
    qs, lat, pos = _instance(3, 512, 20, 32)
    pos[:] = 511
    rng = np.random.default_rng(4)
    sel = np.stack([np.sort(rng.choice(512, 64, replace=False)) for _ in range(20)]).astype(np.int32)
    out, w = oracle.attend_batch(qs, lat, pos, sel, np.full(20, 64, np.uint32), want_weights=True)
    assert (w >= 0).all() and np.abs(w.sum(axis=1) - 1.0).max() <= 1e-6
    # the output is the weighted sum of the selected latents
    want = np.einsum("rk,rkd->rd", w, lat[sel].astype(np.float64))
    assert np.abs(out - want).max() <= 1e-6


def test_dense_examples(oracle):
    lat = np.float32([[3, -1, 2]])
    out = oracle.attend_batch(np.float32([[0.5, 1, -2]]), lat, np.uint32([0]))
    assert np.array_equal(out, lat)                                   # L = 1 -> u = c_0
    rng = np.random.default_rng(5)
    lat = rng.standard_normal((40, 6)).astype(np.float32)
    out = oracle.attend_batch(np.zeros((1, 6), np.float32), lat, np.uint32([39]))
    assert np.abs(out[0] - lat.astype(np.float64).mean(axis=0)).max() <= 1e-6   # uniform scores -> the mean


def test_permutation_invariance(oracle):
    qs, lat, pos = _instance(6, 256, 5, 16)
    pos[:] = 255
    rng = np.random.default_rng(7)
    sel = np.stack([rng.choice(256, 48, replace=False) for _ in range(5)]).astype(np.int32)
    cnt = np.full(5, 48, np.uint32)
    a = oracle.attend_batch(qs, lat, pos, np.sort(sel, axis=1), cnt)
    b = oracle.attend_batch(qs, lat, pos, sel, cnt)
    assert np.abs(a - b).max() <= 1e-6


def test_default_and_explicit_scale(oracle):  # attention.hpp:20-21
    qs, lat, pos = _instance(8, 64, 4, 16)
    a = oracle.attend_batch(qs, lat, pos, scale=0.0)
    b = oracle.attend_batch(qs, lat, pos, scale=0.25)   # 1/sqrt(16)
    c = oracle.attend_batch(qs, lat, pos, scale=1.0)
    assert np.array_equal(a, b) and not np.array_equal(a, c)


def test_errors(oracle):  # attention.hpp:51-52
    qs, lat, pos = _instance(9, 32, 2, 4)
    pos[:] = [10, 20]
    with pytest.raises(oracle.OracleError) as e:
        oracle.attend_batch(qs, lat, pos, np.int32([[1, 2], [-1, -1]]), np.uint32([2, 0]))
    assert e.value.name == "EmptySelection"
    with pytest.raises(oracle.OracleError) as e:
        oracle.attend_batch(qs, lat, pos, np.int32([[1, 11], [3, 4]]), np.uint32([2, 2]))
    assert e.value.name == "CausalViolation"
    with pytest.raises(oracle.OracleError) as e:
        oracle.attend_batch(qs, lat, np.uint32([10, 32]))
    assert e.value.name == "ShapeMismatch"
    bad = lat.copy()
    bad[3, 1] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        oracle.attend_batch(qs, bad, pos)
    assert e.value.name == "NonFiniteValue"


def test_selection_results_of_all_three_strategies_are_accepted(oracle):
    L, H, d, B, m, k = 1024, 4, 16, 32, 4, 64
    pos = np.uint32([100, 700, 1023])
    prob = oracle.make_inputs("random", 11, L, pos, H, d, block_size=B, block_budget=m, token_budget=k)
    qs, lat, _ = _instance(12, L, 3, 16)
    for strat in ("dsa", "hisa", "block"):
        r = oracle.select_batch(strat, prob)
        out, w = oracle.attend_batch(qs, lat, pos, r.idx, r.count, want_weights=True)
        assert np.isfinite(out).all() and np.abs(w.sum(axis=1) - 1).max() <= 1e-6
