"""GPU parity of the downstream consumer (hisa_cuda_sparse_attend / _dense_attend) against the CPU oracle's
sparse_attend / dense_attend (attention.hpp:48-59), through the C ABI.

Tolerance: the oracle computes in f64 over f32 storage, the kernel in fp32 (exact products for bf16 storage, fp32
accumulation); outputs are convex combinations of O(1) latents, so 1e-5 absolute is asserted for f32
storage and bf16 storage alike (the oracle consumes the bf16-rounded values widened to f32)."""
import numpy as np
import pytest

from paper_2603_28458_b200 import capi

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _indexer():
    return capi.Indexer(capi.make_config(128, 64, 2048, 64, 128, capi.DTYPE_BF16), 0)


def _instance(seed, L, Q, dm, bf16):
    rng = np.random.default_rng(seed)
    lat = rng.standard_normal((L, dm)).astype(np.float32)
    qs = rng.standard_normal((Q, dm)).astype(np.float32)
    pos = np.sort(rng.integers(0, L, Q)).astype(np.uint32)
    if bf16:
        lb, qb = capi.f32_to_bf16_bits(lat), capi.f32_to_bf16_bits(qs)
        return qb, lb, pos, capi.bf16_bits_to_f32(qb), capi.bf16_bits_to_f32(lb)
    return qs, lat, pos, qs, lat


def _random_selection(rng, pos, k):
    Q = pos.shape[0]
    sel = np.full((Q, k), -1, np.int32)
    cnt = np.zeros(Q, np.uint32)
    for r in range(Q):
        n = min(k, int(pos[r]) + 1)
        sel[r, :n] = np.sort(rng.choice(int(pos[r]) + 1, n, replace=False))
        cnt[r] = n
    return sel, cnt


@pytest.mark.parametrize("bf16", [False, True])
@pytest.mark.parametrize("dm", [128, 64, 32, 100, 7, 256, 512])
def test_sparse_attend_matches_oracle(oracle, dm, bf16):
    L, Q, k = 3000, 97, 200
    q_in, l_in, pos, q_f, l_f = _instance(dm, L, Q, dm, bf16)
    sel, cnt = _random_selection(np.random.default_rng(dm + 1), pos, k)
    with _indexer() as ix:
        ix.attn_set_latents(l_in)
        out, w = ix.sparse_attend(q_in, pos, sel, cnt, want_weights=True)
        out_nocount = ix.sparse_attend(q_in, pos, sel)      # padding skipped without a count array
    want, ww = oracle.attend_batch(q_f, l_f, pos, sel, cnt, want_weights=True)
    assert np.abs(out - want).max() <= TOL
    assert np.abs(w - ww).max() <= TOL
    assert np.abs(w.sum(axis=1) - 1).max() <= 1e-5 and (w >= 0).all()
    assert (w[sel < 0] == 0).all()
    assert np.array_equal(out, out_nocount)


@pytest.mark.parametrize("bf16", [False, True])
def test_dense_attend_and_sparse_dense_identity(oracle, bf16):
    L, Q, dm = 2048, 64, 128
    q_in, l_in, pos, q_f, l_f = _instance(21, L, Q, dm, bf16)
    pos[-1] = L - 1
    pos[0] = 0
    sel = np.full((Q, L), -1, np.int32)
    for r in range(Q):
        sel[r, :pos[r] + 1] = np.arange(pos[r] + 1)
    with _indexer() as ix:
        ix.attn_set_latents(l_in)
        dense = ix.dense_attend(q_in, pos)
        sparse = ix.sparse_attend(q_in, pos, sel, pos + 1)
    want = oracle.attend_batch(q_f, l_f, pos)
    assert np.abs(dense - want).max() <= TOL
    assert np.abs(sparse - dense).max() <= TOL
    assert np.array_equal(dense[0], l_f[0])                      # L = 1 prefix -> u = c_0 exactly


def test_spec_examples(oracle):
    rng = np.random.default_rng(5)
    lat = rng.standard_normal((40, 6)).astype(np.float32)
    qs = rng.standard_normal((3, 6)).astype(np.float32)
    with _indexer() as ix:
        ix.attn_set_latents(lat)
        one = ix.sparse_attend(qs, np.uint32([39, 39, 39]), np.int32([[4], [0], [39]]), np.uint32([1, 1, 1]))
        assert np.array_equal(one, lat[[4, 0, 39]])              # single token -> that latent exactly
        mean = ix.dense_attend(np.zeros((1, 6), np.float32), np.uint32([39]))
        assert np.abs(mean[0] - lat.astype(np.float64).mean(axis=0)).max() <= 1e-6   # uniform scores -> the mean
        sel = np.stack([rng.choice(40, 17, replace=False) for _ in range(3)]).astype(np.int32)
        a = ix.sparse_attend(qs, np.uint32([39] * 3), sel, scale=0.7)
        b = ix.sparse_attend(qs, np.uint32([39] * 3), np.sort(sel, axis=1), scale=0.7)
        assert np.abs(a - b).max() <= 1e-6                       # permutation invariance
        want = oracle.attend_batch(qs, lat, np.uint32([39] * 3), sel, np.uint32([17] * 3), scale=0.7)
        assert np.abs(a - want).max() <= TOL


def test_consumes_the_selection_matrices_of_all_three_strategies(oracle):
    L, H, d, B, m, k = 4096, 64, 128, 128, 4, 256
    pos = np.arange(0, L, 5, dtype=np.uint32)
    prob = oracle.make_inputs("random", 3, L, pos, H, d, block_size=B, block_budget=m, token_budget=k)
    qb, kb = capi.f32_to_bf16_bits(prob.queries), capi.f32_to_bf16_bits(prob.keys)
    rng = np.random.default_rng(8)
    lat = rng.standard_normal((L, 128)).astype(np.float32)
    hs = rng.standard_normal((pos.shape[0], 128)).astype(np.float32)
    cfg = capi.make_config(B, m, k, H, d, capi.DTYPE_BF16)
    with capi.Indexer(cfg, 0) as ix:
        ix.upload_keys(kb)
        ix.pool_build()
        ix.attn_set_latents(lat)
        for name in ("hisa", "dsa", "block"):
            r = getattr(ix, {"hisa": "hisa_select", "dsa": "dsa_select", "block": "block_sparse_select"}[name])(qb, prob.gates, pos)
            out = ix.sparse_attend(hs, pos, r["idx"], r["count"])
            want = oracle.attend_batch(hs, lat, pos, r["idx"], r["count"])
            assert np.abs(out - want).max() <= TOL, name


def test_error_behaviour():  # attention.hpp:51-52
    rng = np.random.default_rng(9)
    lat = rng.standard_normal((32, 4)).astype(np.float32)
    qs = rng.standard_normal((2, 4)).astype(np.float32)
    pos = np.uint32([10, 20])
    with _indexer() as ix:
        with pytest.raises(capi.HisaError) as e:
            ix._attn_dm = 4
            ix.dense_attend(qs, pos)
        assert e.value.name == "EmptySequence"
        ix.attn_set_latents(lat)
        with pytest.raises(capi.HisaError) as e:
            ix.sparse_attend(qs, pos, np.int32([[1, 2], [-1, -1]]), np.uint32([2, 0]))
        assert e.value.name == "EmptySelection"
        with pytest.raises(capi.HisaError) as e:
            ix.sparse_attend(qs, pos, np.int32([[1, 11], [3, 4]]), np.uint32([2, 2]))
        assert e.value.name == "CausalViolation"
        with pytest.raises(capi.HisaError) as e:
            ix.dense_attend(qs, np.uint32([10, 32]))
        assert e.value.name == "ShapeMismatch"
        bad = lat.copy()
        bad[3, 1] = np.nan
        with pytest.raises(capi.HisaError) as e:
            ix.attn_set_latents(bad, check_finite=True)
        assert e.value.name == "NonFiniteValue"
        with pytest.raises(capi.HisaError) as e:
            ix.attn_set_latents(np.zeros((4, 513), np.float32))
        assert e.value.name == "Unsupported"


def test_full_size_k2048_rows_against_sampled_oracle(oracle):
    """Headline shape of the consumer: L = 64K latents, k = 2048 selected tokens per row, d_model = 128, bf16."""
    L, Q, k, dm = 65536, 4096, 2048, 128
    rng = np.random.default_rng(31)
    lb = capi.f32_to_bf16_bits(rng.standard_normal((L, dm)).astype(np.float32))
    qb = capi.f32_to_bf16_bits(rng.standard_normal((Q, dm)).astype(np.float32))
    pos = np.sort(rng.integers(k, L, Q)).astype(np.uint32)
    sel = np.sort((rng.random((Q, k)) * (pos[:, None] + 1)).astype(np.int32), axis=1)
    with _indexer() as ix:
        ix.attn_set_latents(lb)
        out = ix.sparse_attend(qb, pos, sel, scale=0.05)
        assert ix.attn_last_ms() > 0
    rows = np.arange(0, Q, 37, dtype=np.uint32)
    want = oracle.attend_batch(capi.bf16_bits_to_f32(qb), capi.bf16_bits_to_f32(lb), pos, sel[rows], np.full(rows.shape[0], k, np.uint32),
                               rows=rows, scale=0.05)
    assert np.abs(out[rows] - want).max() <= TOL


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("HISA_STRESS_SEEDS", "10"))))
def test_random_shapes_against_oracle(oracle, seed):
    """Seeded random (L, Q, d_model, k, storage, scale) with ragged selections: duplicates, unsorted order, counts from 1
    to k, padding entries inside the counted range (skipped by both sides), query positions 0 and L - 1."""
    rng = np.random.default_rng(7000 + seed)
    dm = int(rng.choice([1, 3, 16, 31, 33, 64, 65, 96, 128, 129, 200, 256, 384, 512]))
    L = int(rng.integers(1, 5000))
    Q = int(rng.integers(1, 150))
    k = int(rng.integers(1, 300))
    bf16 = bool(rng.integers(0, 2))
    scale = float(rng.choice([0.0, 0.01, 0.3]))
    q_in, l_in, pos, q_f, l_f = _instance(8000 + seed, L, Q, dm, bf16)
    pos[0], pos[-1] = 0, L - 1
    pos.sort()
    sel = np.full((Q, k), -1, np.int32)
    cnt = np.zeros(Q, np.uint32)
    for r in range(Q):
        n = int(rng.integers(1, k + 1))
        sel[r, :n] = rng.integers(0, int(pos[r]) + 1, n)          # duplicates and arbitrary order allowed
        if n > 2 and rng.random() < 0.3:
            sel[r, int(rng.integers(1, n))] = -1                   # a hole inside the counted range
        cnt[r] = n
    with _indexer() as ix:
        ix.attn_set_latents(l_in)
        out, w = ix.sparse_attend(q_in, pos, sel, cnt, scale=scale, want_weights=True)
    # the oracle takes exact index lists: drop the holes, remember where the kept entries sat
    want = np.zeros((Q, dm), np.float32)
    ww = np.zeros((Q, k), np.float64)
    for r in range(Q):
        keep = np.flatnonzero(sel[r, :cnt[r]] >= 0)
        o, wr = oracle.attend_batch(q_f, l_f, pos, sel[r:r + 1, keep], np.uint32([keep.size]), rows=np.uint32([r]), scale=scale,
                                    want_weights=True)
        want[r], ww[r, keep] = o[0], wr[0]
    assert np.abs(out - want).max() <= TOL, (dm, L, Q, k, bf16)
    assert np.abs(w - ww).max() <= TOL


@pytest.mark.parametrize("dm", [64, 100, 128, 256])
def test_bf16_simt_and_mma_kernels_agree_with_the_oracle(oracle, dm, monkeypatch):
    """bf16 latents run on the warp-MMA kernel (d_model <= 256); HISA_ATTEND_SIMT=1 keeps them on the SIMT kernel. Both
    must meet the oracle tolerance, weights included, and agree with each other well inside it."""
    L, Q, k = 2500, 61, 150
    q_in, l_in, pos, q_f, l_f = _instance(40 + dm, L, Q, dm, True)
    sel, cnt = _random_selection(np.random.default_rng(41 + dm), pos, k)
    res = {}
    for simt in ("0", "1"):
        monkeypatch.setenv("HISA_ATTEND_SIMT", simt)
        with _indexer() as ix:
            ix.attn_set_latents(l_in)
            res[simt] = ix.sparse_attend(q_in, pos, sel, cnt, want_weights=True)
    want, ww = oracle.attend_batch(q_f, l_f, pos, sel, cnt, want_weights=True)
    for out, w in res.values():
        assert np.abs(out - want).max() <= TOL and np.abs(w - ww).max() <= TOL
    assert np.abs(res["0"][0] - res["1"][0]).max() <= 2e-6
