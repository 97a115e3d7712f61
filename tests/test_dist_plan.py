"""The row-sharding plan of the multi-GPU driver (hisa_cuda_dist_plan: pure index arithmetic in the C library, no GPU):
a partition of the rows, balanced for causal work, identical to the Python plumbing the gloo test exercises."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def capi():
    from paper_2603_28458_b200 import capi
    capi.build()
    return capi


def test_plan_is_a_partition_and_matches_the_python_sharding(capi):
    from paper_2603_28458_b200 import sharding
    for n, w in [(65536, 8), (131072, 4), (131072, 8), (6000, 3), (511, 2), (512, 2), (513, 5), (1, 1), (1048576, 8)]:
        parts = [capi.dist_plan(n, w, r) for r in range(w)]
        allrows = np.sort(np.concatenate(parts))
        assert np.array_equal(allrows, np.arange(n, dtype=np.uint32)), (n, w)
        for r in range(w):
            assert np.array_equal(parts[r], sharding.rank_rows(n, w, r).astype(np.uint32)), (n, w, r)
            assert np.all(np.diff(parts[r].astype(np.int64)) > 0)


def test_plan_balances_causal_work(capi):
    # flat indexer: work ~ sum of prefix lengths; hierarchical: ~ sum of min(t + 1, (m + 2) B)
    for n in (65536, 131072):
        for w in (2, 4, 8):
            flat = [int((capi.dist_plan(n, w, r).astype(np.int64) + 1).sum()) for r in range(w)]
            hier = [int(np.minimum(capi.dist_plan(n, w, r).astype(np.int64) + 1, 66 * 128).sum()) for r in range(w)]
            assert (max(flat) - min(flat)) / max(flat) < 0.02
            assert (max(hier) - min(hier)) / max(hier) < 0.02


def test_plan_rejects_bad_ranks(capi):
    with pytest.raises(capi.HisaError):
        capi.dist_plan(100, 2, 2)
    with pytest.raises(capi.HisaError):
        capi.dist_plan(100, 0, 0)
