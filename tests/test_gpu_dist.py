"""Multi-GPU driver (hisa_cuda_dist_*, csrc/dist.cu) on the ONE GPU this run has: several logical ranks share device 0
(peer-store gather: the top-k kernel writes each row into every rank's result matrix), a one-rank NCCL communicator
exercises ncclCommInitAll / ncclCommInitRank / ncclBroadcast / the grouped per-tile gather, and the C++ driver program
checks itself against a single context. In every case the sharded result must equal the unsharded one bit for bit."""
import os
import subprocess

import numpy as np
import pytest

from paper_2603_28458_b200 import capi
from tests.gpu_helpers import round_problem_to_bf16

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _problem(oracle, L, H=64, d=128, B=128, m=4, k=512, seed=3):
    pos = np.arange(L, dtype=np.uint32)
    prob = oracle.make_inputs("random", seed, L, pos, H, d, block_size=B, block_budget=m, token_budget=k)
    qb, kb = round_problem_to_bf16(prob)
    return prob, qb, kb


def _single(prob, qb, kb, strategy):
    cfg = capi.make_config(prob.block_size, prob.block_budget, prob.token_budget, prob.H, prob.d, capi.DTYPE_BF16)
    with capi.Indexer(cfg, 0) as ix:
        ix.upload_keys(kb)
        ix.pool_build()
        return (ix.hisa_select if strategy == "hisa" else ix.dsa_select)(qb, prob.gates, prob.positions)


@pytest.mark.parametrize("strategy", ["hisa", "dsa"])
@pytest.mark.parametrize("world,L,slices", [(3, 3000, 2), (4, 6000, 3), (2, 1024, 1)])
def test_logical_ranks_peer_store_gather_equals_single_context(oracle, strategy, world, L, slices):
    prob, qb, kb = _problem(oracle, L)
    want = _single(prob, qb, kb, strategy)
    cfg = capi.make_config(prob.block_size, prob.block_budget, prob.token_budget, prob.H, prob.d, capi.DTYPE_BF16)
    with capi.Dist(cfg, devices=[0] * world) as dist:
        assert dist.world == world and dist.num_local == world and dist.gather == capi.GATHER_PEER
        dist.upload_keys(kb, L)
        rows = [capi.dist_plan(L, world, r) for r in range(world)]
        qs = [np.ascontiguousarray(qb[r]) for r in rows]
        ws = [np.ascontiguousarray(prob.gates[r]) for r in rows]
        ps = [np.ascontiguousarray(prob.positions[r]) for r in rows]
        dist.select(capi.DIST_HISA if strategy == "hisa" else capi.DIST_DSA, qs, ws, ps, L, num_slices=slices)
        for local in range(world):  # every rank holds the whole matrix
            idx, cnt = dist.fetch(L, local)
            assert np.array_equal(cnt, want["count"]), f"rank {local}: counts differ"
            assert np.array_equal(idx, want["idx"]), f"rank {local}: index matrix differs from the single-context result"
        assert dist.last_ms() > 0


def test_one_rank_nccl_communicator_and_grouped_gather(oracle):
    """world = 1 with the NCCL gather forced: ncclCommInitAll, and nothing to exchange (the code path that issues the
    per-tile broadcasts needs world > 1; the rank-mode test below drives ncclBroadcast through the key replication)."""
    L = 2000
    prob, qb, kb = _problem(oracle, L)
    want = _single(prob, qb, kb, "hisa")
    cfg = capi.make_config(prob.block_size, prob.block_budget, prob.token_budget, prob.H, prob.d, capi.DTYPE_BF16)
    with capi.Dist(cfg, devices=[0], gather=capi.GATHER_NCCL) as dist:
        assert dist.gather == capi.GATHER_NCCL
        dist.upload_keys(kb, L)
        dist.select(capi.DIST_HISA, [qb], [prob.gates], [prob.positions], L, num_slices=2)
        idx, cnt = dist.fetch(L)
        assert np.array_equal(idx, want["idx"]) and np.array_equal(cnt, want["count"])


def test_rank_mode_unique_id_and_init_rank(oracle):
    """The multi-process entry (one rank per process, as under torchrun) with world = 1: ncclGetUniqueId +
    ncclCommInitRank, keys staged and ingested through the replicated path."""
    L = 1500
    prob, qb, kb = _problem(oracle, L, m=3, k=300)
    want = _single(prob, qb, kb, "hisa")
    cfg = capi.make_config(prob.block_size, prob.block_budget, prob.token_budget, prob.H, prob.d, capi.DTYPE_BF16)
    uid = capi.dist_unique_id()
    assert len(uid) == 128 and any(uid)
    with capi.Dist(cfg, rank=0, world=1, device=0, unique_id=uid) as dist:
        assert dist.world == 1 and dist.first_rank == 0 and dist.gather == capi.GATHER_NCCL
        dist.upload_keys(kb, L)
        dist.select(capi.DIST_HISA, [qb], [prob.gates], [prob.positions], L)
        idx, cnt = dist.fetch(L)
        assert np.array_equal(idx, want["idx"]) and np.array_equal(cnt, want["count"])


def test_output_placement_rows_and_replicas(oracle):
    """hisa_cuda_set_output_placement on one context: rows land where the row map says, replicas receive the same
    rows (the mechanism under the peer-store gather), for the fused top-k variant and for the copy-kernel variants."""
    import ctypes as C
    L = 2048
    for m, k in [(4, 256), (40, 256)]:   # (m + 2) B = 768 -> warp select + copy kernel; 5376 -> fused top-k stores
        prob, qb, kb = _problem(oracle, L, m=m, k=k)
        want = _single(prob, qb, kb, "hisa")
        cfg = capi.make_config(prob.block_size, m, k, prob.H, prob.d, capi.DTYPE_BF16)
        with capi.Indexer(cfg, 0) as ix:
            ix.upload_keys(kb)
            ix.pool_build()
            perm = np.random.default_rng(1).permutation(L).astype(np.uint32)
            d_map, d_out, d_cnt = ix.device_alloc(L * 4), ix.device_alloc(L * k * 4), ix.device_alloc(L * 4)
            reps = [(ix.device_alloc(L * k * 4), ix.device_alloc(L * 4)) for _ in range(2)]
            ix.memcpy(d_map, perm, L * 4)
            ri = (C.c_void_p * 2)(*[r[0] for r in reps])
            rc = (C.c_void_p * 2)(*[r[1] for r in reps])
            capi._check(capi.lib().hisa_cuda_set_output_placement(ix._ctx, C.c_void_p(d_map), 2, ri, rc), ix._ctx)
            dq, dw, dp = ix.device_alloc(qb.nbytes), ix.device_alloc(prob.gates.nbytes), ix.device_alloc(L * 4)
            ix.memcpy(dq, qb, qb.nbytes), ix.memcpy(dw, prob.gates, prob.gates.nbytes), ix.memcpy(dp, prob.positions, L * 4)
            ix.hisa_select_raw(dq, dw, dp, L, d_out, d_cnt)
            capi._check(capi.lib().hisa_cuda_set_output_placement(ix._ctx, None, 0, None, None), ix._ctx)
            ix.synchronize()
            for oi, oc in [(d_out, d_cnt)] + reps:
                idx, cnt = np.empty((L, k), np.int32), np.empty(L, np.uint32)
                ix.memcpy(idx, oi, idx.nbytes), ix.memcpy(cnt, oc, cnt.nbytes)
                assert np.array_equal(idx[perm], want["idx"]) and np.array_equal(cnt[perm], want["count"])


def test_cpp_driver_program_checks_itself():
    """paper_2603_28458_b200/cpp/multi_bench.cpp (the C++ multi-GPU driver) with two logical ranks on device 0:
    --check compares the gathered matrix with a single-context run and exits non-zero on any difference."""
    exe = os.path.join(ROOT, "paper_2603_28458_b200", "_lib", "hisa_multi_bench")
    assert os.path.exists(exe), "hisa_multi_bench was not built (python -c 'import __graft_entry__ as g; g.build()')"
    for strategy in ("hisa", "dsa"):
        r = subprocess.run([exe, "--devices", "0,0", "--seq-len", "5000", "--block-budget", "8", "--token-budget", "512",
                            "--steps", "2", "--warmup", "1", "--slices", "2", "--strategy", strategy, "--check"],
                           capture_output=True, text=True, timeout=600)
        print(r.stdout[-1500:], r.stderr[-1500:])
        assert r.returncode == 0 and '"bit_equal_to_one_gpu": true' in r.stdout


@pytest.mark.parametrize("seed", range(int(os.environ.get("HISA_STRESS_SEEDS", "4"))))
def test_random_shard_plans_equal_single_context(oracle, seed):
    """Seeded random row counts (not multiples of the 512-row tile), world sizes up to 8 logical ranks, slice counts,
    budgets on both sides of the warp / CTA top-k boundary, random (repeated, unordered) query positions: the matrix
    every rank ends up with must equal the single-context result bit for bit."""
    rng = np.random.default_rng(300 + seed)
    L = int(rng.integers(600, 5000))
    Q = int(rng.integers(1, 4000))
    world = int(rng.choice([2, 3, 5, 8]))
    slices = int(rng.integers(1, 6))
    B = int(rng.choice([64, 128]))
    m = int(rng.choice([2, 6, 20, 40]))
    k = int(rng.integers(1, m * B + 1))
    strategy = "hisa" if rng.integers(0, 2) else "dsa"
    pos = rng.integers(0, L, Q).astype(np.uint32)
    prob = oracle.make_inputs("random", 40 + seed, L, pos, 64, 128, block_size=B, block_budget=m, token_budget=k)
    qb, kb = round_problem_to_bf16(prob)
    want = _single(prob, qb, kb, strategy)
    cfg = capi.make_config(B, m, k, 64, 128, capi.DTYPE_BF16)
    with capi.Dist(cfg, devices=[0] * world) as dist:
        dist.upload_keys(kb, L)
        rows = [capi.dist_plan(Q, world, r) for r in range(world)]
        assert sorted(np.concatenate(rows).tolist()) == list(range(Q))
        qs = [np.ascontiguousarray(qb[r]) for r in rows]
        ws = [np.ascontiguousarray(prob.gates[r]) for r in rows]
        ps = [np.ascontiguousarray(prob.positions[r]) for r in rows]
        dist.select(capi.DIST_HISA if strategy == "hisa" else capi.DIST_DSA, qs, ws, ps, Q, num_slices=slices)
        for local in {0, world - 1, int(rng.integers(0, world))}:
            idx, cnt = dist.fetch(Q, local)
            assert np.array_equal(cnt, want["count"]), f"rank {local}: counts differ (Q={Q} world={world} slices={slices})"
            assert np.array_equal(idx, want["idx"]), f"rank {local}: rows differ (Q={Q} world={world} slices={slices} m={m} k={k})"
