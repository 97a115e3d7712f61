"""Multi-process (world_size 2, gloo, CPU) test of the query-row sharding used by bench.py --gpus N:
keys are broadcast, each rank selects for its round-robin tiles, indices are all-gathered back into global
row order. The per-rank "selection" here is the CPU oracle (test infrastructure) standing in for the GPU
call, so the test checks exactly the distributed plumbing: G-rank result == 1-rank result, bit for bit."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_rank_rows_partition():
    from paper_2603_28458_b200 import sharding
    for n, w, tile in [(65536, 8, 512), (1000, 3, 64), (5, 4, 2), (4096, 2, 512)]:
        parts = [sharding.rank_rows(n, w, r, tile) for r in range(w)]
        allrows = np.sort(np.concatenate(parts))
        assert allrows.tolist() == list(range(n))
        order = sharding.gathered_row_order(n, w, tile)
        assert sorted(order[order >= 0].tolist()) == list(range(n))
    # causal balance: with round-robin tiles the summed prefix length differs by < 2 % across 8 ranks
    work = [int((sharding.rank_rows(65536, 8, r) + 1).sum()) for r in range(8)]
    assert (max(work) - min(work)) / max(work) < 0.02


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import pyoracle
    from paper_2603_28458_b200 import sharding
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = Q = 768
    H, d, B, m, k, tile = 4, 16, 32, 4, 64, 64
    pos = np.arange(Q, dtype=np.uint32)
    prob = pyoracle.make_inputs("random", 1, L, pos, H, d, block_size=B, block_budget=m, token_budget=k)
    keys = torch.from_numpy(prob.keys.copy())
    if rank != 0:
        keys.zero_()                      # only rank 0 holds the sequence before the broadcast
    sharding.broadcast_keys(keys, dist, src=0)
    prob.keys = keys.numpy()
    rows = sharding.rank_rows(Q, world, rank, tile)
    local = pyoracle.select_batch("hisa", prob, rows.astype(np.uint32), threads=1)
    full = sharding.all_gather_indices(torch.from_numpy(local.idx), Q, dist, tile)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), full.numpy())
    dist.destroy_process_group()


def test_two_rank_gather_equals_single_rank(tmp_path, oracle):
    import torch.multiprocessing as mp
    port = 29500 + (os.getpid() % 2000)
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "rank0.npy")
    r1 = np.load(tmp_path / "rank1.npy")
    assert np.array_equal(r0, r1)
    pos = np.arange(768, dtype=np.uint32)
    prob = oracle.make_inputs("random", 1, 768, pos, 4, 16, block_size=32, block_budget=4, token_budget=64)
    single = oracle.select_batch("hisa", prob)
    assert np.array_equal(r0, single.idx)
