"""Query-row sharding for the multi-GPU driver (one process per GPU).

Every query row is independent (reference: SPEC.md:155,246), so the path shards over rows of L; the only
shared state is the read-only key sequence (replicated by broadcast) and the only exchange is the all-gather
of the int32 index rows. Causal work grows with the row index, so rows are dealt out in round-robin TILES
rather than contiguous chunks, in zig-zag order. This module is pure index arithmetic + torch.distributed
plumbing; it works on any backend (the CPU tests use gloo)."""
from __future__ import annotations

import numpy as np

TILE_ROWS = 512


def rank_rows(num_rows: int, world: int, rank: int, tile: int = TILE_ROWS) -> np.ndarray:
    """Sorted global row indices owned by `rank`."""
    tiles = np.arange((num_rows + tile - 1) // tile)
    # zig-zag deal (0 1 .. W-1 W-1 .. 1 0 0 1 ..): keeps the triangular (flat-indexer) work balanced too
    phase = tiles % (2 * world)
    owner = np.where(phase < world, phase, 2 * world - 1 - phase)
    mine = tiles[owner == rank]
    rows = (mine[:, None] * tile + np.arange(tile)[None, :]).reshape(-1)
    return rows[rows < num_rows]


def padded_rows_per_rank(num_rows: int, world: int, tile: int = TILE_ROWS) -> int:
    """all_gather needs equal shapes: every rank pads its row count to this."""
    return max(len(rank_rows(num_rows, world, r, tile)) for r in range(world))


def gathered_row_order(num_rows: int, world: int, tile: int = TILE_ROWS) -> np.ndarray:
    """Global row index of every entry of the rank-major gathered buffer [world * padded, k]; -1 marks padding."""
    pad = padded_rows_per_rank(num_rows, world, tile)
    out = np.full(world * pad, -1, dtype=np.int64)
    for r in range(world):
        rows = rank_rows(num_rows, world, r, tile)
        out[r * pad:r * pad + len(rows)] = rows
    return out


def broadcast_keys(keys, dist, src: int = 0):
    """Replicates the key sequence (torch tensor, any device) from `src` to every rank."""
    dist.broadcast(keys, src=src)
    return keys


def all_gather_indices(local_idx, num_rows: int, dist, tile: int = TILE_ROWS):
    """local_idx: [n_local, k] int32 tensor for this rank's rows (rank_rows order). Returns the full
    [num_rows, k] tensor in global row order on every rank."""
    import torch
    world, rank = dist.get_world_size(), dist.get_rank()
    pad = padded_rows_per_rank(num_rows, world, tile)
    k = local_idx.shape[1]
    buf = torch.full((pad, k), -1, dtype=local_idx.dtype, device=local_idx.device)
    buf[:local_idx.shape[0]] = local_idx
    gathered = torch.empty((world * pad, k), dtype=local_idx.dtype, device=local_idx.device)
    dist.all_gather_into_tensor(gathered, buf)
    order = gathered_row_order(num_rows, world, tile)
    keep = torch.from_numpy(np.nonzero(order >= 0)[0]).to(local_idx.device)
    dest = torch.from_numpy(order[order >= 0]).to(local_idx.device)
    full = torch.empty((num_rows, k), dtype=local_idx.dtype, device=local_idx.device)
    full[dest] = gathered[keep]
    return full
