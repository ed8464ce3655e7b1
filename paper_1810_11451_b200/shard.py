"""Multi-GPU partitioning of the beamforming work.

Every block's output depends only on its own S and its group's W, so the path
shards with no data-path collective: W is replicated (one broadcast over
NCCL / NVLink at setup), blocks are split across ranks, and the only other
collective is a scalar max of the timings.  Host-side logic only; the
partition is a pure function of the tags, so every rank computes it locally.

* c4 "sharded by subband" (BASELINE.json configs[3]): blocks are ordered by
  (tag, block id) and that order is cut into `world` equal contiguous pieces,
  so each rank holds whole runs of a few subbands and the load is balanced to
  one block (contiguous subband ranges would cap efficiency at
  55 / (G * ceil(55 / G))).  Within a rank blocks keep ascending block-id order
  (bf_apply routes them again locally).
* untagged workloads (c2, c3): contiguous, balanced block ranges.
* c5 (4096-block chunks dealt to cells by chunk id c mod 8): chunks are beamformed in
  windows of 8 consecutive chunks (one of every cell, one bf_apply_batch launch each) and
  whole windows are dealt round-robin to ranks (window w -> rank w mod world), so every
  rank holds the same mix of cells' f by construction and each launch keeps whole
  4096-block chunks (splitting every chunk would leave 512 blocks per rank at 8 GPUs,
  ~3.5 per CTA: fill and drain would dominate).  Not c mod world: with 8 ranks that would
  pin one cell (one f) per GPU and imbalance the load up to 36x.
"""
from __future__ import annotations

import numpy as np


def even_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """[first, first + count) of rank's balanced contiguous share of n items."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank / world")
    first = n * rank // world
    return first, n * (rank + 1) // world - first


def subband_shard(tags: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Block ids (ascending int64) of rank's share, cut from the (tag, id) order."""
    order = np.argsort(np.asarray(tags), kind="stable")
    first, count = even_range(len(order), rank, world)
    return np.sort(order[first:first + count]).astype(np.int64)


def chunk_shard(chunk: int, chunk_blocks: int, rank: int, world: int) -> tuple[int, int]:
    """Global [first, first + count) of rank's share of one c5 chunk."""
    f0, c = even_range(chunk_blocks, rank, world)
    return chunk * chunk_blocks + f0, c


def window_shard(n_chunks: int, window: int, rank: int, world: int) -> list[list[int]]:
    """c5: the windows (lists of consecutive chunk ids, `window` per window, the last one
    possibly shorter) that rank processes, window w -> rank w mod world, in order."""
    if world < 1 or not (0 <= rank < world) or window < 1:
        raise ValueError("bad rank / world / window")
    n_win = (n_chunks + window - 1) // window
    return [list(range(w * window, min((w + 1) * window, n_chunks)))
            for w in range(rank, n_win, world)]


def broadcast_precoders(W, src: int = 0):
    """Replicate W (a tensor on this rank's device) from rank `src` (NCCL or gloo)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast(W, src=src)
    return W


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
