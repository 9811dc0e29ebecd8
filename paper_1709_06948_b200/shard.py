"""Multi-GPU pose sharding.

Candidate poses are independent, so a batch is split into contiguous index
ranges, one per rank, with scan A's grid and scan B replicated on every GPU
(built locally; no broadcast).  The only exchange is the per-rank winner
(max MI, global index): one all-gather of 16 bytes per rank over NCCL, after
which every rank applies np.argmax's first-max rule.
"""

from __future__ import annotations

import numpy as np


def shard_bounds(P: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) range of rank ``rank`` (sizes differ by at most ceil)."""
    per = -(-P // world) if world > 0 else P
    lo = min(P, rank * per)
    return lo, min(P, lo + per)


def local_winner(mi: np.ndarray, offset: int) -> tuple[float, int]:
    """np.argmax of one shard, as (value, global index); empty -> (-inf, big)."""
    if mi.size == 0:
        return float("-inf"), np.iinfo(np.int64).max
    k = int(np.argmax(mi))
    return float(mi[k]), offset + k


def pick_global(winners: np.ndarray) -> tuple[float, int]:
    """(W, 2) [mi, index] rows -> the np.argmax winner over the whole batch:
    largest MI, lowest global index among equal maxima."""
    w = np.asarray(winners, dtype=np.float64).reshape(-1, 2)
    k = int(np.lexsort((w[:, 1], -w[:, 0]))[0])
    return float(w[k, 0]), int(w[k, 1])


def all_gather_winner(value: float, index: int, dist, device, group=None) -> tuple[float, int]:
    """Exchange per-rank winners over ``group`` (default: WORLD) with
    torch.distributed (NCCL or gloo).  The global index travels as an int64
    (the MI as a float64 in a separate tensor), so it is exact at any size."""
    import torch
    world = dist.get_world_size(group)
    mine_v = torch.tensor([value], dtype=torch.float64, device=device)
    mine_i = torch.tensor([index], dtype=torch.int64, device=device)
    out_v = torch.empty(world, dtype=torch.float64, device=device)
    out_i = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out_v, mine_v, group=group)
    dist.all_gather_into_tensor(out_i, mine_i, group=group)
    return pick_global_pairs(out_v.cpu().numpy(), out_i.cpu().numpy())


def pick_global_pairs(values: np.ndarray, indices: np.ndarray) -> tuple[float, int]:
    """pick_global on separate (mi, int64 index) arrays: largest MI, lowest
    global index among equal maxima (np.argmax's rule, cli.py:202)."""
    v = np.asarray(values, dtype=np.float64).ravel()
    i = np.asarray(indices, dtype=np.int64).ravel()
    k = int(np.lexsort((i, -v))[0])
    return float(v[k]), int(i[k])
