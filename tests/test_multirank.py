"""Multi-rank host logic on CPU: world_size-2 gloo process group exercising the
pose sharding and the winner all-gather used by the N-GPU path."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1709_06948_b200.shard import local_winner, pick_global, shard_bounds


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mi_all, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_bounds(mi_all.shape[0], world, rank)
    v, i = local_winner(mi_all[lo:hi], lo)
    mine = torch.tensor([v, float(i)], dtype=torch.float64)
    gathered = [torch.empty(2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, mine)
    out[rank] = pick_global(torch.stack(gathered).numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["random", "tie_across_shards", "all_sentinel_but_one"])
def test_two_rank_argmax_matches_np_argmax(case):
    rng = np.random.default_rng(5)
    mi = rng.uniform(0, 1, size=1001)
    if case == "tie_across_shards":
        mi[:] = 0.25
        mi[[700, 300, 900]] = 0.75  # first max lives in rank 0's shard
    elif case == "all_sentinel_but_one":
        mi[:] = -1e300
        mi[999] = 0.01
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, free_port(), mi, out), nprocs=world, join=True)
    want = (float(mi.max()), int(np.argmax(mi)))
    assert out[0] == want and out[1] == want


def test_shard_bounds_cover_batch():
    for P in (1, 7, 64, 1000, 65536):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(P, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == P
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b


def test_pick_global_first_index_rule():
    w = np.array([[0.5, 40.0], [0.5, 10.0], [0.2, 0.0]])
    assert pick_global(w) == (0.5, 10)


def _subgroup_worker(rank, world, port, mi_all, out):
    from paper_1709_06948_b200.shard import all_gather_winner
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sub = dist.new_group([0, 1])  # every rank calls new_group; rank 2 stays out
    if rank in (0, 1):
        r = dist.get_rank(sub)
        lo, hi = shard_bounds(mi_all.shape[0], 2, r)
        v, i = local_winner(mi_all[lo:hi], lo)
        out[rank] = all_gather_winner(v, i, dist, torch.device("cpu"), group=sub)
    else:  # a rank outside the subgroup works on something else meanwhile
        out[rank] = None
    dist.barrier()
    dist.destroy_process_group()


def test_winner_exchange_on_a_subgroup():
    """all_gather_winner honours its group: 2 of 3 ranks shard one batch, the
    third never joins the collective (it used to hang / mix)."""
    rng = np.random.default_rng(9)
    mi = rng.uniform(0, 1, size=777)
    mi[[400, 100]] = 2.0  # first max in the subgroup's rank-0 shard
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_subgroup_worker, args=(3, free_port(), mi, out), nprocs=3, join=True)
    want = (2.0, 100)
    assert out[0] == want and out[1] == want and out[2] is None


def test_pick_global_pairs_int64_index_exact():
    from paper_1709_06948_b200.shard import pick_global_pairs
    big = (1 << 60) + 1  # not representable as float64
    assert pick_global_pairs([0.5, 0.5], [big + 2, big]) == (0.5, big)
