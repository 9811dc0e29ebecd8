"""Sharded search and device top-K on the GPU.

The N-GPU path is exercised with two ranks of a gloo process group that both
use cuda:0 (one GPU is all this box has): each rank scores its own contiguous
shard, re-scores its shard winner from the bit-exact histogram, and the
all-gather of (mi, index) must pick exactly what one process picks over the
whole candidate list.  The ranks' kernels never wait on one another.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import paper_1709_06948_b200 as vmi
from conftest import hdl_pair

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case():
    a, b = hdl_pair()
    from paper_1709_06948_b200.synth import candidate_batch
    poses = candidate_batch(vmi.EulerPose(1.5, 0.3, 0, 0, 0, 0.05), 3001, seed=77)
    return a[:, :3].astype(np.float64), b, poses


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    a, b, poses = _case()
    r = vmi.grid_search_sharded(a, b, poses, device=0)
    out[rank] = (r.best_index, r.best_mi, int(r.mi.size))
    dist.destroy_process_group()


def test_two_rank_sharded_search_matches_single_process():
    import torch.multiprocessing as mp
    a, b, poses = _case()
    want = vmi.grid_search(a, b, poses)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0][0] == out[1][0] == want.best_index
    assert out[0][1] == out[1][1]
    np.testing.assert_allclose(out[0][1], want.best_mi, rtol=1e-12)
    assert out[0][2] + out[1][2] == poses.shape[0]


def test_device_topk_matches_stable_sort():
    a, b, poses = _case()
    eng = vmi.MIEngine(grid=vmi.GridSpec(resolution=1.0),
                       binning=vmi.BinningSpec(kind=vmi.FeatureKind.VARZ))
    eng.set_reference(a, fetch=False)
    eng.set_query(b)
    mi_h, _ = eng.evaluate(poses)
    mi_d, st_d = eng.evaluate_device(poses)
    np.testing.assert_array_equal(mi_d.cpu().numpy(), mi_h)
    for k in (1, 7, 64, poses.shape[0] + 5):
        vals, idx = eng.topk(poses, k)
        order = np.lexsort((np.arange(mi_h.size), -mi_h))[:k]
        np.testing.assert_array_equal(idx, order)
        np.testing.assert_array_equal(vals, mi_h[order])
    assert eng.topk(poses, 1)[1][0] == int(np.argmax(mi_h))
    # ties keep candidate order
    dup = np.repeat(poses[:5], 3, axis=0)
    vals, idx = eng.topk(dup, 15)
    mi_dup, _ = eng.evaluate(dup)
    np.testing.assert_array_equal(idx, np.lexsort((np.arange(15), -mi_dup)))
    eng.close()
