"""Shared fixtures.  `-m gpu` tests need a B200 and the in-tree libvmi.so;
everything else runs on CPU (oracle vs golden vectors, host logic, C-ABI
symbol checks, gloo multi-rank tests)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device and libvmi.so")


def golden(name: str):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def small_scene(seed: int, n: int) -> np.ndarray:
    """The reference test scene (test_mi.py:303-307), regenerated from its seed."""
    rng = np.random.default_rng(seed)
    pts = rng.uniform(-15, 15, size=(n, 3))
    pts[:, 2] = rng.uniform(0, 4, size=n) * (pts[:, 0] > 0)
    return pts


SMALL_CASES = ("s0", "s1", "s2", "s3", "s4", "s5")


def small_case(tag: str):
    g = golden("small_golden.npz")
    seed, n = (int(x) for x in g[f"{tag}_seed"])
    meta = g[f"{tag}_meta"]
    return {
        "a": small_scene(seed, n),
        "b": small_scene(seed + 100, n),
        "res": float(meta[0]),
        "origin": np.asarray(meta[1:4], dtype=np.float64),
        "kind": "varz" if int(meta[4]) == 0 else "count",
        "phi": bool(int(meta[5])),
        "poses": g[f"{tag}_poses"],
        "mi": g[f"{tag}_mi"],
        "status": g[f"{tag}_status"],
        "hist": g[f"{tag}_hist"].astype(np.int64),
        "total": g[f"{tag}_total"],
        "a_keys": g[f"{tag}_a_keys"],
        "a_values": g[f"{tag}_a_values"],
        "a_bounds": g[f"{tag}_a_bounds"],
        "digest": str(g[f"{tag}_digest"]),
    }


_HDL = {}


def hdl_pair():
    """The HDL-64-shaped C2 scan pair (regenerated; digest pinned by golden)."""
    if "pair" not in _HDL:
        from paper_1709_06948_b200.synth import LidarSceneSpec, hdl64_pair
        from paper_1709_06948_b200.geometry import EulerPose
        _HDL["pair"] = hdl64_pair(LidarSceneSpec(), EulerPose(1.5, 0.3, 0.0, 0.0, 0.0, 0.05))
    return _HDL["pair"]


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def hdl():
    return hdl_pair()
