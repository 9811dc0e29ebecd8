"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE, never the product).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this package.  It wraps ``_build/libvoxmi_oracle.so`` (built by
``oracle/Makefile``), a plain-C restatement of the reference `voxmi` hot path;
see voxmi_oracle.c for the per-function reference citations.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libvoxmi_oracle.so")
_lib = None

KIND = {"varz": 0, "count": 1}
SENTINEL = -1e300

_d = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.POINTER(ctypes.c_int64)
_i32 = ctypes.POINTER(ctypes.c_int32)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "voxmi_oracle.c")
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
            build()
        L = ctypes.CDLL(_SO)
        L.orc_poses_to_mats.argtypes = [_d, ctypes.c_int64, _d]
        L.orc_transform.argtypes = [_d, ctypes.c_int64, _d, _d]
        L.orc_voxel_indices.argtypes = [_d, ctypes.c_int64, _d, ctypes.c_double, _i64]
        L.orc_voxel_indices.restype = ctypes.c_int64
        L.orc_voxelize_features.argtypes = [_d, ctypes.c_int64, _d, ctypes.c_double, ctypes.c_int,
                                            _i64, _d, _i64]
        L.orc_voxelize_features.restype = ctypes.c_int64
        L.orc_joint_histogram.argtypes = [_i64, _d, ctypes.c_int64, _i64, _d, ctypes.c_int64,
                                          _i64, ctypes.c_int, ctypes.c_double, _i64]
        L.orc_joint_histogram.restype = ctypes.c_int64
        L.orc_mutual_information.argtypes = [_i64, ctypes.c_int, ctypes.c_int, _d]
        L.orc_entropy.argtypes = [_d, ctypes.c_int64]
        L.orc_entropy.restype = ctypes.c_double
        L.orc_mi_objective.argtypes = [_i64, _d, ctypes.c_int64, _i64, _d, ctypes.c_int64, _d, _d,
                                       ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       ctypes.c_int, _i32, _i64, _i64]
        L.orc_mi_objective.restype = ctypes.c_double
        L.orc_mi_objective_batch.argtypes = [_i64, _d, ctypes.c_int64, _i64, _d, ctypes.c_int64, _d,
                                             ctypes.c_int64, _d, ctypes.c_double, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                             _d, _i32]
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_bin_features.argtypes = [_d, ctypes.c_int64, ctypes.c_int, ctypes.c_double, _i64]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def poses_to_mats(poses) -> np.ndarray:
    poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 6)
    out = np.empty((poses.shape[0], 12))
    lib().orc_poses_to_mats(_p(poses, _d), poses.shape[0], _p(out, _d))
    return out


def transform(points, mat12) -> np.ndarray:
    pts = np.ascontiguousarray(points, dtype=np.float64)
    m = np.ascontiguousarray(mat12, dtype=np.float64)
    out = np.empty_like(pts)
    lib().orc_transform(_p(pts, _d), pts.shape[0], _p(m, _d), _p(out, _d))
    return out


def voxel_indices(points, origin=(0, 0, 0), res=1.0):
    pts = np.ascontiguousarray(points, dtype=np.float64)
    o = np.ascontiguousarray(origin, dtype=np.float64)
    ijk = np.empty((pts.shape[0], 3), dtype=np.int64)
    bad = lib().orc_voxel_indices(_p(pts, _d), pts.shape[0], _p(o, _d), float(res), _p(ijk, _i64))
    return ijk, int(bad)


@dataclass
class OracleFeatureMap:
    kind: str
    keys: np.ndarray
    values: np.ndarray
    bounds: np.ndarray  # (2, 3)


def feature_map(points, origin=(0, 0, 0), res=1.0, kind="varz") -> OracleFeatureMap:
    """voxelize + compute_feature_map (voxel.py:210-222, 267-295)."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    o = np.ascontiguousarray(origin, dtype=np.float64)
    n = pts.shape[0]
    keys = np.empty(max(n, 1), dtype=np.int64)
    vals = np.empty(max(n, 1))
    bounds = np.empty(6, dtype=np.int64)
    v = lib().orc_voxelize_features(_p(pts, _d), n, _p(o, _d), float(res), KIND[kind],
                                    _p(keys, _i64), _p(vals, _d), _p(bounds, _i64))
    if v < 0:
        raise OverflowError(f"point {-v - 1} leaves the voxel key range")
    return OracleFeatureMap(kind, keys[:v].copy(), vals[:v].copy(), bounds.reshape(2, 3).copy())


def joint_histogram(fa: OracleFeatureMap, fb: OracleFeatureMap, bins=32, clamp=None):
    """build_joint_histogram over compute_overlap(fa.bounds, fb.bounds)."""
    clamp = clamp if clamp is not None else (2.0 if fa.kind == "varz" else 64.0)
    mins = np.maximum(fa.bounds[0], fb.bounds[0])
    maxs = np.minimum(fa.bounds[1], fb.bounds[1])
    if (mins > maxs).any():
        return None, 0
    reg = np.ascontiguousarray(np.concatenate([mins, maxs]), dtype=np.int64)
    w = bins + 1
    counts = np.zeros((w, w), dtype=np.int64)
    total = lib().orc_joint_histogram(_p(fa.keys, _i64), _p(fa.values, _d), fa.keys.size,
                                      _p(fb.keys, _i64), _p(fb.values, _d), fb.keys.size,
                                      _p(reg, _i64), bins, float(clamp), _p(counts, _i64))
    return counts, int(total)


def mutual_information(counts, include_phi=True):
    c = np.ascontiguousarray(counts, dtype=np.int64)
    out = np.empty(4)
    rc = lib().orc_mutual_information(_p(c, _i64), c.shape[0], int(include_phi), _p(out, _d))
    if rc:
        raise ValueError("entropy of an all-zero distribution is undefined")
    return tuple(float(x) for x in out)


def mi_objective_batch(fa: OracleFeatureMap, points_b, mats, origin=(0, 0, 0), res=1.0,
                       bins=32, clamp=None, include_phi=True, threads=1):
    """mi_objective (mi.py:194-219) over P pose matrices (P, 12)."""
    clamp = clamp if clamp is not None else (2.0 if fa.kind == "varz" else 64.0)
    pts = np.ascontiguousarray(points_b, dtype=np.float64)
    mats = np.ascontiguousarray(mats, dtype=np.float64).reshape(-1, 12)
    o = np.ascontiguousarray(origin, dtype=np.float64)
    b = np.ascontiguousarray(fa.bounds.reshape(-1), dtype=np.int64)
    P = mats.shape[0]
    mi = np.empty(P)
    st = np.empty(P, dtype=np.int32)
    lib().orc_mi_objective_batch(_p(fa.keys, _i64), _p(fa.values, _d), fa.keys.size, _p(b, _i64),
                                 _p(pts, _d), pts.shape[0], _p(mats, _d), P, _p(o, _d), float(res),
                                 KIND[fa.kind], bins, float(clamp), int(include_phi), int(threads),
                                 _p(mi, _d), _p(st, _i32))
    return mi, st


def mi_objective_full(fa: OracleFeatureMap, points_b, mat, origin=(0, 0, 0), res=1.0, bins=32,
                      clamp=None, include_phi=True):
    """One pose with histogram and region total (for parity tests)."""
    clamp = clamp if clamp is not None else (2.0 if fa.kind == "varz" else 64.0)
    pts = np.ascontiguousarray(points_b, dtype=np.float64)
    m = np.ascontiguousarray(mat, dtype=np.float64)
    o = np.ascontiguousarray(origin, dtype=np.float64)
    b = np.ascontiguousarray(fa.bounds.reshape(-1), dtype=np.int64)
    w = bins + 1
    counts = np.zeros((w, w), dtype=np.int64)
    total = np.zeros(1, dtype=np.int64)
    st = np.zeros(1, dtype=np.int32)
    mi = lib().orc_mi_objective(_p(fa.keys, _i64), _p(fa.values, _d), fa.keys.size, _p(b, _i64),
                                _p(pts, _d), pts.shape[0], _p(m, _d), _p(o, _d), float(res),
                                KIND[fa.kind], bins, float(clamp), int(include_phi), _p(st, _i32),
                                _p(counts, _i64), _p(total, _i64))
    return float(mi), int(st[0]), counts, int(total[0])


def bin_features(values, bins=32, clamp=2.0) -> np.ndarray:
    """bin_features (mi.py:72-79)."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty(v.shape, dtype=np.int64)
    lib().orc_bin_features(_p(v, _d), v.size, int(bins), float(clamp), _p(out, _i64))
    return out


def max_threads() -> int:
    return int(lib().orc_max_threads())
