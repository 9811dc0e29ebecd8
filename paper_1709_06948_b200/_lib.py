"""ctypes binding of libvmi.so (include/vmi.h).

The library is built in-tree (``build.py``) and is REQUIRED: there is no CPU
fallback.  Importing the package works without it (so CPU-only tooling can
inspect the API), but every call that needs the GPU raises ``VmiError`` when
the library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# VMI_LIB overrides the library path (A/B experiments with variant builds)
LIB_PATH = os.environ.get("VMI_LIB") or os.path.join(HERE, "_native", "libvmi.so")

VMI_OK, VMI_EMPTY_REGION, VMI_KEY_RANGE, VMI_PHI_OFF_EMPTY = 0, 1, 2, 3
VMI_FLAG_RECHECK = 0x100
SENTINEL = -1e300

# every exported symbol of include/vmi.h (checked by tests/test_boundary.py)
EXPORTS = (
    "vmi_create", "vmi_destroy", "vmi_last_error", "vmi_version", "vmi_set_params",
    "vmi_set_reference_points", "vmi_set_reference_records_f32", "vmi_set_reference_features", "vmi_get_reference_features",
    "vmi_set_query_points", "vmi_set_query_records_f32", "vmi_set_query_hull",
    "vmi_poses_to_mats", "vmi_eval",
    "vmi_eval_poses", "vmi_eval_device", "vmi_eval_fixups", "vmi_eval_rot_device", "vmi_eval_exact",
    "vmi_query_features",
    "vmi_fast_features",
    "vmi_argmax_device", "vmi_topk_device", "vmi_launch_count", "vmi_set_tuning", "vmi_set_passes",
    "vmi_nm_run", "vmi_set_pairs", "vmi_eval_pairs", "vmi_align_pairs", "vmi_get_counters",
)


# vmi_nm_eval_fn: (user, poses, run, n, g, h) -> int
NM_EVAL_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                              ctypes.POINTER(ctypes.c_int32), ctypes.c_int64,
                              ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64))
NM_TERMINATION = ("converged_f", "converged_x", "max_iter")


def nm_outputs(K: int, trace_cap: int) -> dict:
    """Host output arrays of the lockstep Nelder-Mead entry points."""
    return {"best_x": np.zeros((K, 6)), "best_value": np.zeros(K),
            "iterations": np.zeros(K, np.int32), "termination": np.zeros(K, np.int32),
            "n_evaluations": np.zeros(K, np.int32), "uncertain": np.zeros(K, np.int32),
            "trace": np.zeros((K, trace_cap)), "trace_len": np.zeros(K, np.int32)}


def nm_out_args(o: dict) -> list:
    return [ptr(o["best_x"], _d), ptr(o["best_value"], _d), ptr(o["iterations"], _i32),
            ptr(o["termination"], _i32), ptr(o["n_evaluations"], _i32),
            ptr(o["uncertain"], _i32), ptr(o["trace"], _d), ptr(o["trace_len"], _i32)]


def nm_run(x0: np.ndarray, steps, max_iterations: int, f_tol: float, x_tol: float,
           restarts: int, f_batch, spec_budget: int = -1) -> dict:
    """vmi_nm_run with a Python objective: ``f_batch(poses (n, 6), run (n,))`` ->
    (values (n,), identities (n,) uint64).  Returns the output arrays."""
    x0 = np.ascontiguousarray(x0, dtype=np.float64).reshape(-1, 6)
    K = x0.shape[0]
    st = np.ascontiguousarray(steps, dtype=np.float64).reshape(6)
    cap = max_iterations + restarts + 2
    o = nm_outputs(K, cap)
    err = []

    def cb(user, poses, run, n, g, h):
        try:
            P = np.ctypeslib.as_array(poses, shape=(n, 6)).copy()
            R = np.ctypeslib.as_array(run, shape=(n,)).copy()
            vals, ids = f_batch(P, R)
            np.ctypeslib.as_array(g, shape=(n,))[:] = -np.asarray(vals, dtype=np.float64)
            np.ctypeslib.as_array(h, shape=(n,))[:] = np.asarray(ids, dtype=np.uint64)
            return 0
        except Exception as e:  # noqa: BLE001 -- surfaced after the native call returns
            err.append(e)
            return -1
    fn = NM_EVAL_FN(cb)
    rc = load().vmi_nm_run(K, ptr(x0, _d), ptr(st, _d), int(max_iterations), float(f_tol),
                           float(x_tol), int(restarts), int(spec_budget), fn, None,
                           *nm_out_args(o), cap)
    if err:
        raise err[0]
    if rc:
        raise VmiError(f"vmi_nm_run failed ({rc})")
    return o


class VmiError(RuntimeError):
    """Raised when the native library reports an error (or is missing)."""


_lib = None

_d = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.POINTER(ctypes.c_int64)
_i32 = ctypes.POINTER(ctypes.c_int32)
_f = ctypes.POINTER(ctypes.c_float)
_vp = ctypes.c_void_p
_ctx = ctypes.c_void_p


def load(path: str = LIB_PATH):
    """Load libvmi.so and declare argtypes; raise VmiError if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise VmiError(
            f"{path} is missing: build it with `python -m paper_1709_06948_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    L.vmi_create.argtypes = [ctypes.c_int, ctypes.POINTER(_ctx)]
    L.vmi_destroy.argtypes = [_ctx]
    L.vmi_last_error.argtypes = [_ctx]
    L.vmi_last_error.restype = ctypes.c_char_p
    L.vmi_version.restype = ctypes.c_char_p
    L.vmi_set_params.argtypes = [_ctx, _d, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_double, ctypes.c_int]
    L.vmi_set_reference_points.argtypes = [_ctx, _d, ctypes.c_int64]
    L.vmi_set_reference_records_f32.argtypes = [_ctx, _f, ctypes.c_int64]
    L.vmi_set_reference_features.argtypes = [_ctx, _i64, _d, ctypes.c_int64, _i64]
    L.vmi_get_reference_features.argtypes = [_ctx, _i64, _d, ctypes.c_int64, _i64, _i64]
    L.vmi_set_query_points.argtypes = [_ctx, _d, ctypes.c_int64]
    L.vmi_set_query_records_f32.argtypes = [_ctx, _f, ctypes.c_int64]
    L.vmi_set_query_hull.argtypes = [_ctx, _d, ctypes.c_int64]
    L.vmi_poses_to_mats.argtypes = [_d, ctypes.c_int64, _d, ctypes.c_int]
    L.vmi_eval.argtypes = [_ctx, _d, ctypes.c_int64, _d, _i32, _i64, _i64]
    L.vmi_eval_poses.argtypes = [_ctx, _d, ctypes.c_int64, _d, _i32, _i64, _i64]
    L.vmi_eval_device.argtypes = [_ctx, _vp, ctypes.c_int64, _vp, _vp, _vp, _vp, _vp]
    L.vmi_eval_fixups.argtypes = [_ctx, _vp, ctypes.c_int64, _vp, _vp, _vp, _vp, _vp, _i64]
    L.vmi_eval_rot_device.argtypes = [_ctx, _vp, ctypes.c_int64, _vp, _vp, _vp, ctypes.c_int64, _vp,
                                      _vp, _vp, _vp]
    L.vmi_eval_exact.argtypes = [_ctx, _d, ctypes.c_int64, _d, _i32, _i64, _i64]
    L.vmi_query_features.argtypes = [_ctx, _d, _i64, _d, ctypes.c_int64, _i64, _i64, _i32]
    L.vmi_fast_features.argtypes = [_ctx, _d, _i64, _d, ctypes.c_int64, _i64, _i32]
    L.vmi_argmax_device.argtypes = [_ctx, _vp, ctypes.c_int64, _d, _i64, _vp]
    L.vmi_topk_device.argtypes = [_ctx, _vp, ctypes.c_int64, ctypes.c_int64, _d, _i64, _vp]
    L.vmi_launch_count.argtypes = [_ctx]
    L.vmi_launch_count.restype = ctypes.c_int64
    L.vmi_set_tuning.argtypes = [_ctx, ctypes.c_int, ctypes.c_int]
    L.vmi_get_counters.argtypes = [_ctx, _i64]
    L.vmi_set_passes.argtypes = [_ctx, ctypes.c_int]
    L.vmi_nm_run.argtypes = [ctypes.c_int64, _d, _d, ctypes.c_int, ctypes.c_double,
                             ctypes.c_double, ctypes.c_int, ctypes.c_int64, NM_EVAL_FN, _vp, _d,
                             _d, _i32, _i32, _i32, _i32, _d, _i32, ctypes.c_int64]
    L.vmi_set_pairs.argtypes = [_ctx, ctypes.c_int64, ctypes.POINTER(_vp), _i64,
                                ctypes.POINTER(_vp), _i64, ctypes.c_int]
    L.vmi_eval_pairs.argtypes = [_ctx, _d, _i32, ctypes.c_int64, _d, _i32,
                                 ctypes.POINTER(ctypes.c_uint64), _i64]
    L.vmi_align_pairs.argtypes = [_ctx, ctypes.c_int64, _d, _d, ctypes.c_int, ctypes.c_double,
                                  ctypes.c_double, ctypes.c_int, _d, _d, _i32, _i32, _i32, _i32,
                                  _d, _i32, ctypes.c_int64]
    _lib = L
    return L


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def rotation_plan(poses: np.ndarray, mats: np.ndarray):
    """Rotation-major plan of a pose grid for vmi_eval_rot_device: (rots (R, 12)
    one matrix per distinct (rx, ry, rz), mats in rotation-major slot order,
    rot_idx (P,) i32 per slot, perm (P,) i64 = each slot's pose index)."""
    poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 6)
    keys = np.ascontiguousarray(poses[:, 3:6]).view(np.uint64)
    _, first, inv = np.unique(keys, axis=0, return_index=True, return_inverse=True)
    inv = inv.reshape(-1)
    perm = np.argsort(inv, kind="stable").astype(np.int64)
    rots = np.ascontiguousarray(mats[first])
    return rots, np.ascontiguousarray(mats[perm]), inv[perm].astype(np.int32), perm


def poses_to_mats(poses: np.ndarray, threads: int = 0) -> np.ndarray:
    """euler_to_transform for (P, 6) poses -> (P, 12) [R row-major, t].

    Host C++ with glibc sin/cos, no FP contraction: bit-identical to the
    reference's geometry.py:126-138 (see csrc/pose_host.cpp).
    """
    poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 6)
    out = np.empty((poses.shape[0], 12), dtype=np.float64)
    rc = load().vmi_poses_to_mats(ptr(poses, _d), poses.shape[0], ptr(out, _d), int(threads))
    if rc == -2:
        raise ValueError("poses contain non-finite components")
    if rc:
        raise VmiError(f"vmi_poses_to_mats failed ({rc})")
    return out


class Context:
    """One native context (one CUDA device)."""

    def __init__(self, device: int = 0):
        L = load()
        h = _ctx()
        rc = L.vmi_create(int(device), ctypes.byref(h))
        if rc:
            raise VmiError(f"vmi_create(device={device}) failed ({rc}): no usable sm_100 CUDA device")
        self._h = h
        self._L = L
        self.device = device

    def check(self, rc: int, what: str):
        if rc:
            msg = self._L.vmi_last_error(self._h).decode()
            if rc == -1 and ("empty cloud" in msg or "non-finite components" in msg):
                raise ValueError(msg)
            if rc == -1:
                raise ValueError(f"{what}: {msg}")
            raise VmiError(f"{what} failed ({rc}): {msg}")

    def close(self):
        if getattr(self, "_h", None):
            self._L.vmi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def launches(self) -> int:
        return int(self._L.vmi_launch_count(self._h))

    def counters(self) -> dict:
        """launches, table re-plans, exact-path poses, scan-B occupancy estimate"""
        out = np.zeros(6, dtype=np.int64)
        self.check(self._L.vmi_get_counters(self._h, ptr(out, _i64)), "vmi_get_counters")
        return dict(zip(("launches", "replans", "exact_poses", "b_voxels_estimate", "nm_steps",
                         "nm_probes"), (int(x) for x in out)))

    def set_params(self, origin, res, kind: int, bins: int, clamp: float, include_phi: bool):
        o = np.ascontiguousarray(origin, dtype=np.float64)
        self.check(self._L.vmi_set_params(self._h, ptr(o, _d), float(res), int(kind), int(bins),
                                          float(clamp), int(bool(include_phi))), "vmi_set_params")

    def set_tuning(self, table_cap: int = 0, threads: int = 0):
        self.check(self._L.vmi_set_tuning(self._h, int(table_cap), int(threads)), "vmi_set_tuning")

    def set_passes(self, npass: int = 0):
        self.check(self._L.vmi_set_passes(self._h, int(npass)), "vmi_set_passes")

    def set_reference_points(self, xyz: np.ndarray):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        rc = self._L.vmi_set_reference_points(self._h, ptr(xyz, _d), xyz.shape[0])
        if rc == -5:
            from .errors import OutOfBoundsError
            raise OutOfBoundsError(self._L.vmi_last_error(self._h).decode())
        self.check(rc, "vmi_set_reference_points")

    def set_reference_records(self, rec: np.ndarray):
        rec = np.ascontiguousarray(rec, dtype=np.float32)
        if rec.ndim != 2 or rec.shape[1] != 4:
            raise ValueError("records must be (N, 4) float32")
        rc = self._L.vmi_set_reference_records_f32(self._h, ptr(rec, _f), rec.shape[0])
        if rc == -5:
            from .errors import OutOfBoundsError
            raise OutOfBoundsError(self._L.vmi_last_error(self._h).decode())
        self.check(rc, "vmi_set_reference_records_f32")

    def set_reference_features(self, keys, values, bounds):
        k = np.ascontiguousarray(keys, dtype=np.int64)
        v = np.ascontiguousarray(values, dtype=np.float64)
        b = np.ascontiguousarray(np.asarray(bounds, dtype=np.int64).reshape(6))
        self.check(self._L.vmi_set_reference_features(self._h, ptr(k, _i64), ptr(v, _d), k.size,
                                                      ptr(b, _i64)), "vmi_set_reference_features")

    def get_reference_features(self):
        n = ctypes.c_int64(0)
        b = np.empty(6, dtype=np.int64)
        self.check(self._L.vmi_get_reference_features(self._h, None, None, 0, ctypes.byref(n),
                                                      ptr(b, _i64)), "vmi_get_reference_features")
        keys = np.empty(max(n.value, 1), dtype=np.int64)
        vals = np.empty(max(n.value, 1), dtype=np.float64)
        self.check(self._L.vmi_get_reference_features(self._h, ptr(keys, _i64), ptr(vals, _d),
                                                      keys.size, ctypes.byref(n), ptr(b, _i64)),
                   "vmi_get_reference_features")
        return keys[:n.value], vals[:n.value], b.reshape(2, 3)

    def set_query_points(self, xyz: np.ndarray):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        self.check(self._L.vmi_set_query_points(self._h, ptr(xyz, _d), xyz.shape[0]),
                   "vmi_set_query_points")

    def set_query_hull(self, xyz: np.ndarray):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
        self.check(self._L.vmi_set_query_hull(self._h, ptr(xyz, _d), xyz.shape[0]),
                   "vmi_set_query_hull")

    def set_query_records(self, rec: np.ndarray):
        rec = np.ascontiguousarray(rec, dtype=np.float32)
        if rec.ndim != 2 or rec.shape[1] != 4:
            raise ValueError("records must be (N, 4) float32")
        self.check(self._L.vmi_set_query_records_f32(self._h, ptr(rec, _f), rec.shape[0]),
                   "vmi_set_query_records_f32")

    def set_pairs(self, pairs):
        """vmi_set_pairs: [(scan A, scan B), ...] as (N, 4) float32 records (all
        pairs) or (N, 3) float64 arrays (all pairs)."""
        arrs = []
        rec = None
        for a, b in pairs:
            for x in (a, b):
                is_rec = x.dtype == np.float32 and x.ndim == 2 and x.shape[1] == 4
                if rec is None:
                    rec = is_rec
                if is_rec != rec:
                    raise ValueError("all scans of a pair set must share one format")
                arrs.append(np.ascontiguousarray(x, dtype=np.float32 if rec else np.float64))
        K = len(pairs)
        a_ptr = (_vp * max(K, 1))(*[arrs[2 * i].ctypes.data for i in range(K)])
        b_ptr = (_vp * max(K, 1))(*[arrs[2 * i + 1].ctypes.data for i in range(K)])
        na = np.array([arrs[2 * i].shape[0] for i in range(K)], dtype=np.int64)
        nb = np.array([arrs[2 * i + 1].shape[0] for i in range(K)], dtype=np.int64)
        rc = self._L.vmi_set_pairs(self._h, K, a_ptr, ptr(na, _i64), b_ptr, ptr(nb, _i64),
                                   int(bool(rec)))
        if rc == -5:
            from .errors import OutOfBoundsError
            raise OutOfBoundsError(self._L.vmi_last_error(self._h).decode())
        self.check(rc, "vmi_set_pairs")

    def eval_pairs(self, poses: np.ndarray, pair: np.ndarray, want_hist: bool = False,
                   bins: int = 32):
        poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 6)
        pair = np.ascontiguousarray(pair, dtype=np.int32).reshape(-1)
        P = poses.shape[0]
        if pair.shape[0] != P:
            raise ValueError("one pair index per pose")
        mi = np.empty(P, dtype=np.float64)
        st = np.empty(P, dtype=np.int32)
        h = np.empty(P, dtype=np.uint64)
        hist = np.empty((P, bins + 1, bins + 1), dtype=np.int64) if want_hist else None
        self.check(self._L.vmi_eval_pairs(self._h, ptr(poses, _d), ptr(pair, _i32), P, ptr(mi, _d),
                                          ptr(st, _i32), h.ctypes.data_as(
                                              ctypes.POINTER(ctypes.c_uint64)),
                                          ptr(hist, _i64) if want_hist else None),
                   "vmi_eval_pairs")
        return mi, st, h, hist

    def align_pairs(self, x0: np.ndarray, steps, max_iterations: int, f_tol: float, x_tol: float,
                    restarts: int) -> dict:
        x0 = np.ascontiguousarray(x0, dtype=np.float64).reshape(-1, 6)
        K = x0.shape[0]
        st = np.ascontiguousarray(steps, dtype=np.float64).reshape(6)
        cap = max_iterations + restarts + 2
        o = nm_outputs(K, cap)
        self.check(self._L.vmi_align_pairs(self._h, K, ptr(x0, _d), ptr(st, _d), int(max_iterations),
                                           float(f_tol), float(x_tol), int(restarts),
                                           *nm_out_args(o), cap), "vmi_align_pairs")
        return o

    def eval(self, mats: np.ndarray, want_hist: bool = False, bins: int = 32, exact: bool = False):
        mats = np.ascontiguousarray(mats, dtype=np.float64).reshape(-1, 12)
        P = mats.shape[0]
        mi = np.empty(P, dtype=np.float64)
        st = np.empty(P, dtype=np.int32)
        total = np.empty(P, dtype=np.int64)
        hist = np.empty((P, bins + 1, bins + 1), dtype=np.int64) if want_hist else None
        fn = self._L.vmi_eval_exact if exact else self._L.vmi_eval
        self.check(fn(self._h, ptr(mats, _d), P, ptr(mi, _d), ptr(st, _i32),
                      ptr(hist, _i64) if want_hist else None, ptr(total, _i64)), "vmi_eval")
        return mi, st, hist, total

    def eval_poses(self, poses: np.ndarray, want_hist: bool = False, bins: int = 32):
        """vmi_eval_poses: (P, 6) EulerPose rows in, host pose->matrix overlapped
        with the GPU (same results as poses_to_mats + eval)."""
        poses = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 6)
        P = poses.shape[0]
        mi = np.empty(P, dtype=np.float64)
        st = np.empty(P, dtype=np.int32)
        # region totals only travel with histograms (evaluate() returns them then)
        total = np.empty(P, dtype=np.int64) if want_hist else None
        hist = np.empty((P, bins + 1, bins + 1), dtype=np.int64) if want_hist else None
        self.check(self._L.vmi_eval_poses(self._h, ptr(poses, _d), P, ptr(mi, _d), ptr(st, _i32),
                                          ptr(hist, _i64) if want_hist else None,
                                          ptr(total, _i64) if want_hist else None),
                   "vmi_eval_poses")
        return mi, st, hist, total

    def eval_device(self, mats_ptr: int, P: int, mi_ptr: int, st_ptr: int, stream: int = 0,
                    hist_ptr: int = 0, total_ptr: int = 0):
        self.check(self._L.vmi_eval_device(self._h, mats_ptr, P, mi_ptr, st_ptr, hist_ptr or None,
                                           total_ptr or None, stream or None), "vmi_eval_device")

    def eval_rot_device(self, rots_ptr: int, R: int, mats_ptr: int, ridx_ptr: int, perm_ptr: int,
                        P: int, mi_ptr: int, st_ptr: int, stream: int = 0, total_ptr: int = 0):
        """vmi_eval_rot_device: a rotation-major plan (rotation_plan) on device
        pointers; MI / statuses land in the caller's pose order (fix-ups done)."""
        self.check(self._L.vmi_eval_rot_device(self._h, rots_ptr, R, mats_ptr, ridx_ptr, perm_ptr, P,
                                               mi_ptr, st_ptr, total_ptr or None, stream or None),
                   "vmi_eval_rot_device")

    def eval_fixups(self, mats_ptr: int, P: int, mi_ptr: int, st_ptr: int, stream: int = 0,
                    hist_ptr: int = 0, total_ptr: int = 0) -> int:
        n = ctypes.c_int64(0)
        self.check(self._L.vmi_eval_fixups(self._h, mats_ptr, P, mi_ptr, st_ptr, hist_ptr or None,
                                           total_ptr or None, stream or None, ctypes.byref(n)),
                   "vmi_eval_fixups")
        return int(n.value)

    def argmax_device(self, mi_ptr: int, P: int, stream: int = 0):
        v = ctypes.c_double(0)
        i = ctypes.c_int64(0)
        self.check(self._L.vmi_argmax_device(self._h, mi_ptr, P, ctypes.byref(v), ctypes.byref(i),
                                             stream or None), "vmi_argmax_device")
        return float(v.value), int(i.value)

    def topk_device(self, mi_ptr: int, P: int, k: int, stream: int = 0):
        """The min(k, P) largest MI values on the device (descending, ties in
        ascending index order) -> (mi[k], idx[k]) on the host."""
        n = max(0, min(int(k), int(P)))
        vals = np.empty(max(n, 1), dtype=np.float64)
        idx = np.empty(max(n, 1), dtype=np.int64)
        self.check(self._L.vmi_topk_device(self._h, mi_ptr, P, k, ptr(vals, _d), ptr(idx, _i64),
                                           stream or None), "vmi_topk_device")
        return vals[:n], idx[:n]

    def fast_features(self, mat12: np.ndarray, cap: int):
        """B's features at one pose from the fast path (inside A's AABB), sorted by key."""
        m = np.ascontiguousarray(mat12, dtype=np.float64).reshape(12)
        keys = np.empty(max(cap, 1), dtype=np.int64)
        vals = np.empty(max(cap, 1), dtype=np.float64)
        n = ctypes.c_int64(0)
        st = ctypes.c_int32(0)
        self.check(self._L.vmi_fast_features(self._h, ptr(m, _d), ptr(keys, _i64), ptr(vals, _d),
                                             keys.size, ctypes.byref(n), ctypes.byref(st)),
                   "vmi_fast_features")
        if n.value > cap:
            raise VmiError(f"fast_features: {n.value} voxels > capacity {cap}")
        order = np.argsort(keys[:n.value], kind="stable")
        return keys[:n.value][order], vals[:n.value][order], int(st.value)

    def query_features(self, mat12: np.ndarray, cap: int):
        m = np.ascontiguousarray(mat12, dtype=np.float64).reshape(12)
        keys = np.empty(max(cap, 1), dtype=np.int64)
        vals = np.empty(max(cap, 1), dtype=np.float64)
        n = ctypes.c_int64(0)
        b = np.empty(6, dtype=np.int64)
        st = ctypes.c_int32(0)
        self.check(self._L.vmi_query_features(self._h, ptr(m, _d), ptr(keys, _i64), ptr(vals, _d),
                                              keys.size, ctypes.byref(n), ptr(b, _i64),
                                              ctypes.byref(st)), "vmi_query_features")
        return keys[:n.value], vals[:n.value], b.reshape(2, 3), int(st.value)
