"""Point clouds and 6-DOF poses, mirroring the reference's hot-path types.

Mirrors `voxmi.geometry` (`geometry.py:36-166`): ``PointCloud`` (validated
(N, 3) float64, optional intensity), ``EulerPose`` (tx, ty, tz, rx, ry, rz;
R = Rz @ Ry @ Rx), and ``euler_to_transform``.  Batched pose -> matrix
conversion for the GPU path happens in the native library
(``vmi_poses_to_mats``), built with glibc ``sin``/``cos`` and
``-ffp-contract=off`` so every matrix entry is bit-identical to the
reference's ``math.sin``/``math.cos`` products (`geometry.py:126-138`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class PointCloud:
    """(N, 3) float64 points in meters with optional (N,) intensity.

    Same validation as the reference (`geometry.py:36-65`): finite
    coordinates, matching intensity length.
    """

    points: np.ndarray
    intensity: np.ndarray | None = None
    # the (N, 4) float32 KITTI records the cloud was read from, when it was
    # (scan_io.load_kitti_bin): the engine uploads those as they are
    records: np.ndarray | None = field(default=None, compare=False, repr=False)

    def __post_init__(self):
        pts = np.ascontiguousarray(self.points, dtype=np.float64)
        if pts.ndim != 2 or pts.shape[1] != 3:
            raise ValueError(f"points must be (N, 3), got shape {pts.shape}")
        if not np.isfinite(pts).all():
            raise ValueError("points contain non-finite coordinates")
        object.__setattr__(self, "points", pts)
        if self.intensity is not None:
            inten = np.asarray(self.intensity, dtype=np.float64)
            if inten.shape != (pts.shape[0],):
                raise ValueError(
                    f"intensity length {inten.shape} does not match "
                    f"{pts.shape[0]} points")
            object.__setattr__(self, "intensity", inten)

    def __len__(self) -> int:
        return self.points.shape[0]

    @classmethod
    def from_records(cls, rec: np.ndarray) -> "PointCloud":
        """From KITTI-style (N, 4) float32 (x, y, z, i) records."""
        rec = np.asarray(rec)
        return cls(rec[:, :3].astype(np.float64),
                   rec[:, 3].astype(np.float64) if rec.shape[1] > 3 else None)


@dataclass(frozen=True)
class EulerPose:
    """6-DOF pose: translation in meters, ZYX Euler angles in radians
    (`geometry.py:68-102`)."""

    tx: float = 0.0
    ty: float = 0.0
    tz: float = 0.0
    rx: float = 0.0
    ry: float = 0.0
    rz: float = 0.0

    def __post_init__(self):
        vals = (self.tx, self.ty, self.tz, self.rx, self.ry, self.rz)
        if not all(math.isfinite(v) for v in vals):
            raise ValueError(f"pose has non-finite component: {vals}")

    def as_vector(self) -> np.ndarray:
        return np.array([self.tx, self.ty, self.tz, self.rx, self.ry, self.rz])

    @classmethod
    def from_vector(cls, v) -> "EulerPose":
        v = np.asarray(v, dtype=np.float64)
        if v.shape != (6,):
            raise ValueError(f"pose vector must have 6 entries, got {v.shape}")
        return cls(*(float(x) for x in v))


def euler_to_transform(pose: EulerPose) -> np.ndarray:
    """4x4 transform of one pose, R = Rz(rz) @ Ry(ry) @ Rx(rx).

    Evaluated by the native library so single poses and batches share one
    bit pattern (see module docstring).
    """
    from ._lib import poses_to_mats
    m = poses_to_mats(pose.as_vector()[None, :])[0]
    t = np.eye(4)
    t[:3, :3] = m[:9].reshape(3, 3)
    t[:3, 3] = m[9:]
    return t


def as_pose_array(poses, check_finite: bool = True) -> np.ndarray:
    """Accept EulerPose objects, (6,) or (P, 6) arrays; return (P, 6) f64.
    ``check_finite=False``: the caller's native conversion validates instead
    (vmi_poses_to_mats fails on a non-finite component)."""
    if isinstance(poses, EulerPose) or (hasattr(poses, "as_vector")
                                        and hasattr(poses, "rz")):
        return np.asarray(poses.as_vector(), dtype=np.float64)[None, :]
    if isinstance(poses, (list, tuple)) and poses and hasattr(poses[0], "as_vector"):
        return np.stack([np.asarray(p.as_vector(), dtype=np.float64) for p in poses])
    arr = np.ascontiguousarray(poses, dtype=np.float64)
    if arr.ndim == 1:
        arr = arr[None, :]
    if arr.ndim != 2 or arr.shape[1] != 6:
        raise ValueError(f"poses must be (P, 6), got {arr.shape}")
    # any NaN / inf makes the sum non-finite; a finite sum proves every entry
    # finite (one pass instead of a full boolean mask on large batches)
    if check_finite and not np.isfinite(arr.sum()) and not np.isfinite(arr).all():
        raise ValueError("poses contain non-finite components")
    return arr


ORTHONORMAL_TOL = 1e-9
GIMBAL_GUARD = math.pi / 2 - 1e-6


def wrap_angle(a: float) -> float:
    """Wrap into (-pi, pi]; exact no-op when already in range (geometry.py:26-33)."""
    if -math.pi < a <= math.pi:
        return a
    w = math.remainder(a, math.tau)
    if w <= -math.pi:
        w += math.tau
    return w


def normalized(p: EulerPose) -> EulerPose:
    """EulerPose with angles wrapped into (-pi, pi] (geometry.py:94-99)."""
    return EulerPose(p.tx, p.ty, p.tz, wrap_angle(p.rx), wrap_angle(p.ry), wrap_angle(p.rz))


def validate_transform(t) -> np.ndarray:
    """Rigid-transform invariants (geometry.py:109-123): 4x4, finite, last row
    [0,0,0,1], orthonormal rotation with det +1 (1e-9)."""
    t = np.asarray(t, dtype=np.float64)
    if t.shape != (4, 4):
        raise ValueError(f"transform must be 4x4, got {t.shape}")
    if not np.isfinite(t).all():
        raise ValueError("transform contains non-finite entries")
    if not np.array_equal(t[3], [0.0, 0.0, 0.0, 1.0]):
        raise ValueError(f"last row must be [0, 0, 0, 1], got {t[3]}")
    r = t[:3, :3]
    if np.abs(r.T @ r - np.eye(3)).max() > ORTHONORMAL_TOL:
        raise ValueError("rotation block is not orthonormal within 1e-9")
    if abs(np.linalg.det(r) - 1.0) > ORTHONORMAL_TOL:
        raise ValueError("rotation block determinant is not +1")
    return t


def transform_to_euler(t) -> EulerPose:
    """ZYX Euler angles of a transform (geometry.py:141-159); raises near gimbal lock."""
    from .errors import VoxmiError
    t = validate_transform(t)
    r = t[:3, :3]
    sp = max(-1.0, min(1.0, -float(r[2, 0])))
    ry = math.asin(sp)
    if abs(ry) >= GIMBAL_GUARD:
        raise VoxmiError(f"pitch {ry:.6f} rad is within 1e-6 of +/-pi/2")
    rx = math.atan2(r[2, 1], r[2, 2])
    rz = math.atan2(r[1, 0], r[0, 0])
    return EulerPose(float(t[0, 3]), float(t[1, 3]), float(t[2, 3]), rx, ry, rz)
