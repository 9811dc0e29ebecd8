"""KITTI ``.bin`` scans straight into the kernel's input format.

Mirrors the reference's ``load_kitti_bin`` / ``save_kitti_bin``
(``scan_io.py:57-85``): packed little-endian float32 ``(x, y, z, intensity)``
records, no header; a size that is not a multiple of 16 bytes or a non-finite
value raises ``FormatError`` with the offending byte offset; an empty file
warns and gives an empty cloud.  The returned ``PointCloud`` carries, besides
the reference's float64 ``points``/``intensity``, the raw ``records`` array --
read straight from the file into page-locked (pinned) host memory when
``pinned=True`` -- which ``MIEngine`` uploads as the kernel's native 16-byte
float4 records (no float64 upcast, one host validation pass in the library).
"""

from __future__ import annotations

import os
import warnings
from pathlib import Path

import numpy as np

from .errors import FormatError
from .geometry import PointCloud


def _pinned_empty(n_bytes: int) -> np.ndarray:
    """Page-locked host buffer owned by torch (buffer ownership only)."""
    import torch
    t = torch.empty(max(n_bytes, 1), dtype=torch.uint8, pin_memory=True)
    return t.numpy()[:n_bytes]  # the view's base chain keeps the tensor alive


def pinned_copy(arr: np.ndarray) -> np.ndarray:
    """A page-locked copy of ``arr`` (what read_kitti_records(pinned=True) gives
    for a scan read from disk); plain memory without a CUDA runtime."""
    arr = np.ascontiguousarray(arr)
    try:
        buf = _pinned_empty(arr.nbytes)
    except Exception:  # noqa: BLE001
        return arr.copy()
    out = buf.view(arr.dtype).reshape(arr.shape)
    out[...] = arr
    return out


def read_kitti_records(path, pinned: bool = False) -> np.ndarray:
    """(N, 4) float32 records of a KITTI ``.bin`` file, validated like the
    reference (size multiple of 16, finite values)."""
    path = Path(path)
    size = os.path.getsize(path)
    if size % 16 != 0:
        raise FormatError(path, f"file size {size} is not a multiple of 16 bytes "
                          "(x, y, z, intensity float32 records)", byte_offset=size - size % 16)
    if pinned and size > 0:
        try:
            buf = _pinned_empty(size)
        except Exception:  # no CUDA runtime: plain memory
            buf = np.empty(size, dtype=np.uint8)
    else:
        buf = np.empty(size, dtype=np.uint8)
    with open(path, "rb", buffering=0) as fh:
        got = fh.readinto(memoryview(buf))
    if got != size:
        raise FormatError(path, f"short read ({got} of {size} bytes)")
    rec = buf.view("<f4").reshape(-1, 4)
    if rec.size and not np.isfinite(rec).all():
        bad = int(np.flatnonzero(~np.isfinite(rec).all(axis=1))[0])
        raise FormatError(path, f"non-finite value in record {bad}", byte_offset=bad * 16)
    return rec


def load_kitti_bin(path, pinned: bool = False) -> PointCloud:
    """Read a packed float32 (x, y, z, intensity) scan (scan_io.py:57-75)."""
    rec = read_kitti_records(path, pinned=pinned)
    if rec.shape[0] == 0:
        warnings.warn(f"{path}: empty scan file", stacklevel=2)
        return PointCloud(np.zeros((0, 3)), intensity=np.zeros(0))
    return PointCloud(rec[:, :3].astype(np.float64), intensity=rec[:, 3].astype(np.float64),
                      records=rec)


def save_kitti_bin(cloud, path) -> None:
    """Write a cloud as float32 records (scan_io.py:78-85); (N, 4) float32
    record arrays are written as they are."""
    if isinstance(cloud, np.ndarray) and cloud.dtype == np.float32 and cloud.ndim == 2 \
            and cloud.shape[1] == 4:
        Path(path).write_bytes(np.ascontiguousarray(cloud, dtype="<f4").tobytes())
        return
    intensity = cloud.intensity
    if intensity is None:
        intensity = np.zeros(len(cloud))
    data = np.empty((len(cloud), 4), dtype="<f4")
    data[:, :3] = cloud.points
    data[:, 3] = intensity
    Path(path).write_bytes(data.tobytes())
