"""KITTI .bin ingest (scan_io.py:57-85 mirror), CPU side."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1709_06948_b200.errors import FormatError
from paper_1709_06948_b200.scan_io import load_kitti_bin, read_kitti_records, save_kitti_bin


def test_round_trip_keeps_records(tmp_path):
    rng = np.random.default_rng(0)
    rec = rng.normal(size=(1000, 4)).astype(np.float32)
    p = tmp_path / "s.bin"
    save_kitti_bin(rec, p)
    cloud = load_kitti_bin(p)
    np.testing.assert_array_equal(cloud.records, rec)
    np.testing.assert_array_equal(cloud.points, rec[:, :3].astype(np.float64))
    np.testing.assert_array_equal(cloud.intensity, rec[:, 3].astype(np.float64))
    save_kitti_bin(cloud, tmp_path / "t.bin")  # PointCloud path, like the reference
    assert (tmp_path / "t.bin").read_bytes() == p.read_bytes()


def test_bad_size_and_non_finite(tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(b"\0" * 20)
    with pytest.raises(FormatError) as e:
        load_kitti_bin(p)
    assert e.value.byte_offset == 16 and "multiple of 16" in e.value.reason
    rec = np.zeros((4, 4), np.float32)
    rec[2, 1] = np.nan
    p.write_bytes(rec.tobytes())
    with pytest.raises(FormatError) as e:
        read_kitti_records(p)
    assert e.value.byte_offset == 32


def test_empty_file_warns(tmp_path):
    p = tmp_path / "e.bin"
    p.write_bytes(b"")
    with pytest.warns(UserWarning):
        c = load_kitti_bin(p)
    assert len(c) == 0


def test_pinned_request_falls_back_without_cuda(tmp_path):
    rec = np.arange(64, dtype=np.float32).reshape(16, 4)
    p = tmp_path / "p.bin"
    save_kitti_bin(rec, p)
    np.testing.assert_array_equal(read_kitti_records(p, pinned=True), rec)
