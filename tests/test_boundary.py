"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/vmi.h declares, rejects misuse without a device, and its
host-side pose->matrix step is bit-identical to the reference."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from conftest import ROOT, golden, hdl_pair

from paper_1709_06948_b200 import _lib


def header_symbols() -> list[str]:
    with open(os.path.join(ROOT, "include", "vmi.h")) as fh:
        src = fh.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\*?\s+\*?(vmi_[a-z0-9_]+)\(", src,
                                 re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_1709_06948_b200 import build
        build.build()
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 18
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.EXPORTS)


def test_version_string(lib):
    assert b"sm_100a" in lib.vmi_version()


def test_create_without_device_fails_cleanly(lib):
    h = ctypes.c_void_p()
    rc = lib.vmi_create(0, ctypes.byref(h))
    assert rc in (0, -2, -6)  # OK on a B200 box, VMI_ERR_CUDA / UNSUPPORTED elsewhere
    if rc == 0:
        lib.vmi_destroy(h)
    else:
        assert not h.value


def test_null_context_is_rejected(lib):
    assert lib.vmi_set_params(None, None, 1.0, 0, 32, 2.0, 1) == -1
    assert lib.vmi_eval(None, None, 0, None, None, None, None) == -1
    assert lib.vmi_last_error(None) == b"null context"


def test_pose_matrices_bit_exact(lib):
    rng = np.random.default_rng(3)
    poses = rng.uniform(-4, 4, size=(20000, 6))
    got = _lib.poses_to_mats(poses)
    want = oracle.poses_to_mats(poses)
    np.testing.assert_array_equal(got.view(np.int64), want.view(np.int64))
    # single-thread and threaded paths agree
    np.testing.assert_array_equal(_lib.poses_to_mats(poses, threads=1).view(np.int64),
                                  got.view(np.int64))


def test_pose_matrices_reproduce_reference_transform(lib):
    g = golden("hdl_golden.npz")
    _, b = hdl_pair()
    mats = _lib.poses_to_mats(g["poses"][:8])
    pts = b[g["xform_sample"], :3].astype(np.float64)
    for k in range(8):
        moved = oracle.transform(pts, mats[k])
        np.testing.assert_array_equal(moved.view(np.int64), g["xform_moved"][k].view(np.int64))


def test_missing_library_fails_loudly(tmp_path):
    saved = _lib._lib
    _lib._lib = None
    try:
        with pytest.raises(_lib.VmiError, match="no CPU fallback"):
            _lib.load(str(tmp_path / "libvmi.so"))
    finally:
        _lib._lib = saved
