"""Pin the CPU oracle (oracle/voxmi_oracle.c) to the reference's own outputs.

Every expected value here was produced by the real `voxmi` package
(tests/golden/make_golden.py).  The oracle must match bit for bit wherever
the reference is integer/byte work or a fixed-order numpy reduction
(transform, voxel keys, bounds, COUNT and VARZ features, histograms), and to
1e-12 for MI (glibc log vs numpy's SIMD log differ by <= 1 ulp).
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import SMALL_CASES, golden, hdl_pair, small_case


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def test_pose_matrices_bit_exact_vs_reference():
    g = golden("hdl_golden.npz")
    poses = g["poses"][:8]
    a, b = hdl_pair()
    pts = b[:, :3].astype(np.float64)
    mats = oracle.poses_to_mats(poses)
    for k in range(8):
        moved = oracle.transform(pts[g["xform_sample"]], mats[k])
        np.testing.assert_array_equal(bits(moved), bits(g["xform_moved"][k]))


def test_hdl_scans_match_golden_digest():
    import hashlib
    a, b = hdl_pair()
    g = golden("hdl_golden.npz")
    assert hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() == str(g["a_digest"])
    assert hashlib.sha256(np.ascontiguousarray(b).tobytes()).hexdigest() == str(g["b_digest"])


@pytest.mark.parametrize("tag", SMALL_CASES)
def test_small_feature_maps_bit_exact(tag):
    c = small_case(tag)
    fa = oracle.feature_map(c["a"], c["origin"], c["res"], c["kind"])
    np.testing.assert_array_equal(fa.keys, c["a_keys"])
    np.testing.assert_array_equal(bits(fa.values), bits(c["a_values"]))
    np.testing.assert_array_equal(fa.bounds, c["a_bounds"])


@pytest.mark.parametrize("tag", SMALL_CASES)
def test_small_objective_matches_reference(tag):
    c = small_case(tag)
    fa = oracle.feature_map(c["a"], c["origin"], c["res"], c["kind"])
    mats = oracle.poses_to_mats(c["poses"])
    for k in range(mats.shape[0]):
        mi, st, counts, total = oracle.mi_objective_full(fa, c["b"], mats[k], c["origin"], c["res"],
                                                         include_phi=c["phi"])
        assert st == c["status"][k]
        if st in (0, 3):
            np.testing.assert_array_equal(counts, c["hist"][k])
            assert total == c["total"][k]
        if st == 0:
            assert mi == pytest.approx(c["mi"][k], rel=1e-12, abs=1e-14)
        else:
            assert mi == -1e300 == c["mi"][k]


@pytest.mark.parametrize("tag,res,kind", [("v1", 1.0, "varz"), ("v02", 0.2, "varz"),
                                          ("c1", 1.0, "count")])
def test_hdl_feature_maps_and_histograms(tag, res, kind):
    g = golden("hdl_golden.npz")
    a, b = hdl_pair()
    fa = oracle.feature_map(a[:, :3].astype(np.float64), (0, 0, 0), res, kind)
    np.testing.assert_array_equal(fa.keys, g[f"{tag}_a_keys"])
    np.testing.assert_array_equal(bits(fa.values), bits(g[f"{tag}_a_values"]))
    np.testing.assert_array_equal(fa.bounds, g[f"{tag}_a_bounds"])
    mats = oracle.poses_to_mats(g["poses"])
    pts_b = b[:, :3].astype(np.float64)
    fb = oracle.feature_map(oracle.transform(pts_b, mats[0]), (0, 0, 0), res, kind)
    np.testing.assert_array_equal(fb.keys, g[f"{tag}_b_keys"])
    np.testing.assert_array_equal(bits(fb.values), bits(g[f"{tag}_b_values"]))
    n = g[f"{tag}_mi"].shape[0]
    for k in range(0, n, 3 if n > 16 else 1):
        mi, st, counts, total = oracle.mi_objective_full(fa, pts_b, mats[k], (0, 0, 0), res)
        assert st == g[f"{tag}_status"][k]
        np.testing.assert_array_equal(counts, g[f"{tag}_hist"][k].astype(np.int64))
        assert total == g[f"{tag}_total"][k]
        assert mi == pytest.approx(g[f"{tag}_mi"][k], rel=1e-12, abs=1e-14)


def test_c1_grid_mi_and_argmax():
    g = golden("c1_golden.npz")
    s = golden("c1_scans.npz")
    fa = oracle.feature_map(s["a"], (0, 0, 0), 0.5, "count")
    np.testing.assert_array_equal(fa.keys, g["a_keys"])
    np.testing.assert_array_equal(fa.values, g["a_values"])
    poses = g["poses"]
    sel = np.arange(0, poses.shape[0], 41)
    mi, st = oracle.mi_objective_batch(fa, s["b"], oracle.poses_to_mats(poses[sel]), res=0.5,
                                       threads=0)
    np.testing.assert_allclose(mi, g["mi"][sel], rtol=1e-12, atol=1e-14)
    for j, i in enumerate(g["sub"][:20]):
        _, st1, counts, total = oracle.mi_objective_full(fa, s["b"], oracle.poses_to_mats(poses[i])[0],
                                                         res=0.5)
        np.testing.assert_array_equal(counts, g["hist"][j].astype(np.int64))
        assert total == g["total"][j]
    assert int(g["argmax"]) == int(np.argmax(g["mi"]))


def test_mutual_information_matches_reference():
    g = golden("mi_golden.npz")
    for h, r, r2 in zip(g["hists"], g["res"], g["res_nophi"]):
        got = oracle.mutual_information(h.astype(np.int64))
        np.testing.assert_allclose(got, r, rtol=1e-13, atol=1e-15)
        got2 = oracle.mutual_information(h.astype(np.int64), include_phi=False)
        np.testing.assert_allclose(got2, r2, rtol=1e-13, atol=1e-15)


def test_bins_match_reference():
    g = golden("bins_golden.npz")
    np.testing.assert_array_equal(oracle.bin_features(g["values"], 32, 2.0), g["varz"])
    np.testing.assert_array_equal(oracle.bin_features(g["values"], 32, 64.0), g["count"])
    # known answers from the reference's own tests (test_mi.py:56-98)
    np.testing.assert_array_equal(oracle.bin_features([0.0, 0.0624, 0.0625, 1.0, 2.0, 999.0]),
                                  [1, 1, 2, 17, 32, 32])
    np.testing.assert_array_equal(oracle.bin_features([63.9, 2.0], 32, 64.0), [32, 2])


def test_entropy_known_answer():
    # test_mi.py:107-110
    assert oracle.lib().orc_entropy(np.array([1.0, 2.0, 3.0]).ctypes.data_as(oracle._d), 3) == \
        pytest.approx(1.0114042647073518, abs=1e-12)


def test_small_scene_digests():
    import hashlib
    for tag in SMALL_CASES:
        c = small_case(tag)
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(c["a"]).tobytes())
        h.update(np.ascontiguousarray(c["b"]).tobytes())
        assert h.hexdigest() == c["digest"]


def test_oracle_nm_port_matches_reference_optimizer():
    """oracle/nm.py (the C5 CPU baseline's optimizer) is the reference's run
    on the reference's own golden (nm_golden.npz)."""
    from oracle.nm import nelder_mead_maximize
    g = golden("nm_golden.npz")

    def f(x):
        c = np.array([1.0, -2.0, 0.5, 0.1, -0.05, 0.3])
        w = np.array([1.0, 0.5, 2.0, 10.0, 10.0, 4.0])
        return float(np.exp(-np.sum(w * (x - c) ** 2)) + 0.1 * np.cos(x[0] - x[1]))
    for tag in ("default", "restarts", "maxiter"):
        cfg = g[f"{tag}_cfg"]
        bx, bv, it, term, trace, ne = nelder_mead_maximize(
            f, g[f"{tag}_x0"], g[f"{tag}_steps"], int(cfg[0]), float(cfg[1]), float(cfg[2]),
            int(cfg[3]))
        np.testing.assert_array_equal(bx, g[f"{tag}_best_x"])
        assert bv == float(g[f"{tag}_best_value"]) and it == int(g[f"{tag}_iterations"])
        assert term == str(g[f"{tag}_termination"]) and ne == int(g[f"{tag}_n_eval"])
        np.testing.assert_array_equal(trace, g[f"{tag}_trace"])
