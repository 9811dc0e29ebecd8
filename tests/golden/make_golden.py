"""Generate the golden parity fixtures from the REAL reference package.

Run here (the reference is importable only in the build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every number in the fixtures comes from `voxmi` itself (the reference's own
public functions); nothing in tests/ or bench.py reads /root/reference at run
time.  Outputs (all .npz, committed):

  c1_scans.npz   C1 scan pair: synth_scene_pair(SceneSpec(seed=0, n_points=20_000))
                 with scan B moved by inverse(truth) (bench.py:188-200)
  c1_golden.npz  C1 = 0.5 m COUNT over the 6069-pose grid: MI of every pose,
                 np.argmax, histograms/totals of a strided subset, A feature map
  hdl_golden.npz HDL-64-shaped pair (our generator, digest pinned): A feature maps
                 and 48 poses' MI / status / histogram at 1 m VARZ and 0.2 m VARZ,
                 1 m COUNT, plus transform bit patterns of sampled points
  small_golden.npz small seeded scenes (test_mi.py:303-345 style): VARZ/COUNT at
                 several grids incl. non-zero origin and phi excluded, sentinels
  mi_golden.npz  300 random 33x33 histograms -> mutual_information (crit. 1)
  bins_golden.npz bin_features on random values + the test_mi.py known answers
  c4_golden.npz  bench.py's C4 scene (100 m, HDL-64-shaped, 0.2 m VARZ): 16 poses'
                 MI / status / histogram / total
  c2ref_golden.npz bench.py's C2 batch (65,536 poses, seed 2024): the reference's MI
                 and status for every 16th pose (4,096 poses)
  c5_golden.npz  the first 20 pairs of bench.py's C5 drive: per pair the reference's
                 pick over the 4,096-pose grid (np.argmax, MI) and voxmi.align from the
                 prior (pose, final MI, iterations, termination)
"""

from __future__ import annotations

import hashlib
import math
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import voxmi  # noqa: E402  (reference, PYTHONPATH=/root/reference/pkg/src)
from voxmi import (BinningSpec, EulerPose, FeatureKind, GridSpec, PointCloud, SceneSpec,  # noqa: E402
                   apply_transform, build_joint_histogram, compute_feature_map, compute_overlap,
                   euler_to_transform, inverse, mi_objective, mutual_information,
                   synth_scene_pair, voxelize)

from paper_1709_06948_b200.synth import LidarSceneSpec, grid_poses, hdl64_pair  # noqa: E402

C1_TRUTH = (1.0, 0.5, 0.0, 0.0, 0.0, 0.1)
HDL_TRUTH = (1.5, 0.3, 0.0, 0.0, 0.0, 0.05)


def c1_grid() -> np.ndarray:
    """tx, ty = truth ± 2 m step 0.25; yaw = truth ± 5° step 0.5°."""
    t = np.asarray(C1_TRUTH)
    return grid_poses(t, {
        "tx": t[0] + np.arange(-8, 9) * 0.25,
        "ty": t[1] + np.arange(-8, 9) * 0.25,
        "rz": t[5] + np.radians(np.arange(-10, 11) * 0.5),
    })


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def full_eval(feat_a, scan_b, pose_vec, grid, spec, include_phi=True):
    """mi_objective plus, when valid, the histogram it scored."""
    pose = EulerPose.from_vector(pose_vec)
    mi = mi_objective(feat_a, scan_b, pose, grid, spec, include_phi=include_phi)
    w = spec.bin_count + 1
    counts = np.zeros((w, w), dtype=np.int64)
    total = 0
    status = 0
    moved = apply_transform(scan_b, euler_to_transform(pose))
    try:
        vox = voxelize(moved, grid)
    except voxmi.OutOfBoundsError:
        return mi, 2, counts, 0
    fb = compute_feature_map(vox, moved, spec.kind)
    region = compute_overlap(feat_a.bounds, fb.bounds)
    if region.is_empty:
        return mi, 1, counts, 0
    hist = build_joint_histogram(feat_a, fb, region, spec)
    counts, total = hist.counts, hist.total
    if mi == voxmi.NO_OVERLAP_SENTINEL:
        status = 3
    return mi, status, counts, total


_W = {}


def _c1_worker(chunk):
    fa, scan_b, grid, spec = _W["args"]
    return [mi_objective(fa, scan_b, EulerPose.from_vector(p), grid, spec) for p in chunk]


def _init(args):
    _W["args"] = args


def make_c1():
    a, b_world = synth_scene_pair(SceneSpec(seed=0, n_points=20_000))
    truth = EulerPose(*C1_TRUTH)
    scan_b = apply_transform(b_world, inverse(euler_to_transform(truth)))
    np.savez_compressed(os.path.join(HERE, "c1_scans.npz"), a=a.points, b=scan_b.points)
    grid = GridSpec(resolution=0.5)
    spec = BinningSpec(kind=FeatureKind.COUNT)
    fa = compute_feature_map(voxelize(a, grid), a, FeatureKind.COUNT)
    poses = c1_grid()
    chunks = np.array_split(poses, 64)
    with ProcessPoolExecutor(8, initializer=_init, initargs=((fa, scan_b, grid, spec),)) as ex:
        mi = np.concatenate([np.asarray(r) for r in ex.map(_c1_worker, chunks)])
    sub = np.arange(0, poses.shape[0], 37)
    hs, ts, st = [], [], []
    for i in sub:
        m, s, c, t = full_eval(fa, scan_b, poses[i], grid, spec)
        assert m == mi[i]
        hs.append(c); ts.append(t); st.append(s)
    np.savez_compressed(os.path.join(HERE, "c1_golden.npz"), poses=poses, mi=mi,
                        argmax=np.int64(np.argmax(mi)), sub=sub, hist=np.asarray(hs, np.int32),
                        total=np.asarray(ts), status=np.asarray(st, np.int32),
                        a_keys=fa.keys, a_values=fa.values, a_bounds=fa.bounds)
    print("C1: argmax", int(np.argmax(mi)), poses[int(np.argmax(mi))], mi.max())


def make_hdl():
    spec_scene = LidarSceneSpec()
    a_rec, b_rec = hdl64_pair(spec_scene, EulerPose(*HDL_TRUTH))
    a = PointCloud(a_rec[:, :3].astype(np.float64))
    b = PointCloud(b_rec[:, :3].astype(np.float64))
    rng = np.random.default_rng(7)
    hw = np.array([3.0, 3.0, 0.3, math.radians(1.5), math.radians(1.5), math.radians(10.0)])
    poses = np.asarray(HDL_TRUTH) + rng.uniform(-1, 1, size=(48, 6)) * hw
    poses[0] = HDL_TRUTH
    poses[1] = (0, 0, 0, 0, 0, 0)
    poses[2] = (1e4, 0, 0, 0, 0, 0)    # disjoint -> empty region
    poses[3] = (3e6, 0, 0, 0, 0, 0)    # key range
    out = {"a_digest": digest(a_rec), "b_digest": digest(b_rec), "poses": poses}
    sample = np.arange(0, a.points.shape[0], 997)
    moved = np.stack([apply_transform(b, euler_to_transform(EulerPose.from_vector(p))).points[sample]
                      for p in poses[:8]])
    out["xform_sample"] = sample
    out["xform_moved"] = moved
    for tag, res, kind in (("v1", 1.0, FeatureKind.VARZ), ("v02", 0.2, FeatureKind.VARZ),
                           ("c1", 1.0, FeatureKind.COUNT)):
        grid = GridSpec(resolution=res)
        spec = BinningSpec(kind=kind)
        fa = compute_feature_map(voxelize(a, grid), a, kind)
        out[f"{tag}_a_keys"], out[f"{tag}_a_values"], out[f"{tag}_a_bounds"] = fa.keys, fa.values, fa.bounds
        n = 48 if tag == "v1" else 16
        mis, sts, hs, ts = [], [], [], []
        for p in poses[:n]:
            m, s, c, t = full_eval(fa, b, p, grid, spec)
            mis.append(m); sts.append(s); hs.append(c); ts.append(t)
        out[f"{tag}_mi"] = np.asarray(mis)
        out[f"{tag}_status"] = np.asarray(sts, np.int32)
        out[f"{tag}_hist"] = np.asarray(hs, np.int32)
        out[f"{tag}_total"] = np.asarray(ts)
        # B feature map at the truth pose (VARZ values for the 1e-6 check)
        moved_b = apply_transform(b, euler_to_transform(EulerPose(*HDL_TRUTH)))
        fb = compute_feature_map(voxelize(moved_b, grid), moved_b, kind)
        out[f"{tag}_b_keys"], out[f"{tag}_b_values"], out[f"{tag}_b_bounds"] = fb.keys, fb.values, fb.bounds
        print("HDL", tag, "mi[0]", mis[0], "|VA|", len(fa.keys))
    np.savez_compressed(os.path.join(HERE, "hdl_golden.npz"), **out)


def small_scene(seed, n):
    """test_mi.py:303-307 scene: half flat, half tall."""
    rng = np.random.default_rng(seed)
    pts = rng.uniform(-15, 15, size=(n, 3))
    pts[:, 2] = rng.uniform(0, 4, size=n) * (pts[:, 0] > 0)
    return PointCloud(pts)


def make_small():
    out = {}
    cases = [
        ("s0", 60, 5000, 1.0, (0, 0, 0), FeatureKind.VARZ, True),
        ("s1", 61, 5000, 0.5, (0, 0, 0), FeatureKind.COUNT, True),
        ("s2", 62, 3000, 0.2, (0, 0, 0), FeatureKind.VARZ, True),
        ("s3", 63, 3000, 0.7, (0.3, -0.2, 0.15), FeatureKind.VARZ, True),
        ("s4", 64, 3000, 1.0, (0, 0, 0), FeatureKind.VARZ, False),
        ("s5", 65, 2000, 0.25, (-1.0, 2.0, 0.5), FeatureKind.COUNT, False),
    ]
    rng = np.random.default_rng(99)
    for tag, seed, n, res, origin, kind, phi in cases:
        a = small_scene(seed, n)
        b = small_scene(seed + 100, n)
        grid = GridSpec(origin=np.asarray(origin, dtype=np.float64), resolution=res)
        spec = BinningSpec(kind=kind)
        fa = compute_feature_map(voxelize(a, grid), a, kind)
        poses = np.concatenate([
            np.zeros((1, 6)),
            rng.uniform(-1, 1, size=(20, 6)) * np.array([3, 3, 0.5, 0.05, 0.05, 0.3]),
            np.array([[1e4, 0, 0, 0, 0, 0], [3e6, 0, 0, 0, 0, 0], [0, 0, 40.0, 0, 0, 0]]),
        ])
        mis, sts, hs, ts = [], [], [], []
        for p in poses:
            m, s, c, t = full_eval(fa, b, p, grid, spec, include_phi=phi)
            mis.append(m); sts.append(s); hs.append(c); ts.append(t)
        out[f"{tag}_digest"] = np.array(digest(a.points, b.points))
        out[f"{tag}_seed"] = np.array([seed, n])
        out[f"{tag}_meta"] = np.array([res, *origin, 0 if kind is FeatureKind.VARZ else 1,
                                       1 if phi else 0])
        out[f"{tag}_poses"] = poses
        out[f"{tag}_mi"] = np.asarray(mis)
        out[f"{tag}_status"] = np.asarray(sts, np.int32)
        out[f"{tag}_hist"] = np.asarray(hs, np.int32)
        out[f"{tag}_total"] = np.asarray(ts)
        out[f"{tag}_a_keys"], out[f"{tag}_a_values"], out[f"{tag}_a_bounds"] = fa.keys, fa.values, fa.bounds
    np.savez_compressed(os.path.join(HERE, "small_golden.npz"), **out)
    print("small cases:", [c[0] for c in cases])


def make_mi():
    rng = np.random.default_rng(20)
    hists = rng.integers(0, 40, size=(300, 33, 33))
    hists[:, 0, 0] += rng.integers(0, 100000, size=300)
    hists[::7] *= (rng.random((hists[::7].shape)) < 0.1)  # sparse ones
    hists[:, 1, 1] += 1
    res = []
    res_nophi = []
    for h in hists:
        r = mutual_information(voxmi.JointHistogram(counts=h, total=int(h.sum()),
                                                    spec=BinningSpec(kind=FeatureKind.VARZ)))
        res.append((r.mi, r.h_x, r.h_y, r.h_xy))
        r2 = mutual_information(voxmi.JointHistogram(counts=h, total=int(h.sum()),
                                                     spec=BinningSpec(kind=FeatureKind.VARZ)),
                                include_phi=False)
        res_nophi.append((r2.mi, r2.h_x, r2.h_y, r2.h_xy))
    np.savez_compressed(os.path.join(HERE, "mi_golden.npz"), hists=hists.astype(np.int32),
                        res=np.asarray(res), res_nophi=np.asarray(res_nophi))


def make_bins():
    rng = np.random.default_rng(21)
    v = np.concatenate([rng.uniform(0, 3, 2000), rng.uniform(0, 80, 2000),
                        np.arange(0, 2.2, 0.0625), np.arange(0, 70, 2.0)])
    out = {"values": v}
    for name, kind in (("varz", FeatureKind.VARZ), ("count", FeatureKind.COUNT)):
        out[name] = voxmi.bin_features(v, BinningSpec(kind=kind))
    np.savez_compressed(os.path.join(HERE, "bins_golden.npz"), **out)


def make_align():
    """voxmi.align on the C1 scans: two configurations, every report field."""
    from voxmi import AlignmentConfig, SimplexConfig, align
    s = np.load(os.path.join(HERE, "c1_scans.npz"))
    a, b = PointCloud(s["a"]), PointCloud(s["b"])
    cases = {
        "varz1": (AlignmentConfig(), EulerPose(0.6, 0.2, 0.0, 0.0, 0.0, 0.06)),
        "count05": (AlignmentConfig(feature=FeatureKind.COUNT, grid=GridSpec(resolution=0.5),
                                    simplex=SimplexConfig(initial_steps=(2.0, 2.0, 0.5, 0.05, 0.05, 0.2),
                                                          max_iterations=150, restarts=1)),
                    EulerPose()),
    }
    out = {}
    for tag, (cfg, p0) in cases.items():
        rep = align(a, b, euler_to_transform(p0), cfg)
        out[f"{tag}_t0"] = p0.as_vector()
        out[f"{tag}_pose"] = rep.estimated_pose.as_vector()
        out[f"{tag}_matrix"] = rep.estimated
        out[f"{tag}_final_mi"] = np.float64(rep.final_mi)
        out[f"{tag}_trace"] = np.asarray(rep.mi_trace)
        out[f"{tag}_iterations"] = np.int64(rep.iterations)
        out[f"{tag}_termination"] = np.array(rep.termination)
        print("align", tag, rep.iterations, rep.termination, rep.final_mi, rep.wall_time)
    np.savez_compressed(os.path.join(HERE, "align_golden.npz"), **out)


def nm_test_function(x):
    """Smooth 6-D test objective with a unique maximum (for optimizer parity)."""
    x = np.asarray(x, dtype=np.float64)
    c = np.array([1.0, -2.0, 0.5, 0.1, -0.05, 0.3])
    w = np.array([1.0, 0.5, 2.0, 10.0, 10.0, 4.0])
    return float(np.exp(-np.sum(w * (x - c) ** 2)) + 0.1 * np.cos(x[0] - x[1]))


def make_nm():
    """voxmi.nelder_mead_maximize on a closed-form objective: every OptimResult field."""
    from voxmi import SimplexConfig, nelder_mead_maximize
    out = {}
    cases = {
        "default": (np.zeros(6), SimplexConfig()),
        "restarts": (np.array([3.0, 1.0, 0.0, 0.0, 0.0, 0.0]),
                     SimplexConfig(initial_steps=(1.0, 1.0, 0.5, 0.05, 0.05, 0.2),
                                   max_iterations=400, restarts=2, f_tol=1e-9, x_tol=1e-7)),
        "maxiter": (np.ones(6), SimplexConfig(max_iterations=25)),
    }
    for tag, (x0, cfg) in cases.items():
        r = nelder_mead_maximize(nm_test_function, x0, cfg)
        out[f"{tag}_x0"] = x0
        out[f"{tag}_steps"] = np.asarray(cfg.initial_steps)
        out[f"{tag}_cfg"] = np.array([cfg.max_iterations, cfg.f_tol, cfg.x_tol, cfg.restarts])
        out[f"{tag}_best_x"] = r.best_x
        out[f"{tag}_best_value"] = np.float64(r.best_value)
        out[f"{tag}_iterations"] = np.int64(r.iterations)
        out[f"{tag}_termination"] = np.array(r.termination)
        out[f"{tag}_trace"] = np.asarray(r.trace)
        out[f"{tag}_spread"] = np.asarray(r.trace_spread)
        out[f"{tag}_n_eval"] = np.int64(r.n_evaluations)
        print("nm", tag, r.iterations, r.termination, r.n_evaluations)
    np.savez_compressed(os.path.join(HERE, "nm_golden.npz"), **out)


def _mi_worker(job):
    fa, scan_b, grid, spec, chunk = job
    out = []
    for p in chunk:
        m, s, _, _ = full_eval(fa, scan_b, p, grid, spec)
        out.append((m, s))
    return out


def make_c4():
    """bench.py C4 workload: 100 m scene, 0.2 m VARZ, 16 poses."""
    from paper_1709_06948_b200.synth import candidate_batch
    spec_scene = LidarSceneSpec(extent=100.0, n_boxes=120, box_height=(1.0, 10.0))
    a_rec, b_rec = hdl64_pair(spec_scene, EulerPose(*HDL_TRUTH))
    a = PointCloud(a_rec[:, :3].astype(np.float64))
    b = PointCloud(b_rec[:, :3].astype(np.float64))
    batch = candidate_batch(EulerPose(*HDL_TRUTH), 65536, seed=2024)
    idx = np.arange(0, 65536, 4681)[:14]
    poses = np.concatenate([np.asarray([HDL_TRUTH, (0, 0, 0, 0, 0, 0)]), batch[idx]])
    grid = GridSpec(resolution=0.2)
    spec = BinningSpec(kind=FeatureKind.VARZ)
    fa = compute_feature_map(voxelize(a, grid), a, FeatureKind.VARZ)
    mis, sts, hs, ts = [], [], [], []
    for p in poses:
        m, st, c, t = full_eval(fa, b, p, grid, spec)
        mis.append(m); sts.append(st); hs.append(c); ts.append(t)
    np.savez_compressed(os.path.join(HERE, "c4_golden.npz"), a_digest=digest(a_rec),
                        b_digest=digest(b_rec), poses=poses, batch_idx=idx, mi=np.asarray(mis),
                        status=np.asarray(sts, np.int32), hist=np.asarray(hs, np.int32),
                        total=np.asarray(ts), a_nvox=np.int64(len(fa.keys)))
    print("C4: |VA|", len(fa.keys), "mi", mis[:3])


def make_c2ref():
    """bench.py C2 batch: the reference's MI for every 16th of the 65,536 poses."""
    from paper_1709_06948_b200.synth import candidate_batch
    a_rec, b_rec = hdl64_pair(LidarSceneSpec(), EulerPose(*HDL_TRUTH))
    a = PointCloud(a_rec[:, :3].astype(np.float64))
    b = PointCloud(b_rec[:, :3].astype(np.float64))
    batch = candidate_batch(EulerPose(*HDL_TRUTH), 65536, seed=2024)
    sel = np.arange(0, 65536, 16)
    grid = GridSpec(resolution=1.0)
    spec = BinningSpec(kind=FeatureKind.VARZ)
    fa = compute_feature_map(voxelize(a, grid), a, FeatureKind.VARZ)
    jobs = [(fa, b, grid, spec, c) for c in np.array_split(batch[sel], 64)]
    with ProcessPoolExecutor(8) as ex:
        res = [r for part in ex.map(_mi_worker, jobs) for r in part]
    np.savez_compressed(os.path.join(HERE, "c2ref_golden.npz"), a_digest=digest(a_rec),
                        b_digest=digest(b_rec), sel=sel, mi=np.array([r[0] for r in res]),
                        status=np.array([r[1] for r in res], np.int32))
    print("C2ref:", len(res), "poses; argmax", sel[int(np.argmax([r[0] for r in res]))])


def _c5_pair(job):
    from voxmi import AlignmentConfig, SimplexConfig, align
    a_rec, b_rec, prior, steps = job
    from paper_1709_06948_b200.synth import c5_grid
    a = PointCloud(a_rec[:, :3].astype(np.float64))
    b = PointCloud(b_rec[:, :3].astype(np.float64))
    grid = GridSpec(resolution=1.0)
    spec = BinningSpec(kind=FeatureKind.VARZ)
    fa = compute_feature_map(voxelize(a, grid), a, FeatureKind.VARZ)
    poses = c5_grid(prior)
    mi = np.array([mi_objective(fa, b, EulerPose.from_vector(p), grid, spec) for p in poses])
    rep = align(a, b, euler_to_transform(EulerPose.from_vector(prior)),
                AlignmentConfig(simplex=SimplexConfig(initial_steps=steps)))
    return (int(np.argmax(mi)), float(mi.max()), mi[::64].copy(), rep.estimated_pose.as_vector(),
            float(rep.final_mi), int(rep.iterations), str(rep.termination),
            np.asarray(rep.mi_trace))


def make_c5():
    """First 20 pairs of bench.py's C5 drive: grid picks + voxmi.align results."""
    from paper_1709_06948_b200.synth import C5_SIMPLEX_STEPS, c5_priors, drive_sequence
    n = 20
    scans, wp = drive_sequence(1001, workers=8, subset=(0, n + 1))
    priors, _ = c5_priors(wp)
    jobs = [(scans[i], scans[i + 1], priors[i], C5_SIMPLEX_STEPS) for i in range(n)]
    with ProcessPoolExecutor(8) as ex:
        res = list(ex.map(_c5_pair, jobs))
    out = {"digests": np.array([digest(scans[i]) for i in range(n + 1)]),
           "priors": np.asarray(priors[:n]),
           "grid_argmax": np.array([r[0] for r in res]), "grid_best_mi": np.array([r[1] for r in res]),
           "grid_mi_sub": np.stack([r[2] for r in res]),
           "align_pose": np.stack([r[3] for r in res]), "align_final_mi": np.array([r[4] for r in res]),
           "align_iterations": np.array([r[5] for r in res]),
           "align_termination": np.array([r[6] for r in res])}
    for i, r in enumerate(res):
        out[f"align_trace_{i}"] = r[7]
    np.savez_compressed(os.path.join(HERE, "c5_golden.npz"), **out)
    print("C5: picks", out["grid_argmax"], "align iters", out["align_iterations"])


if __name__ == "__main__":
    what = sys.argv[1:] or ["small", "mi", "bins", "hdl", "c1", "align", "nm", "c4", "c2ref",
                            "c5"]
    for w in what:
        globals()[f"make_{w}"]()
