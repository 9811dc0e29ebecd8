"""HDL-64-shaped synthetic lidar scans (the reference ships no such generator).

The reference's only scene generator (`voxmi.bench.synth_scene_pair`,
bench.py:188-200) samples box surfaces uniformly; it has no beam structure,
no occlusion and no range-dependent density.  The north-star workload is
"120k-point HDL-64-shaped scans", so this module ray-casts a 64-beam spinning
sensor against a ground plane plus axis-aligned boxes:

* 64 beams, elevations ``linspace(+2.0°, -24.8°, 64)``; ``azimuths`` steps per
  revolution; sensor 1.73 m above the ground; max range 120 m; range noise
  N(0, 0.02 m).
* Scene: ground plane z = 0 and ``n_boxes`` boxes in a ``extent`` square,
  heights U(1, 8) m, half-widths U(0.75, 6) m, none centred on the road
  (|y| < 10 m) or within 8 m of the first sensor position.
* Points are emitted ring-major (beam by beam, azimuth inner), the order of a
  KITTI ``.bin`` file, expressed in the sensor frame (ground near z = -1.73)
  and rounded to float32 like KITTI input (`scan_io.py:69-75` upcasts float32
  to float64), then truncated to exactly ``n_points``.

Everything is seeded and deterministic; nothing here is on the timed path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .geometry import EulerPose

SENSOR_HEIGHT = 1.73
ELEV_TOP_DEG = 2.0
ELEV_BOTTOM_DEG = -24.8
N_BEAMS = 64


@dataclass(frozen=True)
class LidarSceneSpec:
    """A ground plane plus boxes, scanned by a 64-beam spinning lidar."""

    seed: int = 0
    extent: float = 200.0
    n_boxes: int = 200
    n_points: int = 120_000
    azimuths: int = 2000
    max_range: float = 120.0
    range_noise: float = 0.02
    box_height: tuple[float, float] = (1.0, 8.0)
    box_half_width: tuple[float, float] = (0.75, 6.0)


def _boxes(spec: LidarSceneSpec, rng: np.random.Generator) -> np.ndarray:
    """(n_boxes, 6) array of [xmin, ymin, zmin, xmax, ymax, zmax] in world."""
    out = []
    half = spec.extent / 2
    while len(out) < spec.n_boxes:
        cx, cy = rng.uniform(-half, half, size=2)
        hx, hy = rng.uniform(*spec.box_half_width, size=2)
        h = rng.uniform(*spec.box_height)
        if abs(cy) < 10.0 or math.hypot(cx, cy) < 8.0:
            continue
        out.append([cx - hx, cy - hy, 0.0, cx + hx, cy + hy, h])
    return np.asarray(out, dtype=np.float64)


def _ray_dirs(spec: LidarSceneSpec) -> np.ndarray:
    """Unit ray directions in the sensor frame, ring-major (R, 3)."""
    el = np.radians(np.linspace(ELEV_TOP_DEG, ELEV_BOTTOM_DEG, N_BEAMS))
    az = np.arange(spec.azimuths) * (2 * np.pi / spec.azimuths)
    ce, se = np.cos(el)[:, None], np.sin(el)[:, None]
    d = np.stack([np.broadcast_to(ce * np.cos(az), (N_BEAMS, spec.azimuths)),
                  np.broadcast_to(ce * np.sin(az), (N_BEAMS, spec.azimuths)),
                  np.broadcast_to(se, (N_BEAMS, spec.azimuths))], axis=-1)
    return d.reshape(-1, 3)


def _slab(origin, d, inv, b):
    """Slab-method entry distance of rays ``d`` into boxes ``b`` (inf = miss)."""
    t0 = (b[None, :, :3] - origin) * inv[:, None, :]
    t1 = (b[None, :, 3:] - origin) * inv[:, None, :]
    tn = np.nanmax(np.minimum(t0, t1), axis=2)
    tf = np.nanmin(np.maximum(t0, t1), axis=2)
    hit = (tn <= tf) & (tf > 0) & (tn > 0)
    return np.where(hit, tn, np.inf).min(axis=1)


def _cast(origin: np.ndarray, dirs: np.ndarray, boxes: np.ndarray,
          max_range: float, azimuths: int | None = None, yaw: float = 0.0) -> np.ndarray:
    """Nearest hit distance per ray (inf = no return) against plane + boxes.

    With ``azimuths`` given (ring-major rays, azimuth step 2*pi/azimuths in the
    sensor frame, sensor yaw ``yaw``), each box is only tested against the rays
    inside its conservative azimuth window; the per (ray, box) arithmetic is
    unchanged, so the result is identical to testing every box.
    """
    t = np.full(dirs.shape[0], np.inf)
    dz = dirs[:, 2]
    down = dz < 0
    t[down] = -origin[2] / dz[down]
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / dirs
        if azimuths is None:
            for chunk in range(0, boxes.shape[0], 32):
                t = np.minimum(t, _slab(origin, dirs, inv, boxes[chunk:chunk + 32]))
        else:
            n_beams = dirs.shape[0] // azimuths
            step = 2 * np.pi / azimuths
            for b in boxes:
                cx = np.array([b[0], b[3], b[3], b[0]]) - origin[0]
                cy = np.array([b[1], b[1], b[4], b[4]]) - origin[1]
                if b[0] <= origin[0] <= b[3] and b[1] <= origin[1] <= b[4]:
                    cols = np.arange(azimuths)
                else:
                    ang = np.arctan2(cy, cx)
                    mid = np.arctan2(cy.mean(), cx.mean())
                    rel = np.angle(np.exp(1j * (ang - mid)))
                    lo = mid + rel.min() - yaw
                    hi = mid + rel.max() - yaw
                    k0 = int(np.floor(lo / step)) - 2
                    k1 = int(np.ceil(hi / step)) + 2
                    cols = np.arange(k0, k1 + 1) % azimuths
                idx = (np.arange(n_beams)[:, None] * azimuths + cols[None, :]).ravel()
                th = _slab(origin, dirs[idx], inv[idx], b[None, :])
                t[idx] = np.minimum(t[idx], th)
    t[t > max_range] = np.inf
    return t


def scan_from(spec: LidarSceneSpec, boxes: np.ndarray, sensor: EulerPose,
              rng: np.random.Generator) -> np.ndarray:
    """One scan from a sensor at planar pose ``sensor`` (tx, ty, rz used).

    Returns (n_points, 4) float32 records (x, y, z, intensity) in the sensor
    frame, ring-major.
    """
    dirs_s = _ray_dirs(spec)
    c, s = math.cos(sensor.rz), math.sin(sensor.rz)
    rot = np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])
    dirs_w = dirs_s @ rot.T
    origin = np.array([sensor.tx, sensor.ty, SENSOR_HEIGHT + sensor.tz])
    t = _cast(origin, dirs_w, boxes, spec.max_range, azimuths=spec.azimuths, yaw=sensor.rz)
    keep = np.isfinite(t)
    t = t + rng.normal(0.0, spec.range_noise, size=t.shape)
    pts = dirs_s[keep] * t[keep, None]
    if pts.shape[0] < spec.n_points:
        raise ValueError(
            f"only {pts.shape[0]} returns for {spec.n_points} requested points; "
            "raise azimuths")
    pts = pts[:spec.n_points]
    out = np.empty((spec.n_points, 4), dtype=np.float32)
    out[:, :3] = pts.astype(np.float32)
    out[:, 3] = (np.linalg.norm(pts, axis=1) / spec.max_range).astype(np.float32)
    return out


def hdl64_pair(spec: LidarSceneSpec = LidarSceneSpec(),
               truth: EulerPose = EulerPose(1.5, 0.3, 0.0, 0.0, 0.0, 0.05)
               ) -> tuple[np.ndarray, np.ndarray]:
    """Scan A from the world origin and scan B from ``truth`` (planar).

    ``truth`` maps scan-B coordinates into scan A's frame, i.e. it is the pose
    the MI objective should peak at.  Returns two (n_points, 4) float32 arrays.
    """
    ss = np.random.SeedSequence(spec.seed).spawn(3)
    boxes = _boxes(spec, np.random.default_rng(ss[0]))
    a = scan_from(spec, boxes, EulerPose(), np.random.default_rng(ss[1]))
    b = scan_from(spec, boxes, truth, np.random.default_rng(ss[2]))
    return a, b


def candidate_batch(truth: EulerPose, n: int, seed: int = 0,
                    half_width=(3.0, 3.0, 0.3, math.radians(1.5),
                                math.radians(1.5), math.radians(10.0))
                    ) -> np.ndarray:
    """(n, 6) float64 poses uniform in ``truth ± half_width`` (C2 batch)."""
    rng = np.random.default_rng(seed)
    hw = np.asarray(half_width, dtype=np.float64)
    return truth_vector(truth) + rng.uniform(-1.0, 1.0, size=(n, 6)) * hw


def truth_vector(p: EulerPose) -> np.ndarray:
    return np.array([p.tx, p.ty, p.tz, p.rx, p.ry, p.rz], dtype=np.float64)


def grid_poses(center, axes: dict[str, np.ndarray]) -> np.ndarray:
    """C-order Cartesian product of per-axis offsets around ``center``.

    ``axes`` maps a subset of (tx, ty, tz, rx, ry, rz) to absolute values;
    missing axes stay at ``center``.  Order follows (tx, ty, tz, rx, ry, rz),
    last axis fastest, like nested loops.
    """
    names = ("tx", "ty", "tz", "rx", "ry", "rz")
    center = np.asarray(center, dtype=np.float64)
    cols = [np.asarray(axes[k], dtype=np.float64) if k in axes
            else np.array([center[i]]) for i, k in enumerate(names)]
    mesh = np.meshgrid(*cols, indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=1)


def _frame_job(job):
    spec, near, pose, seed, i = job
    return scan_from(spec, near, pose, np.random.default_rng([seed, 1000 + i]))


def drive_sequence(n_frames: int, spec: LidarSceneSpec = LidarSceneSpec(), seed: int = 0,
                   step: float = 1.0, workers: int = 1,
                   subset: tuple[int, int] | None = None) -> tuple[list, list[EulerPose]]:
    """C5: a synthetic drive, ``n_frames`` HDL-64-shaped scans ~``step`` m apart.

    The sensor follows the road (x axis) with a slow lateral / yaw drift
    through a corridor of boxes; returns the scans (float32 records, each in
    its own sensor frame) and the world sensor poses (planar).  The relative
    pose mapping frame i+1 into frame i is ``relative_pose(poses[i], poses[i+1])``.
    ``workers`` > 1 builds the frames in that many spawned processes (same scans);
    ``subset=(lo, hi)`` builds only frames lo..hi-1 (the others are None).
    """
    rng = np.random.default_rng(np.random.SeedSequence(seed).spawn(1)[0])
    length = n_frames * step
    corridor = LidarSceneSpec(seed=seed, extent=spec.extent, n_boxes=spec.n_boxes,
                              n_points=spec.n_points, azimuths=spec.azimuths,
                              max_range=spec.max_range, range_noise=spec.range_noise,
                              box_height=spec.box_height, box_half_width=spec.box_half_width)
    # boxes along the whole corridor: tile the square scene every `extent` metres
    boxes = []
    for k, x0 in enumerate(np.arange(-spec.extent / 2, length + spec.extent / 2, spec.extent)):
        b = _boxes(corridor, np.random.default_rng([seed, k]))
        b[:, [0, 3]] += x0 + spec.extent / 2
        boxes.append(b)
    boxes = np.concatenate(boxes)
    poses, scans = [], []
    for i in range(n_frames):
        x = i * step
        y = 0.6 * math.sin(x / 37.0)
        yaw = 0.03 * math.sin(x / 23.0)
        poses.append(EulerPose(x, y, 0.0, 0.0, 0.0, yaw))

    def frame(i):  # every frame has its own generator: independent of the order
        x = poses[i].tx
        near = boxes[(np.abs((boxes[:, 0] + boxes[:, 3]) / 2 - x) < spec.max_range + 10.0)]
        return scan_from(spec, near, poses[i], np.random.default_rng([seed, 1000 + i]))

    idx = range(*subset) if subset is not None else range(n_frames)
    if workers > 1 and len(idx) > 1:  # spawned processes (scan_from holds the GIL)
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor
        jobs = []
        for i in idx:
            x = poses[i].tx
            near = boxes[(np.abs((boxes[:, 0] + boxes[:, 3]) / 2 - x) < spec.max_range + 10.0)]
            jobs.append((spec, near, poses[i], seed, i))
        with ProcessPoolExecutor(workers, mp_context=mp.get_context("spawn")) as pool:
            built = list(pool.map(_frame_job, jobs, chunksize=max(1, len(idx) // (4 * workers))))
    else:
        built = [frame(i) for i in idx]
    scans = [None] * n_frames
    for i, sc in zip(idx, built):
        scans[i] = sc
    return scans, poses


def relative_pose(p_i: EulerPose, p_j: EulerPose) -> EulerPose:
    """Planar pose of sensor j expressed in sensor i's frame (maps scan j into scan i)."""
    c, s = math.cos(p_i.rz), math.sin(p_i.rz)
    dx, dy = p_j.tx - p_i.tx, p_j.ty - p_i.ty
    return EulerPose(c * dx + s * dy, -s * dx + c * dy, 0.0, 0.0, 0.0, p_j.rz - p_i.rz)


C5_SIMPLEX_STEPS = (1.0, 1.0, 0.1, 0.01, 0.01, 0.05)  # C5 --c5-mode nm initial simplex


def c5_priors(world_poses, seed: int = 5) -> tuple[list, list[EulerPose]]:
    """C5 per-pair priors: the true relative pose of (i, i+1) perturbed by
    0.5 m in a random planar direction and +-1 deg of yaw (bench.py:203-224
    `perturb_pose` style).  Returns (priors as (6,) arrays, truths)."""
    rng = np.random.default_rng(seed)
    priors, truths = [], []
    for i in range(len(world_poses) - 1):
        t = relative_pose(world_poses[i], world_poses[i + 1])
        h = rng.uniform(0, 2 * np.pi)
        truths.append(t)
        priors.append(np.array([t.tx + 0.5 * np.cos(h), t.ty + 0.5 * np.sin(h), 0.0, 0.0, 0.0,
                                t.rz + np.radians(1.0) * (1 if rng.random() < 0.5 else -1)]))
    return priors, truths


def c5_grid(prior) -> np.ndarray:
    """C5 grid mode: 16 x 16 x 16 (tx, ty, yaw) candidates around a prior."""
    c = np.asarray(prior, dtype=np.float64)
    offs = np.linspace(-0.75, 0.75, 16)
    yaw_offs = np.radians(np.linspace(-1.5, 1.5, 16))
    return grid_poses(c, {"tx": c[0] + offs, "ty": c[1] + offs, "rz": c[5] + yaw_offs})
