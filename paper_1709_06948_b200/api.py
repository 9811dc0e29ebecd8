"""Drop-in replacements for the reference's hot-path entry points.

Same names, argument meaning, return values and error behaviour as the
reference `voxmi` functions they replace; the work runs on the GPU through
MIEngine.  Engines are cached per (scan A map, scan B cloud, grid, binning,
phi) so an optimizer that calls ``mi_objective`` in a loop uploads each scan
once, like the reference's `_prepare` computes scan A once (align.py:114-119).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .engine import MIEngine, mutual_information_exact
from .errors import EmptyOverlapError, NoOverlapError
from .geometry import EulerPose, as_pose_array
from .synth import grid_poses
from .types import (NO_OVERLAP_SENTINEL, AlignmentConfig, BinningSpec, FeatureKind, FeatureMap,
                    GridSpec, JointHistogram, MIResult, as_kind)

SWEEP_AXES = ("tx", "ty", "tz", "rx", "ry", "rz")  # align.py:44

_cache: dict = {}
_CACHE_MAX = 4


def _spec_key(grid, spec, include_phi):
    return (tuple(np.asarray(grid.origin, dtype=np.float64).tolist()), float(grid.resolution),
            as_kind(spec.kind).value, int(spec.bin_count), float(spec.upper_clamp),
            bool(include_phi))


def engine_for(feat_a, cloud_b, grid, spec, include_phi=True, device: int = 0) -> MIEngine:
    """Cached engine with ``feat_a`` and ``cloud_b`` resident."""
    key = (id(feat_a), id(cloud_b), _spec_key(grid, spec, include_phi), device)
    hit = _cache.get(key)
    if hit is not None and hit[1] is feat_a and hit[2] is cloud_b:
        return hit[0]
    eng = MIEngine(grid=grid, binning=spec, include_phi=include_phi, device=device)
    eng.set_reference_features(feat_a)
    eng.set_query(cloud_b)
    if len(_cache) >= _CACHE_MAX:
        _cache.pop(next(iter(_cache)))[0].close()
    _cache[key] = (eng, feat_a, cloud_b)  # strong refs keep the ids unique
    return eng


def clear_cache() -> None:
    while _cache:
        _cache.popitem()[1][0].close()


def compute_feature_map(cloud, grid: GridSpec | None = None, kind=FeatureKind.VARZ,
                        device: int = 0) -> FeatureMap:
    """voxelize + compute_feature_map (voxel.py:210-222, :267-295) on the GPU.

    Bit-exact with the reference, VARZ included (stable sort + numpy's
    pairwise reduceat order).  Raises OutOfBoundsError for points outside
    the key range and ValueError for an empty cloud, like the reference.
    """
    grid = grid if grid is not None else GridSpec()
    eng = MIEngine(grid=grid, binning=BinningSpec(kind=as_kind(kind)), device=device)
    try:
        return eng.set_reference(cloud)
    finally:
        eng.close()


def mi_objective(feat_a, cloud_b, pose, grid, spec, include_phi: bool = True,
                 n_jobs: int = 1) -> float:
    """One objective evaluation (mi.py:194-219): MI, or NO_OVERLAP_SENTINEL.

    ``n_jobs`` is the reference's thread-count knob; it is accepted and
    ignored (the GPU replaces the thread pool).
    """
    del n_jobs
    if as_kind(feat_a.kind) is not as_kind(spec.kind):
        raise ValueError("feature map and binning spec must share one kind")
    eng = engine_for(feat_a, cloud_b, grid, spec, include_phi)
    mi, _ = eng.evaluate(as_pose_array(pose))
    return float(mi[0])


def mi_objective_batch(feat_a, cloud_b, poses, grid, spec, include_phi: bool = True,
                       return_status: bool = False):
    """mi_objective for P poses at once: (P,) float64 (status codes optional)."""
    if as_kind(feat_a.kind) is not as_kind(spec.kind):
        raise ValueError("feature map and binning spec must share one kind")
    eng = engine_for(feat_a, cloud_b, grid, spec, include_phi)
    mi, st = eng.evaluate(as_pose_array(poses))
    return (mi, st) if return_status else mi


def _prepare(scan_a, scan_b, cfg: AlignmentConfig, device: int = 0) -> MIEngine:
    if len(getattr(scan_a, "points", scan_a)) == 0 or len(getattr(scan_b, "points", scan_b)) == 0:
        raise ValueError("both scans must be non-empty")
    eng = MIEngine(grid=cfg.grid, binning=cfg.binning, include_phi=cfg.phi_enabled, device=device)
    eng.set_reference(scan_a)
    eng.set_query(scan_b)
    return eng


def mi_at(scan_a, scan_b, pose, cfg: AlignmentConfig | None = None) -> MIResult:
    """Single evaluation with the entropy breakdown (align.py:162-174).

    Raises EmptyOverlapError when the occupied bounds do not intersect.
    """
    cfg = cfg or AlignmentConfig()
    eng = _prepare(scan_a, scan_b, cfg)
    try:
        mi, st, hist, total = eng.evaluate(as_pose_array(pose), histograms=True)
    finally:
        eng.close()
    if st[0] == 2:
        from .errors import OutOfBoundsError
        raise OutOfBoundsError("a point of scan B maps outside the voxel key range")
    if st[0] == 1:
        raise EmptyOverlapError("scans do not overlap at this pose")
    r = mutual_information_exact(hist[0], cfg.phi_enabled)
    return MIResult(mi=r[0], h_x=r[1], h_y=r[2], h_xy=r[3])


def joint_histogram_at(scan_a, scan_b, pose, cfg: AlignmentConfig | None = None) -> JointHistogram:
    """The JointHistogram mi_at scores (mi.py:124-160), from the GPU."""
    cfg = cfg or AlignmentConfig()
    eng = _prepare(scan_a, scan_b, cfg)
    try:
        _, st, hist, total = eng.evaluate(as_pose_array(pose), histograms=True)
    finally:
        eng.close()
    if st[0] == 1:
        raise EmptyOverlapError("scans do not overlap at this pose")
    return JointHistogram(counts=hist[0], total=int(total[0]), spec=cfg.binning)


def sweep_axis(scan_a, scan_b, base_pose: EulerPose, axis: str, values,
               cfg: AlignmentConfig | None = None) -> list[tuple[float, float]]:
    """MI along one pose axis (align.py:177-198), all values in one batch."""
    if axis not in SWEEP_AXES:
        raise ValueError(f"axis must be one of {SWEEP_AXES}, got {axis!r}")
    cfg = cfg or AlignmentConfig()
    values = [float(v) for v in values]
    base = np.asarray(base_pose.as_vector(), dtype=np.float64)
    poses = np.repeat(base[None, :], len(values), axis=0)
    poses[:, SWEEP_AXES.index(axis)] = values
    if not values:
        return []
    eng = _prepare(scan_a, scan_b, cfg)
    try:
        mi, _ = eng.evaluate(poses)
    finally:
        eng.close()
    return [(v, float(m)) for v, m in zip(values, mi)]


@dataclass
class SearchResult:
    """Outcome of a batched candidate-pose search."""

    best_pose: EulerPose
    best_mi: float
    best_index: int
    mi: np.ndarray
    status: np.ndarray
    n_poses: int


def grid_search(scan_a, scan_b, poses=None, cfg: AlignmentConfig | None = None, center=None,
                axes: dict | None = None, device: int = 0) -> SearchResult:
    """Score every candidate pose and return the np.argmax-selected one.

    Candidates are either ``poses`` ((P, 6) array / EulerPose list) or the
    C-order Cartesian product ``axes`` around ``center`` (see synth.grid_poses).
    Raises NoOverlapError when every candidate is the sentinel, like
    align.py:144-147.
    """
    cfg = cfg or AlignmentConfig()
    if poses is None:
        if axes is None:
            raise ValueError("give poses or axes")
        c = center.as_vector() if hasattr(center, "as_vector") else (
            np.zeros(6) if center is None else np.asarray(center, dtype=np.float64))
        poses = grid_poses(c, axes)
    poses = as_pose_array(poses)
    eng = _prepare(scan_a, scan_b, cfg, device=device)
    try:
        mi, st = eng.evaluate(poses)
        idx, best = eng.best(poses, mi)
    finally:
        eng.close()
    if best <= NO_OVERLAP_SENTINEL:
        raise NoOverlapError("no candidate pose produced overlapping occupied bounds")
    return SearchResult(best_pose=EulerPose.from_vector(poses[idx]), best_mi=best, best_index=idx,
                        mi=mi, status=st, n_poses=poses.shape[0])


def grid_search_sharded(scan_a, scan_b, poses=None, cfg: AlignmentConfig | None = None,
                        center=None, axes: dict | None = None, device: int | None = None,
                        group=None) -> SearchResult:
    """``grid_search`` across the ranks of a torch.distributed group
    (SURVEY.md 8(e)): every rank holds the same candidate list and both scans,
    scores its contiguous shard on its own GPU, re-scores its shard winner
    exactly from the bit-exact histogram, and one all-gather of (mi, global
    index) per rank picks np.argmax's first maximum.  ``mi``/``status`` of the
    result are this rank's shard; ``best_*`` are global and identical on every
    rank (and to ``grid_search`` on one GPU).
    """
    import torch
    import torch.distributed as dist

    from .shard import all_gather_winner, shard_bounds
    cfg = cfg or AlignmentConfig()
    if poses is None:
        if axes is None:
            raise ValueError("give poses or axes")
        c = center.as_vector() if hasattr(center, "as_vector") else (
            np.zeros(6) if center is None else np.asarray(center, dtype=np.float64))
        poses = grid_poses(c, axes)
    poses = as_pose_array(poses)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if device is None:
        device = torch.cuda.current_device()
    lo, hi = shard_bounds(poses.shape[0], world, rank)
    mi = np.empty(0)
    st = np.empty(0, dtype=np.int32)
    value, index = float("-inf"), np.iinfo(np.int64).max
    if hi > lo:
        eng = _prepare(scan_a, scan_b, cfg, device=device)
        try:
            mi, st = eng.evaluate(poses[lo:hi])
            k, value = eng.best(poses[lo:hi], mi, exact_value=True)
            index = lo + k
        finally:
            eng.close()
    xdev = torch.device("cuda", device) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    best, idx = all_gather_winner(value, index, dist, xdev, group=group)
    if best <= NO_OVERLAP_SENTINEL:
        raise NoOverlapError("no candidate pose produced overlapping occupied bounds")
    return SearchResult(best_pose=EulerPose.from_vector(poses[idx]), best_mi=best, best_index=idx,
                        mi=mi, status=st, n_poses=poses.shape[0])

