"""MIEngine: resident scan pair on one B200, batched candidate-pose scoring.

This is the host side of the hot path.  It owns one native context
(libvmi.so) per device and replaces, for a batch of P poses, P calls of the
reference's ``mi_objective`` (mi.py:194-219) made by ``align``'s objective
closure (align.py:134-136) and ``sweep_axis`` (align.py:191-197):

* ``set_reference``  -- _prepare (align.py:114-119): scan A voxelized and
  featurized ON THE GPU (exact sort-based path), or an existing FeatureMap
  uploaded as is; kept resident as a dense u8 bin grid.
* ``set_query``      -- scan B uploaded once, in the kernel's span layout.
* ``evaluate``       -- one fused kernel over all poses (k_fast.cu), then an
  exact re-evaluation of the rare flagged poses (k_exact.cu).
* ``best``           -- np.argmax semantics (first max, cli.py:202), with exact
  host re-scoring of near-ties from their bit-exact GPU histograms.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib
from .errors import OutOfBoundsError
from .geometry import PointCloud, as_pose_array
from .types import (NO_OVERLAP_SENTINEL, BinningSpec, FeatureKind, FeatureMap, GridSpec, as_kind)


def _points_of(cloud) -> np.ndarray:
    """(N, 3|4) array of a cloud: a PointCloud's KITTI records when it carries
    them (scan_io.load_kitti_bin), else its points, else the array itself."""
    rec = getattr(cloud, "records", None)
    if rec is not None:
        return rec
    pts = getattr(cloud, "points", cloud)
    pts = np.asarray(pts)
    if pts.ndim != 2 or pts.shape[1] not in (3, 4):
        raise ValueError(f"points must be (N, 3), got shape {pts.shape}")
    return pts


def entropy_exact(counts) -> float:
    """The reference's entropy (mi.py:163-174) on the host, bit for bit.

    Used only to break near-ties between candidate poses from their GPU
    histograms; the sort makes the result independent of cell order.
    """
    arr = np.asarray(counts, dtype=np.float64).ravel()
    total = arr.sum()
    if not total > 0:
        raise ValueError("entropy of an all-zero distribution is undefined")
    p = arr[arr > 0] / total
    return float(-np.sort(p * np.log(p)).sum())


def mutual_information_exact(counts, include_phi: bool = True) -> tuple[float, float, float, float]:
    """(mi, h_x, h_y, h_xy) of a joint histogram, mi.py:177-191 semantics."""
    c = np.asarray(counts)
    m = c if include_phi else c[1:, 1:]
    h_x = entropy_exact(m.sum(axis=1))
    h_y = entropy_exact(m.sum(axis=0))
    h_xy = entropy_exact(m)
    mi = h_x + h_y - h_xy
    if -1e-12 <= mi < 0.0:
        mi = 0.0
    return mi, h_x, h_y, h_xy


HULL_MIN_POINTS = 50_000


def hull_vertices(pts: np.ndarray):
    """Scan B's convex-hull vertices (qhull, via scipy) as float64 (h, 3) -- the
    points the kernel takes each pose's voxel bounds from (vmi_set_query_hull)
    -- or None (no scipy, a degenerate scan, or VMI_NO_HULL=1).  Small scans
    keep per-point bounds: below ~50k points the per-pose hull pass (plus its
    two barriers) costs about what it saves (A/B: C2 120k points 29.3 -> 28.5
    ms per 65,536 poses; C1 20k points 1.84 -> 1.92 ms)."""
    if os.environ.get("VMI_NO_HULL") == "1" or pts.shape[0] < HULL_MIN_POINTS:
        return None
    try:
        from scipy.spatial import ConvexHull
        xyz = np.ascontiguousarray(pts[:, :3], dtype=np.float64)
        return xyz[ConvexHull(xyz).vertices]
    except Exception:  # noqa: BLE001 -- QhullError (flat / degenerate scans), ImportError
        return None


class MIEngine:
    """Batched MI pose evaluation on one GPU.

    ``grid``/``binning`` take this package's GridSpec/BinningSpec or the
    reference's own objects (duck-typed).
    """

    def __init__(self, grid=None, binning=None, kind=None, include_phi: bool = True,
                 device: int = 0, threads: int = 0, table_cap: int = 0, passes: int = 0):
        grid = grid if grid is not None else GridSpec()
        if binning is None:
            binning = BinningSpec(kind=as_kind(kind) if kind is not None else FeatureKind.VARZ)
        self.kind = as_kind(binning.kind)
        if kind is not None and as_kind(kind) is not self.kind:
            raise ValueError("feature map and binning spec must share one kind")
        self.bins = int(binning.bin_count)
        self.clamp = float(binning.upper_clamp)
        self.origin = np.asarray(grid.origin, dtype=np.float64).reshape(3)
        self.resolution = float(grid.resolution)
        self.include_phi = bool(include_phi)
        self.ctx = _lib.Context(device)
        self.ctx.set_tuning(table_cap=table_cap, threads=threads)
        self.ctx.set_passes(passes)
        self.ctx.set_params(self.origin, self.resolution, self.kind.code, self.bins, self.clamp,
                            self.include_phi)
        self._feat_a: FeatureMap | None = None

    # ---- scan A ---------------------------------------------------------------
    def set_reference(self, scan_a, fetch: bool = True) -> FeatureMap | None:
        """Voxelize + featurize scan A on the GPU (bit-exact), keep it resident.

        Returns the FeatureMap (copied back to the host) unless ``fetch`` is
        False; ``reference`` fetches it lazily later.
        """
        pts = _points_of(scan_a)
        if pts.shape[0] == 0:
            raise ValueError("cannot voxelize an empty cloud")
        if pts.dtype == np.float32 and pts.shape[1] == 4:
            self.ctx.set_reference_records(pts)  # KITTI records, 16 B/point, widened on the GPU
        else:
            self.ctx.set_reference_points(np.ascontiguousarray(pts[:, :3], dtype=np.float64))
        self._feat_a = None
        return self.reference if fetch else None

    def set_reference_features(self, feat_a) -> None:
        """Upload an existing FeatureMap (this package's or the reference's)."""
        if as_kind(feat_a.kind) is not self.kind:
            raise ValueError("feature map and binning spec must share one kind")
        self.ctx.set_reference_features(feat_a.keys, feat_a.values, feat_a.bounds)
        self._feat_a = feat_a

    @property
    def reference(self) -> FeatureMap | None:
        if self._feat_a is None:
            keys, vals, bounds = self.ctx.get_reference_features()
            self._feat_a = FeatureMap(kind=self.kind, keys=keys, values=vals, bounds=bounds)
        return self._feat_a

    # ---- scan B ---------------------------------------------------------------
    def set_query(self, scan_b) -> None:
        pts = _points_of(scan_b)
        if pts.shape[0] == 0:
            raise ValueError("cannot voxelize an empty cloud")
        if pts.dtype == np.float32 and pts.shape[1] == 4:
            self.ctx.set_query_records(pts)  # KITTI .bin records, float4 as is
        else:
            self.ctx.set_query_points(np.asarray(pts[:, :3], dtype=np.float64))
        hull = hull_vertices(pts)
        if hull is not None:
            self.ctx.set_query_hull(hull)

    # ---- many resident pairs (multi-pair kernel) ----------------------------------
    def set_pairs(self, pairs) -> None:
        """Make ``pairs`` = [(scan A, scan B), ...] resident at once (vmi_set_pairs):
        every scan A voxelized + featurized on the GPU, every scan B laid out.
        KITTI records (float32 (N, 4), or clouds read by scan_io) are uploaded as
        they are when every scan has them; otherwise all go as float64 points."""
        arrs = [(_points_of(a), _points_of(b)) for a, b in pairs]
        for a, b in arrs:
            if a.shape[0] == 0 or b.shape[0] == 0:
                raise ValueError("cannot voxelize an empty cloud")
        recs = all(x.dtype == np.float32 and x.shape[1] == 4 for ab in arrs for x in ab)
        if not recs:
            arrs = [tuple(np.ascontiguousarray(x[:, :3], dtype=np.float64) for x in ab)
                    for ab in arrs]
        self.ctx.set_pairs(arrs)
        self.n_pairs = len(arrs)

    def evaluate_pairs(self, poses, pair, histograms: bool = False):
        """mi_objective for pose i against resident pair ``pair[i]``, one launch:
        (mi, status, histogram identity) [+ counts (P, B+1, B+1)]."""
        mi, st, h, hist = self.ctx.eval_pairs(as_pose_array(poses), np.asarray(pair),
                                              want_hist=histograms, bins=self.bins)
        return (mi, st, h, hist) if histograms else (mi, st, h)

    # ---- scoring --------------------------------------------------------------
    @staticmethod
    def mats(poses) -> np.ndarray:
        return _lib.poses_to_mats(as_pose_array(poses))

    def evaluate(self, poses, histograms: bool = False, exact: bool = False):
        """Score P poses.  Returns (mi[P], status[P]) or, with histograms=True,
        (mi, status, counts[P, B+1, B+1], total[P])."""
        if exact:
            mi, st, hist, total = self.ctx.eval(self.mats(poses), want_hist=histograms,
                                                bins=self.bins, exact=True)
        else:  # pose -> matrix on the host, overlapped with the GPU (vmi_eval_poses)
            mi, st, hist, total = self.ctx.eval_poses(as_pose_array(poses, check_finite=False),
                                                      want_hist=histograms,
                                                      bins=self.bins)
        if histograms:
            return mi, st, hist, total
        return mi, st

    def evaluate_mats(self, mats: np.ndarray, histograms: bool = False, exact: bool = False):
        mi, st, hist, total = self.ctx.eval(mats, want_hist=histograms, bins=self.bins, exact=exact)
        return (mi, st, hist, total) if histograms else (mi, st)

    def evaluate_device(self, poses):
        """Score P poses leaving the results on the GPU: (mi, status) torch
        tensors on this engine's device (flagged poses already re-run on the
        exact path).  For device-side consumers (top-K, argmax)."""
        import torch
        mats_h = self.mats(poses)
        P = mats_h.shape[0]
        dev = torch.device("cuda", self.ctx.device)
        mats = torch.from_numpy(mats_h).to(dev)
        mi = torch.empty(P, dtype=torch.float64, device=dev)
        st = torch.empty(P, dtype=torch.int32, device=dev)
        s = torch.cuda.current_stream(dev).cuda_stream
        self.ctx.eval_device(mats.data_ptr(), P, mi.data_ptr(), st.data_ptr(), stream=s)
        self.ctx.eval_fixups(mats.data_ptr(), P, mi.data_ptr(), st.data_ptr(), stream=s)
        return mi, st

    def topk(self, poses, k: int):
        """The k best candidates by GPU MI: (mi[k] descending, index[k]);
        equal MI keep candidate order, so entry 0 is np.argmax's pick
        (before the near-tie re-score that ``best`` applies)."""
        mi, _ = self.evaluate_device(poses)
        s = __import__("torch").cuda.current_stream(mi.device).cuda_stream
        return self.ctx.topk_device(mi.data_ptr(), mi.numel(), k, stream=s)

    def best(self, poses, mi: np.ndarray | None = None, rel_tie: float = 1e-9,
             exact_value: bool = False):
        """np.argmax over the candidates' MI with the reference's tie semantics.

        GPU MI agrees with the reference to ~1e-14 relative (measured over the
        full C2 batch and a C3 slice: tests/test_gpu_headline_parity.py); the
        order of two poses can only differ when their MI values are that
        close.  Every candidate within ``rel_tie`` (1e-9, a wide margin over
        that bound) of the maximum is re-scored on the host from its
        bit-exact GPU histogram with the reference's own formula, and the
        first maximum in candidate order wins.  Returns (index, mi); with
        ``exact_value`` the winner's MI is always the host re-score (what a
        sharded search compares across ranks).
        """
        if mi is None:
            mi, _ = self.evaluate(poses)
        top = float(np.max(mi))
        if top <= NO_OVERLAP_SENTINEL:
            return int(np.argmax(mi)), top
        tied = np.nonzero(mi >= top - abs(top) * rel_tie)[0]
        if tied.size == 1 and not exact_value:
            return int(tied[0]), float(mi[tied[0]])
        _, _, hist, _ = self.evaluate(as_pose_array(poses)[tied], histograms=True)
        exact = np.array([mutual_information_exact(h, self.include_phi)[0] for h in hist])
        k = int(np.argmax(exact))
        return int(tied[k]), float(exact[k])

    def close(self):
        self.ctx.close()


def check_points(cloud) -> None:
    """Raise like the reference for invalid clouds (PointCloud validation)."""
    if isinstance(cloud, PointCloud):
        return
    PointCloud(np.asarray(_points_of(cloud))[:, :3])


__all__ = ["MIEngine", "entropy_exact", "mutual_information_exact", "OutOfBoundsError"]
