"""align(): the reference's Algorithm-1 driver on the GPU objective.

Same contract as the reference `align` (align.py:122-159): scan A voxelized
once, Nelder-Mead over the 6-DOF pose from ``t0``, NoOverlapError when every
probe is the sentinel, report with the normalised estimate and a final MI.
Candidates are scored in batches on the GPU (optim.nelder_mead_maximize_batched);
each objective value is the reference's own MI formula (numpy sort + sum,
mi.py:163-191) applied on the host to the bit-exact GPU histogram, so values
-- and hence every simplex decision -- are identical to the reference's.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass

import numpy as np

from ._lib import poses_to_mats
from .engine import MIEngine, mutual_information_exact
from .errors import NoOverlapError
from .geometry import (EulerPose, as_pose_array, euler_to_transform, normalized,
                       transform_to_euler, validate_transform)
from .optim import OptimResult, SimplexConfig, nelder_mead_maximize_batched
from .types import NO_OVERLAP_SENTINEL, AlignmentConfig


@dataclass
class AlignmentReport:
    """Estimated transform plus optimisation diagnostics (align.py:70-111)."""

    estimated: np.ndarray
    estimated_pose: EulerPose
    initial_pose: EulerPose
    final_mi: float
    mi_trace: list
    iterations: int
    wall_time: float
    termination: str
    n_evaluations: int = 0
    n_batches: int = 0

    def to_dict(self) -> dict:
        def pose(p):
            return {"tx": p.tx, "ty": p.ty, "tz": p.tz, "rx": p.rx, "ry": p.ry, "rz": p.rz}
        return {
            "estimated_matrix": [[float(v) for v in row] for row in self.estimated],
            "estimated_pose": pose(self.estimated_pose),
            "initial_pose": pose(self.initial_pose),
            "final_mi": self.final_mi,
            "mi_trace": list(self.mi_trace),
            "iterations": self.iterations,
            "wall_time": self.wall_time,
            "termination": self.termination,
            "kitti_line": self.kitti_line(),
        }

    def kitti_line(self) -> str:
        return " ".join(repr(float(v)) for v in self.estimated[:3, :].ravel())

    def write_json(self, path) -> None:
        with open(path, "w") as fh:
            json.dump(self.to_dict(), fh, indent=2)
            fh.write("\n")


def exact_objective(eng: MIEngine):
    """(k, 6) poses -> reference-identical MI values (sentinel when invalid)."""
    def f_batch(x: np.ndarray) -> np.ndarray:
        poses = as_pose_array(np.asarray(x, dtype=np.float64))
        _, st, hist, _ = eng.evaluate(poses, histograms=True)
        out = np.empty(poses.shape[0])
        for i in range(poses.shape[0]):
            out[i] = (mutual_information_exact(hist[i], eng.include_phi)[0] if st[i] == 0
                      else NO_OVERLAP_SENTINEL)
        return out
    return f_batch


def _simplex_of(cfg: AlignmentConfig) -> SimplexConfig:
    simplex = cfg.simplex if isinstance(cfg.simplex, SimplexConfig) else (
        SimplexConfig(**{k: getattr(cfg.simplex, k) for k in
                         ("initial_steps", "max_iterations", "f_tol", "x_tol", "restarts")})
        if cfg.simplex is not None else SimplexConfig())
    if len(simplex.initial_steps) != 6:
        raise ValueError("simplex initial_steps must have 6 entries")
    return simplex


def align(scan_a, scan_b, t0, cfg: AlignmentConfig | None = None,
          device: int = 0) -> AlignmentReport:
    """Estimate the transform projecting scan B onto scan A (align.py:122-159)."""
    cfg = cfg or AlignmentConfig()
    simplex = _simplex_of(cfg)
    t0 = validate_transform(t0)
    n_a = len(getattr(scan_a, "points", scan_a))
    n_b = len(getattr(scan_b, "points", scan_b))
    if n_a == 0 or n_b == 0:
        raise ValueError("both scans must be non-empty")
    eng = MIEngine(grid=cfg.grid, binning=cfg.binning, include_phi=cfg.phi_enabled, device=device)
    try:
        eng.set_reference(scan_a)
        eng.set_query(scan_b)
        initial_pose = transform_to_euler(t0)
        f_batch = exact_objective(eng)
        start = time.perf_counter()
        result: OptimResult = nelder_mead_maximize_batched(f_batch, initial_pose.as_vector(),
                                                           simplex)
        wall = time.perf_counter() - start
        if result.best_value <= NO_OVERLAP_SENTINEL:
            raise NoOverlapError("no candidate pose produced overlapping occupied bounds")
        estimated_pose = normalized(EulerPose.from_vector(result.best_x))
        final_mi = float(f_batch(estimated_pose.as_vector()[None, :])[0])
    finally:
        eng.close()
    return AlignmentReport(
        estimated=euler_to_transform(estimated_pose),
        estimated_pose=estimated_pose,
        initial_pose=initial_pose,
        final_mi=final_mi,
        mi_trace=[*result.trace, final_mi],
        iterations=result.iterations,
        wall_time=wall,
        termination=result.termination,
        n_evaluations=result.n_evaluations,
        n_batches=result.n_batches,
    )


def align_batch(pairs, t0s, cfg: AlignmentConfig | None = None, device: int = 0,
                raise_errors: bool = True, stats: dict | None = None,
                engine: MIEngine | None = None) -> list:
    """``align`` for many scan pairs at once (C5: a drive's consecutive pairs).

    Every pair's scans are resident together and all Nelder-Mead runs advance
    in lockstep inside the library (vmi_align_pairs): one multi-pair kernel
    launch per step scores every run's pending probes.  Decisions are the
    reference's (align.py:122-159 / optim.py:62-175) on GPU MI values; a run
    that met a comparison those values cannot decide exactly (operands within
    the GPU's error bound, different histograms) is redone with ``align`` on
    exact values, so every report is the reference's.  Each report's
    ``final_mi`` is the reference formula on the estimate's bit-exact
    histogram; ``mi_trace`` holds GPU MI values (within ~1e-13).  A pair with
    no overlapping probe raises ``NoOverlapError`` (or, with ``raise_errors``
    False, gets the exception in its slot).  ``wall_time`` is the batch's
    optimisation time (all pairs together); ``stats`` (a dict) receives counts.
    ``engine``: an MIEngine built for ``cfg`` to reuse (its grow-only device
    buffers survive across calls, e.g. a drive aligned in batches).
    """
    from ._lib import NM_TERMINATION
    cfg = cfg or AlignmentConfig()
    simplex = _simplex_of(cfg)
    pairs = list(pairs)
    if len(t0s) != len(pairs):
        raise ValueError("one start transform per pair")
    if not pairs:
        return []
    init = [transform_to_euler(validate_transform(t)) for t in t0s]
    eng = engine or MIEngine(grid=cfg.grid, binning=cfg.binning, include_phi=cfg.phi_enabled,
                             device=device)
    K = len(pairs)
    t_set = time.perf_counter()
    try:
        eng.set_pairs(pairs)
        start = time.perf_counter()
        o = eng.ctx.align_pairs(np.stack([p.as_vector() for p in init]), simplex.initial_steps,
                                simplex.max_iterations, simplex.f_tol, simplex.x_tol,
                                simplex.restarts)
        wall = time.perf_counter() - start
        est = [normalized(EulerPose.from_vector(o["best_x"][k])) for k in range(K)]
        est_vec = np.stack([e.as_vector() for e in est])
        _, st, _, hist = eng.evaluate_pairs(est_vec, np.arange(K), histograms=True)
        t_final = time.perf_counter()
    finally:
        if engine is None:
            eng.close()
    # euler_to_transform of every estimate in one native call (the same bits)
    est_mats = poses_to_mats(est_vec)
    out = []
    redo = 0
    for k in range(K):
        if o["uncertain"][k]:
            redo += 1
            try:
                out.append(align(pairs[k][0], pairs[k][1], t0s[k], cfg, device))
            except NoOverlapError as e:
                if raise_errors:
                    raise
                out.append(e)
            continue
        if o["best_value"][k] <= NO_OVERLAP_SENTINEL:
            err = NoOverlapError("no candidate pose produced overlapping occupied bounds")
            if raise_errors:
                raise err
            out.append(err)
            continue
        final_mi = (mutual_information_exact(hist[k], cfg.phi_enabled)[0] if st[k] == 0
                    else NO_OVERLAP_SENTINEL)
        n = int(o["trace_len"][k])
        estimated = np.eye(4)
        estimated[:3, :3] = est_mats[k, :9].reshape(3, 3)
        estimated[:3, 3] = est_mats[k, 9:]
        out.append(AlignmentReport(
            estimated=estimated, estimated_pose=est[k], initial_pose=init[k],
            final_mi=float(final_mi), mi_trace=[*o["trace"][k, :n].tolist(), float(final_mi)],
            iterations=int(o["iterations"][k]), wall_time=wall,
            termination=NM_TERMINATION[int(o["termination"][k])],
            n_evaluations=int(o["n_evaluations"][k])))
    if stats is not None:
        stats.update(pairs=K, redone_exact=redo, wall_time=wall,
                     evaluations=int(np.sum(o["n_evaluations"])),
                     set_pairs_s=start - t_set, final_eval_s=t_final - start - wall,
                     reports_s=time.perf_counter() - t_final)
    return out
