"""The native lockstep Nelder-Mead driver (csrc/nm_lockstep.cpp) on CPU, with
a Python objective: decision-for-decision the reference's optimizer
(nm_golden.npz: voxmi.nelder_mead_maximize on a closed-form objective), many
runs at once, and the numpy arithmetic it restates."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from paper_1709_06948_b200 import _lib
from paper_1709_06948_b200.optim import SimplexConfig, nelder_mead_maximize_batched


def nm_test_function(x):
    """tests/golden/make_golden.py's objective (unique maximum)."""
    x = np.asarray(x, dtype=np.float64)
    c = np.array([1.0, -2.0, 0.5, 0.1, -0.05, 0.3])
    w = np.array([1.0, 0.5, 2.0, 10.0, 10.0, 4.0])
    return float(np.exp(-np.sum(w * (x - c) ** 2)) + 0.1 * np.cos(x[0] - x[1]))


def _f_batch(P, R):
    vals = np.array([nm_test_function(p) for p in P])
    ids = np.array([hash(p.tobytes()) & 0xFFFFFFFFFFFFFFFF for p in P], dtype=np.uint64)
    return vals, ids


def _case(g, tag):
    cfg = g[f"{tag}_cfg"]
    return g[f"{tag}_x0"], g[f"{tag}_steps"], int(cfg[0]), float(cfg[1]), float(cfg[2]), int(cfg[3])


@pytest.mark.parametrize("spec", [-1, 0])
@pytest.mark.parametrize("tag", ["default", "restarts", "maxiter"])
def test_lockstep_matches_reference_optimizer(tag, spec):
    """spec -1: every iteration scores its four candidates at once; 0: the
    reflection first, then only the follow-up the reference needs."""
    g = golden("nm_golden.npz")
    x0, steps, it, ft, xt, rs = _case(g, tag)
    o = _lib.nm_run(x0[None, :], steps, it, ft, xt, rs, _f_batch, spec_budget=spec)
    np.testing.assert_array_equal(o["best_x"][0], g[f"{tag}_best_x"])
    assert o["best_value"][0] == float(g[f"{tag}_best_value"])
    assert o["iterations"][0] == int(g[f"{tag}_iterations"])
    assert _lib.NM_TERMINATION[o["termination"][0]] == str(g[f"{tag}_termination"])
    assert o["n_evaluations"][0] == int(g[f"{tag}_n_eval"])
    n = o["trace_len"][0]
    np.testing.assert_array_equal(o["trace"][0, :n], g[f"{tag}_trace"])


@pytest.mark.parametrize("lanes", ["1", "3"])
@pytest.mark.parametrize("spec", [-1, 0, 12])
def test_many_runs_in_lockstep_equal_single_runs(spec, lanes, monkeypatch):
    """K runs from different starts advance together (different iteration
    counts, restarts; spec 12 switches between one-probe and four-probe
    iterations as runs finish; 3 lanes deal the runs to interleaved batches as
    the GPU driver does): each equals the one-run optimizer exactly."""
    monkeypatch.setenv("VMI_NM_LANES", lanes)
    rng = np.random.default_rng(4)
    x0 = rng.normal(size=(9, 6)) * np.array([2, 2, 0.5, 0.1, 0.1, 0.3])
    cfg = SimplexConfig(initial_steps=(1.0, 1.0, 0.5, 0.05, 0.05, 0.2), max_iterations=120,
                        restarts=1, f_tol=1e-9, x_tol=1e-6)
    o = _lib.nm_run(x0, cfg.initial_steps, cfg.max_iterations, cfg.f_tol, cfg.x_tol, cfg.restarts,
                    _f_batch, spec_budget=spec)
    for k in range(x0.shape[0]):
        r = nelder_mead_maximize_batched(lambda P: np.array([nm_test_function(p) for p in P]),
                                         x0[k], cfg)
        np.testing.assert_array_equal(o["best_x"][k], r.best_x)
        assert o["best_value"][k] == r.best_value
        assert o["iterations"][k] == r.iterations
        assert _lib.NM_TERMINATION[o["termination"][k]] == r.termination
        assert o["n_evaluations"][k] == r.n_evaluations
        np.testing.assert_array_equal(o["trace"][k, :o["trace_len"][k]], r.trace)


def test_near_ties_of_different_sources_are_flagged():
    """Values that differ by less than the GPU error bound but come from
    different histograms cannot be ordered exactly: the run is `uncertain`."""
    def flat(P, R):  # all values equal, every pose its own source
        return np.full(P.shape[0], 0.5), np.arange(P.shape[0], dtype=np.uint64) + 1
    o = _lib.nm_run(np.zeros((1, 6)), np.ones(6), 10, 1e-5, 1e-3, 0, flat)
    assert o["uncertain"][0] == 1

    def same(P, R):  # all values equal and from one source: exact ties, certain
        return np.full(P.shape[0], 0.5), np.full(P.shape[0], 7, dtype=np.uint64)
    o = _lib.nm_run(np.zeros((1, 6)), np.ones(6), 10, 1e-5, 1e-3, 0, same)
    assert o["uncertain"][0] == 0


def test_bad_arguments():
    with pytest.raises(_lib.VmiError):
        _lib.nm_run(np.zeros((1, 6)), np.zeros(6), 10, 1e-5, 1e-3, 0, _f_batch)
