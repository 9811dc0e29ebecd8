"""The batched speculative Nelder-Mead reproduces the reference optimizer
(optim.py:62-175) decision for decision on a closed-form objective: same
best point, trace, spreads, iterations, termination and evaluation count
(golden vectors from voxmi.nelder_mead_maximize)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from paper_1709_06948_b200.optim import SimplexConfig, nelder_mead_maximize_batched


def f(x):
    x = np.asarray(x, dtype=np.float64)
    c = np.array([1.0, -2.0, 0.5, 0.1, -0.05, 0.3])
    w = np.array([1.0, 0.5, 2.0, 10.0, 10.0, 4.0])
    return float(np.exp(-np.sum(w * (x - c) ** 2)) + 0.1 * np.cos(x[0] - x[1]))


@pytest.mark.parametrize("tag", ["default", "restarts", "maxiter"])
def test_batched_nm_matches_reference(tag):
    g = golden("nm_golden.npz")
    mi, ft, xt, rs = g[f"{tag}_cfg"]
    cfg = SimplexConfig(initial_steps=tuple(g[f"{tag}_steps"]), max_iterations=int(mi),
                        f_tol=float(ft), x_tol=float(xt), restarts=int(rs))
    batches = []

    def fb(X):
        batches.append(len(X))
        return np.array([f(x) for x in X])

    r = nelder_mead_maximize_batched(fb, g[f"{tag}_x0"], cfg)
    np.testing.assert_array_equal(r.best_x, g[f"{tag}_best_x"])
    assert r.best_value == float(g[f"{tag}_best_value"])
    assert r.iterations == int(g[f"{tag}_iterations"])
    assert r.termination == str(g[f"{tag}_termination"])
    np.testing.assert_array_equal(r.trace, g[f"{tag}_trace"])
    np.testing.assert_array_equal(r.trace_spread, g[f"{tag}_spread"])
    assert r.n_evaluations == int(g[f"{tag}_n_eval"])
    assert len(batches) < r.n_evaluations  # evaluations were batched


def test_config_validation():
    with pytest.raises(ValueError):
        SimplexConfig(initial_steps=(1.0, 0.0))
    with pytest.raises(ValueError):
        SimplexConfig(max_iterations=0)
    with pytest.raises(ValueError):
        SimplexConfig(restarts=-1)
    with pytest.raises(ValueError):
        nelder_mead_maximize_batched(lambda X: np.zeros(len(X)), np.zeros(3), SimplexConfig())
