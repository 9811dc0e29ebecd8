"""Serial Nelder-Mead + align loop of the reference, restated (TEST INFRASTRUCTURE).

Only tests/ and bench.py's CPU-baseline legs use this.  ``nelder_mead_maximize``
restates the reference optimizer (pkg/src/voxmi/optim.py:62-175: one objective
call per probe, canonical coefficients, anisotropic initial simplex, stable
sort, f/x spread tests, restarts with halved steps, best-ever tracking), and
``align_pair`` the reference's align loop (align.py:122-159) on the oracle's
mi_objective -- the CPU baseline of C5's scan-pair alignments/s.  Pinned to
the reference's own optimizer run (tests/golden/nm_golden.npz) by
tests/test_oracle.py.
"""

from __future__ import annotations

import numpy as np

from . import feature_map, mi_objective_full, poses_to_mats

SENTINEL = -1e300


def nelder_mead_maximize(f, x0, steps, max_iterations=300, f_tol=1e-5, x_tol=1e-3, restarts=0):
    """optim.py:62-175.  Returns (best_x, best_value, iterations, termination,
    trace, n_evaluations)."""
    x0 = np.asarray(x0, dtype=np.float64)
    n = x0.size
    state = {"x": None, "g": np.inf, "n": 0}

    def g(x):
        v = -f(x)
        state["n"] += 1
        if v < state["g"]:
            state["g"] = v
            state["x"] = x.copy()
        return v

    def initial(center, st):
        s = np.tile(center, (n + 1, 1))
        for i in range(n):
            s[i + 1, i] += st[i]
        return s

    st = np.asarray(steps, dtype=np.float64)
    simplex = initial(x0, st)
    values = np.array([g(v) for v in simplex])
    iteration, left, trace, term = 0, restarts, [], "max_iter"
    while True:
        order = np.argsort(values, kind="stable")
        simplex, values = simplex[order], values[order]
        f_spread = float(values[-1] - values[0])
        x_spread = float(np.linalg.norm(simplex - simplex[0], axis=1).max())
        trace.append(-float(values[0]))
        conv = "converged_f" if f_spread < f_tol else ("converged_x" if x_spread < x_tol else None)
        if conv is not None:
            if left > 0 and iteration < max_iterations:
                left -= 1
                st = st * 0.5
                simplex = initial(simplex[0], st)
                values = np.concatenate([values[:1], [g(v) for v in simplex[1:]]])
                continue
            term = conv
            break
        if iteration >= max_iterations:
            break
        iteration += 1
        c = simplex[:-1].mean(axis=0)
        w = simplex[-1]
        r = c + 1.0 * (c - w)
        gr = g(r)
        if gr < values[0]:
            e = c + 2.0 * (c - w)
            ge = g(e)
            simplex[-1], values[-1] = (e, ge) if ge < gr else (r, gr)
            continue
        if gr < values[-2]:
            simplex[-1], values[-1] = r, gr
            continue
        if gr < values[-1]:
            k = c + 0.5 * (r - c)
            gk = g(k)
            if gk <= gr:
                simplex[-1], values[-1] = k, gk
                continue
        else:
            k = c - 0.5 * (c - w)
            gk = g(k)
            if gk < values[-1]:
                simplex[-1], values[-1] = k, gk
                continue
        for i in range(1, n + 1):
            simplex[i] = simplex[0] + 0.5 * (simplex[i] - simplex[0])
            values[i] = g(simplex[i])
    return state["x"], -state["g"], iteration, term, trace, state["n"]


def align_pair(a_pts, b_pts, x0, steps, res=1.0, kind="varz", max_iterations=300, f_tol=1e-5,
               x_tol=1e-3, restarts=0):
    """align.py:122-159 on the oracle: scan A's feature map once, then the
    serial optimizer over mi_objective.  Returns nelder_mead_maximize's tuple."""
    fa = feature_map(np.asarray(a_pts, dtype=np.float64), (0, 0, 0), res, kind)
    pts = np.ascontiguousarray(b_pts, dtype=np.float64)

    def objective(x):
        return mi_objective_full(fa, pts, poses_to_mats(x)[0], res=res)[0]
    return nelder_mead_maximize(objective, x0, steps, max_iterations, f_tol, x_tol, restarts)
