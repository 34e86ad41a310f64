"""Pins of the quadtree (Barnes-Hut) oracle O9 (oracle/bh.py): theta = 0 is the
exact gradient O4a (itself pinned by finite differences) including Z and the
entropy sums; the error against it shrinks as theta shrinks; every node's
points lie inside its cell and the levels nest; translation invariance."""
import numpy as np
import pytest

import oracle
from oracle import bh as B
from workloads import clustered_layout, grid2d, uniform_layout


def relL2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def P1():
    ip, ix = grid2d(14, 13)                           # n = 182: the O(n^2) Python sums stay fast
    return oracle.build_P(ip, ix, 10.0, seed=0)


LAM = (1.0, 0.01, 0.6)


def layouts(n):
    return [clustered_layout(n, 20.0, 5, 1.5, 7).astype(np.float64), uniform_layout(n, 3.0, 4).astype(np.float64)]


def test_theta_zero_is_exact(P1):
    for X in layouts(P1["n"]):
        r = B.bh_gradient(X, P1["indptr"], P1["indices"], P1["values"], *LAM, eps=0.05, theta=0.0)
        g, Z = oracle.exact_grad(X, P1["indptr"], P1["indices"], P1["values"], *LAM, eps=0.05)
        assert relL2(r["g"], g) <= 1e-12
        assert abs(r["Z"] - Z) <= 1e-12 * Z
        e = B.bh_gradient(X, P1["indptr"], P1["indices"], P1["values"], *LAM, eps=0.05, theta=0.0, repulsion=False)
        ge, _ = oracle.exact_grad(X, P1["indptr"], P1["indices"], P1["values"], 0.0, 0.0, LAM[2], eps=0.05)
        assert relL2(e["g"], ge) <= 1e-12


def test_error_shrinks_with_theta(P1):
    X = layouts(P1["n"])[0]
    g, _ = oracle.exact_grad(X, P1["indptr"], P1["indices"], P1["values"], *LAM, eps=0.05)
    errs = [relL2(B.bh_gradient(X, P1["indptr"], P1["indices"], P1["values"], *LAM, eps=0.05, theta=t)["g"], g)
            for t in (0.8, 0.5, 0.25, 0.1)]
    assert errs[-1] < 2e-3 and errs[-1] < errs[0]
    assert all(b <= a * 1.2 for a, b in zip(errs, errs[1:]))


@pytest.mark.parametrize("n", [1, 2, 17, 500])
def test_tree_cells_and_nesting(n):
    X = uniform_layout(n, 5.0, n).astype(np.float64)
    X[: n // 4] = X[0]                               # coincident points (depth-16 leaves)
    T = B.Quadtree(X)
    Xs = X[T.perm]
    for lev in range(B.DEPTH + 1):
        st = T.starts[lev]
        if lev < B.DEPTH:
            assert set(st.tolist()) <= set(T.starts[lev + 1].tolist())
        side = T.S / 2.0 ** lev
        for k in range(len(st) - 1):
            s, e = st[k], st[k + 1]
            pre = int(T.code[s]) >> (2 * (B.DEPTH - lev))
            cx = sum(((pre >> (2 * b)) & 1) << b for b in range(lev))
            cy = sum(((pre >> (2 * b + 1)) & 1) << b for b in range(lev))
            pts = Xs[s:e]
            tol = 1e-12 * T.S
            assert np.all(pts[:, 0] >= T.lo_x + cx * side - tol) and np.all(pts[:, 0] <= T.lo_x + (cx + 1) * side + tol)
            assert np.all(pts[:, 1] >= T.lo_y + cy * side - tol) and np.all(pts[:, 1] <= T.lo_y + (cy + 1) * side + tol)


def test_translation_invariance(P1):
    X = layouts(P1["n"])[0]
    a = B.bh_gradient(X, P1["indptr"], P1["indices"], P1["values"], 1.0, 0.0, 0.6, theta=0.5)
    b = B.bh_gradient(X + np.array([0.375, -1.25]), P1["indptr"], P1["indices"], P1["values"], 1.0, 0.0, 0.6,
                      theta=0.5)
    assert relL2(b["g"], a["g"]) <= 1e-9
