"""Pins of the Pivot MDS oracle (O8, oracle/pmds.py) against what mathematics
and SPEC.md's worked examples fix: farthest-first pivots on paths and cycles,
the max-min property against Floyd-Warshall distances (no BFS), the closed
form of the path graph with every vertex a pivot (C = x x^T, Y = -|x| x), the
square of C4, zero row/column sums of the double-centred matrix, and the
power-iteration eigenpairs against LAPACK's symmetric eigensolver."""
import numpy as np
import pytest

import oracle
from oracle import pmds as O
from workloads import cycle_graph, erdos_renyi, grid2d, path_graph, random_tree


def floyd_warshall(indptr, indices):
    n = len(indptr) - 1
    INF = 10 ** 9
    D = np.full((n, n), INF, dtype=np.int64)
    np.fill_diagonal(D, 0)
    for i in range(n):
        D[i, indices[indptr[i]:indptr[i + 1]]] = 1
    for m in range(n):
        D = np.minimum(D, D[:, m:m + 1] + D[m:m + 1, :])
    D[D >= INF] = n                                   # R21: unreachable counts as n
    return D


def test_spec_pivot_examples():
    ip, ix = path_graph(5)
    piv, _ = O.select_pivots(ip, ix, 2, first=0)
    assert piv == [0, 4]                              # farthest point on a path
    ip, ix = cycle_graph(6)
    piv, _ = O.select_pivots(ip, ix, 2, first=0)
    assert piv == [0, 3]                              # antipode
    ip, ix = path_graph(7)
    piv, _ = O.select_pivots(ip, ix, 7, seed=3)
    assert sorted(piv) == list(range(7))              # pivot_count = n takes every vertex


@pytest.mark.parametrize("make", [lambda: erdos_renyi(40, 0.08, 1), lambda: random_tree(35, 2),
                                  lambda: grid2d(6, 5), lambda: erdos_renyi(30, 0.04, 5)])
@pytest.mark.parametrize("seed", [0, 7])
def test_max_min_property_brute_force(make, seed):
    ip, ix = make()
    n = len(ip) - 1
    D = floyd_warshall(ip, ix)
    p = min(n, 9)
    piv, hops = O.select_pivots(ip, ix, p, seed)
    assert piv[0] == O.first_pivot(n, seed)
    assert np.array_equal(hops, D[:, piv])
    for t in range(1, p):
        dmin = D[:, piv[:t]].min(axis=1)
        best = dmin.max()
        assert piv[t] == int(np.flatnonzero(dmin == best)[0])


@pytest.mark.parametrize("n", [5, 12, 31])
def test_path_closed_form(n):
    """Every vertex a pivot on P_n: D2 = (i - j)^2, so C = x x^T with
    x_i = i - (n-1)/2; G = |x|^2 x x^T; v1 = -x/|x| after orientation (the
    largest |entries| are the two ends, the first of them, i = 0, is made
    positive); Y[:, 0] = C v1 = -|x| x; rank 1, so Y[:, 1] = 0 (R22)."""
    ip, ix = path_graph(n)
    piv, hops = O.select_pivots(ip, ix, n, seed=1)
    order = np.argsort(piv)
    Y, (l1, l2, V) = O.embed(hops[:, order], seed=1)
    x = np.arange(n) - (n - 1) / 2.0
    assert np.allclose(Y[:, 0], -np.linalg.norm(x) * x, rtol=1e-9, atol=1e-9 * np.linalg.norm(x) ** 2)
    assert np.all(Y[:, 1] == 0.0)
    assert abs(l1 - np.linalg.norm(x) ** 4) <= 1e-9 * l1


def test_c4_square():
    ip, ix = cycle_graph(4)
    r = O.pmds(ip, ix, 4, seed=0)
    Y = r["Y"]
    d = sorted(np.linalg.norm(Y[i] - Y[j]) for i in range(4) for j in range(i + 1, 4))
    assert np.allclose(d[:4], d[0], rtol=1e-9) and np.allclose(d[4:], d[0] * np.sqrt(2), rtol=1e-9)


@pytest.mark.parametrize("make,p", [(lambda: grid2d(9, 7), 20), (lambda: erdos_renyi(120, 0.05, 3), 30),
                                    (lambda: random_tree(90, 4), 25)])
def test_centring_and_eigenpairs(make, p):
    ip, ix = make()
    r = O.pmds(ip, ix, p, seed=2)
    C = O.centred(r["hops"])
    assert np.abs(C.sum(axis=0)).max() <= 1e-9 * np.abs(C).max() * C.shape[0]
    assert np.abs(C.sum(axis=1)).max() <= 1e-9 * np.abs(C).max() * C.shape[1]
    G = C.T @ C
    ev = np.linalg.eigvalsh(G)[::-1]                  # LAPACK, not power iteration
    assert abs(r["l1"] - ev[0]) <= 1e-8 * ev[0]
    if ev[1] - ev[2] > 1e-3 * ev[0]:                  # a gap: the second pair is unique
        assert abs(r["l2"] - ev[1]) <= 1e-6 * ev[0]
    for k, lam in ((0, r["l1"]), (1, r["l2"])):
        v = r["V"][:, k]
        assert np.linalg.norm(G @ v - lam * v) <= 1e-6 * ev[0]
    assert abs(r["V"][:, 0] @ r["V"][:, 1]) <= 1e-8
    assert np.abs(r["Y"].mean(axis=0)).max() <= 1e-9 * np.abs(r["Y"]).max()


def test_disconnected_counts_unreachable_as_n():
    ip, ix = erdos_renyi(25, 0.02, 11)               # several components
    n = len(ip) - 1
    piv, hops = O.select_pivots(ip, ix, 5, seed=0)
    D = floyd_warshall(ip, ix)
    assert np.array_equal(hops, D[:, piv]) and (hops == n).any()
