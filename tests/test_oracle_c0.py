"""Pins of the C0 oracle (O1-O3) against things the paper and mathematics fix:
brute-force all-pairs shortest paths (Floyd-Warshall / scipy), reference
SplitMix64 outputs, SPEC.md worked examples, an independent root-finder for
the perplexity equation, and a dense Eq. 2-3 build when k = n-1."""
import math
import os

import numpy as np
import pytest
from scipy.optimize import brentq
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import shortest_path

import oracle
from workloads import (complete_graph, cycle_graph, erdos_renyi, grid2d, path_graph, random_tree,
                       star_graph)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.strip() for ln in f if ln.strip() and not ln.startswith("#")]


def floyd_warshall(indptr, indices):
    """Plain O(n^3) Floyd-Warshall on hop counts (independent of any BFS)."""
    n = len(indptr) - 1
    INF = 10 ** 9
    D = np.full((n, n), INF, dtype=np.int64)
    np.fill_diagonal(D, 0)
    for i in range(n):
        D[i, indices[indptr[i]:indptr[i + 1]]] = 1
    for m in range(n):
        D = np.minimum(D, D[:, m:m + 1] + D[m:m + 1, :])
    return D


def test_splitmix64_reference_vectors():
    ref = [int(x, 16) for x in _golden_lines("splitmix64_seed0.txt")]
    g = 0x9E3779B97F4A7C15
    got = [oracle.splitmix64((i * g) & 0xFFFFFFFFFFFFFFFF) for i in range(4)]
    assert got == ref


def test_tie_key_definition():
    # key(v,w) = SplitMix64(seed ^ (v<<32 | w)) -- R4
    for seed, v, w in [(0, 0, 1), (7, 3, 9), (123456789, 1000, 999_999)]:
        assert oracle.tie_key(seed, v, w) == oracle.splitmix64(seed ^ ((v << 32) | w))


SMALL_GRAPHS = [
    ("path7", lambda: path_graph(7)),
    ("cycle9", lambda: cycle_graph(9)),
    ("star6", lambda: star_graph(6)),
    ("grid5x4", lambda: grid2d(5, 4)),
    ("tree25", lambda: random_tree(25, 3)),
    ("er30", lambda: erdos_renyi(30, 0.12, 5)),
    ("er40_disconnected", lambda: erdos_renyi(40, 0.04, 11)),
]


@pytest.mark.parametrize("name,make", SMALL_GRAPHS)
@pytest.mark.parametrize("k", [1, 3, 6, 12])
@pytest.mark.parametrize("seed", [0, 99])
def test_knn_matches_floyd_warshall(name, make, k, seed):
    """O1 equals the brute-force definition: all vertices sorted by
    (hop distance, key(v,w), w), first k of those reachable."""
    ip, ix = make()
    n = len(ip) - 1
    D = floyd_warshall(ip, ix)
    kk = min(k, n - 1)
    idx, hop, ln = oracle.knn(ip, ix, kk, seed)
    for v in range(n):
        cand = [(int(D[v, w]), oracle.tie_key(seed, v, w), w) for w in range(n)
                if w != v and D[v, w] < 10 ** 9]
        cand.sort()
        want = sorted((d, w) for d, _, w in cand[:kk])
        got = sorted(zip(hop[v, :ln[v]].tolist(), idx[v, :ln[v]].tolist()))
        assert got == want, (name, v)
        # rows are stored sorted by (hop, w)
        assert list(zip(hop[v, :ln[v]], idx[v, :ln[v]])) == want


def test_knn_distances_match_scipy_on_grid():
    ip, ix = grid2d(12, 9)
    n = len(ip) - 1
    A = csr_matrix((np.ones(len(ix)), ix, ip), shape=(n, n))
    D = shortest_path(A, unweighted=True)
    idx, hop, ln = oracle.knn(ip, ix, 30, 4)
    for v in range(n):
        assert np.array_equal(hop[v, :ln[v]], D[v, idx[v, :ln[v]]].astype(np.int32))


def test_spec_partial_knn_examples():
    # SPEC.md:104 P5, v=2, k=2 -> {(1,1),(3,1)}
    ip, ix = path_graph(5)
    idx, hop, ln = oracle.knn(ip, ix, 2, 0, src=[2])
    assert sorted(zip(idx[0, :ln[0]], hop[0, :ln[0]])) == [(1, 1), (3, 1)]
    # SPEC.md:106 P3, v=0, k=10 -> capped {(1,1),(2,2)}
    ip, ix = path_graph(3)
    idx, hop, ln = oracle.knn(ip, ix, 10, 0, src=[0])
    assert ln[0] == 2 and sorted(zip(idx[0, :2], hop[0, :2])) == [(1, 1), (2, 2)]


def test_star_tie_break_is_uniform():
    # SPEC.md:105 star K1,5 centre, k=3: each leaf chosen with prob 3/5;
    # over 10000 seeded trials 6000 +- 200 (4 sigma of Binomial(10000, 0.6)).
    ip, ix = star_graph(5)
    counts = np.zeros(6, dtype=np.int64)
    for seed in range(10000):
        idx, _, ln = oracle.knn(ip, ix, 3, seed, src=[0])
        counts[idx[0, :3]] += 1
    assert counts[0] == 0
    assert np.all(np.abs(counts[1:] - 6000) <= 200), counts


def test_knn_k_equals_n_minus_1_takes_everything():
    ip, ix = erdos_renyi(30, 0.2, 2)
    idx, hop, ln = oracle.knn(ip, ix, 29, 1)
    for v in range(30):
        assert sorted(idx[v, :ln[v]].tolist()) == [w for w in range(30) if w != v]


def test_resolve_k():
    assert oracle.resolve_k(10 ** 6, 40.0) == 120     # k = 3u
    assert oracle.resolve_k(50, 40.0) == 49           # capped at n-1 (R5)
    assert oracle.resolve_k(1000, 2.5) == 8           # round half up


# ----------------------------------------------------------------- calibration
def perplexity2(p):
    p = p[p > 0]
    return 2.0 ** (-(p * np.log2(p)).sum())


def test_calibration_hits_perplexity_and_sums_to_one():
    rng = np.random.default_rng(0)
    for _ in range(200):
        L = int(rng.integers(10, 150))
        u = float(rng.uniform(1.5, 0.9 * L))
        hops = np.sort(rng.integers(1, 8, size=L)).astype(np.int32)
        cmin = int((hops == hops.min()).sum())
        p, beta = oracle.calibrate_row(hops, u)
        assert abs(p.sum() - 1.0) < 1e-12
        if cmin < u:
            # north star: |log2 Perp - log2 u| <= 1e-5
            assert abs(math.log2(perplexity2(p)) - math.log2(u)) <= 1e-5


def test_calibration_matches_independent_root_finder():
    """Eq. 3 solved independently with brentq on sigma."""
    rng = np.random.default_rng(1)
    for _ in range(50):
        L = int(rng.integers(20, 130))
        hops = np.sort(rng.integers(1, 7, size=L)).astype(np.int32)
        cmin = int((hops == hops.min()).sum())
        u = float(rng.uniform(cmin + 0.5, L - 0.5)) if cmin + 1 < L else None
        if u is None:
            continue
        d2 = hops.astype(np.float64) ** 2

        def logperp(log_sigma):
            s2 = math.exp(2 * log_sigma)
            e = np.exp(-(d2 - d2.min()) / (2 * s2))
            q = e / e.sum()
            q = q[q > 0]
            return -(q * np.log2(q)).sum() - math.log2(u)

        ls = brentq(logperp, -6.0, 12.0, xtol=1e-15, rtol=1e-15, maxiter=500)
        s2 = math.exp(2 * ls)
        e = np.exp(-(d2 - d2.min()) / (2 * s2))
        want = e / e.sum()
        p, beta = oracle.calibrate_row(hops, u)
        assert np.allclose(p, want, rtol=1e-9, atol=1e-15)
        assert abs(beta - 1.0 / (2 * s2)) <= 1e-8 * max(1.0, beta)


def test_calibration_spec_examples_and_special_cases():
    # SPEC.md:114 three neighbours at distance 1, u=3 -> uniform 1/3
    p, _ = oracle.calibrate_row(np.array([1, 1, 1], np.int32), 3.0)
    assert np.allclose(p, 1 / 3)
    # SPEC.md:116 distances {1,1,4,4}, u=2: all mass on the two distance-1 entries (perplexity 2)
    p, beta = oracle.calibrate_row(np.array([1, 1, 4, 4], np.int32), 2.0)
    assert np.allclose(p, [0.5, 0.5, 0, 0]) and math.isinf(beta)
    # row length <= u -> beta = 0, uniform (perplexity cannot exceed the row length)
    p, beta = oracle.calibrate_row(np.array([1, 2, 3, 3, 5], np.int32), 40.0)
    assert beta == 0.0 and np.allclose(p, 0.2)
    # c_min >= u (R6, unreachable perplexity): uniform on the min-distance set
    p, beta = oracle.calibrate_row(np.array([1] * 50 + [2] * 70, np.int32), 40.0)
    assert math.isinf(beta) and np.allclose(p[:50], 1 / 50) and np.all(p[50:] == 0)


def test_entropy_monotone_in_sigma():
    # increasing sigma never decreases the perplexity.
    hops = np.array([1, 1, 2, 2, 2, 3, 3, 4, 5, 6] * 5, np.int32)
    perps = []
    for u in np.linspace(6, 45, 30):
        p, beta = oracle.calibrate_row(hops, float(u))
        perps.append((beta, perplexity2(p)))
    perps.sort(key=lambda t: -t[0])            # decreasing beta = increasing sigma
    vals = [pp for _, pp in perps]
    assert all(b >= a - 1e-9 for a, b in zip(vals, vals[1:]))


# -------------------------------------------------------------- symmetrise
def test_eq2_arithmetic():
    # p_j|i = 1/3, p_i|j = 0, n = 10 -> p_ij = 1/60
    val = float(_golden_lines("spec_closed_forms.txt")[5].split("|")[1])
    n, k = 10, 1
    idx = np.full((n, k), -1, np.int32)
    ln = np.zeros(n, np.int32)
    pc = np.zeros((n, k))
    idx[0, 0], ln[0], pc[0, 0] = 1, 1, 1.0 / 3.0
    ip, ix, v = oracle.symmetrize(n, idx, ln, pc)
    assert ip[1] - ip[0] == 1 and ix[0] == 1 and abs(v[0] - val) < 1e-18
    assert ip[2] - ip[1] == 1 and ix[1] == 0 and abs(v[1] - val) < 1e-18


@pytest.mark.parametrize("make", [lambda: grid2d(10, 10), lambda: erdos_renyi(60, 0.08, 3),
                                  lambda: random_tree(80, 1), lambda: star_graph(70)])
def test_symmetric_P_invariants(make):
    ip, ix = make()
    P = oracle.build_P(ip, ix, u=8.0, seed=5)
    n = P["n"]
    A = csr_matrix((P["values"], P["indices"], P["indptr"]), shape=(n, n))
    # total mass: each non-empty conditional row contributes 1/n
    assert abs(A.sum() - (P["knn_len"] > 0).sum() / n) < 1e-12
    assert abs(A - A.T).max() < 1e-18                       # p_ij = p_ji exactly
    assert np.all(P["values"] > 0)
    for i in range(n):                                       # columns strictly ascending
        assert np.all(np.diff(P["indices"][P["indptr"][i]:P["indptr"][i + 1]]) > 0)
    assert np.allclose(P["p_cond"].sum(axis=1)[P["knn_len"] > 0], 1.0, atol=1e-12)


def test_C4_all_entries_equal():
    # SPEC.md:125 C4, u=1 (k=3): all 8 stored p_ij equal, total mass 1.
    ip, ix = cycle_graph(4)
    P = oracle.build_P(ip, ix, u=1.0, seed=0)
    assert P["k"] == 3
    A = csr_matrix((P["values"], P["indices"], P["indptr"]), shape=(4, 4)).toarray()
    nz = A[A > 0]
    assert len(nz) == 8 and np.allclose(nz, nz[0]) and abs(A.sum() - 1) < 1e-15


@pytest.mark.parametrize("make,u", [(lambda: erdos_renyi(25, 0.15, 7), 6.0),
                                    (lambda: grid2d(6, 5), 9.0),
                                    (lambda: random_tree(30, 4), 4.0)])
def test_dense_oracle_k_n_minus_1(make, u):
    """with k = n-1, P equals a dense Eq. 2-3 build from all-pairs
    shortest paths and an independent (brentq) sigma search, within 1e-8."""
    ip, ix = make()
    n = len(ip) - 1
    A = csr_matrix((np.ones(len(ix)), ix, ip), shape=(n, n))
    Dm = shortest_path(A, unweighted=True)
    Pc = np.zeros((n, n))
    for i in range(n):
        js = np.array([j for j in range(n) if j != i and np.isfinite(Dm[i, j])])
        d2 = Dm[i, js] ** 2
        cmin = int((d2 == d2.min()).sum())
        if len(js) <= u:
            q = np.full(len(js), 1.0 / len(js))
        elif cmin >= u:
            q = (d2 == d2.min()).astype(float) / cmin
        else:
            def f(ls):
                e = np.exp(-(d2 - d2.min()) / (2 * math.exp(2 * ls)))
                qq = e / e.sum()
                qq = qq[qq > 0]
                return -(qq * np.log(qq)).sum() - math.log(u)
            ls = brentq(f, -8.0, 12.0, xtol=1e-15, rtol=1e-15, maxiter=500)
            e = np.exp(-(d2 - d2.min()) / (2 * math.exp(2 * ls)))
            q = e / e.sum()
        Pc[i, js] = q
    dense = (Pc + Pc.T) / (2 * n)
    P = oracle.build_P(ip, ix, u=u, k=n - 1, seed=0)
    got = csr_matrix((P["values"], P["indices"], P["indptr"]), shape=(n, n)).toarray()
    assert np.allclose(got, dense, rtol=1e-8, atol=1e-14)


def test_config1_sparsity_matches_survey():
    # 2-D grid 32x32 at u=40 has nnz/n = 134.0
    from workloads import config_graph
    ip, ix = config_graph(1)
    P = oracle.build_P(ip, ix, 40.0)
    assert P["k"] == 120 and np.all(P["knn_len"] == 120)
    assert abs(len(P["values"]) / 1024 - 134.05) < 0.5
