"""O10 drawing-quality metrics of §4.3 -- TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).  NEXT-4.

Neighbourhood preservation: NP = mean over v of
|N_G(v, r) ∩ N_D(v, r)| / |N_G(v, r) ∪ N_D(v, r)|, N_G(v, r) = vertices within
r hops of v (v excluded), N_D(v, r) = the |N_G(v, r)| vertices closest to v in
the drawing; r = 2.  The printed formula is a sum; the text
calls NP a value in [0, 1], so the mean is used (R25).  Layout distances are
compared as fp64 squared distances of the fp32 coordinates, ties broken by
the smaller vertex id; a vertex with no other vertex within r hops scores 1
(two empty sets, R25).

Stress, the aggregated stress with the optimal layout scale
(SPEC.md stress; R26): with r_ij = |X_i - X_j| / d(i, j) over ordered pairs
i != j of a connected graph, s* = sum r / sum r^2 and
ST = 1/(n(n-1)) sum (1 - s* r_ij)^2.

Plain fp64 numpy, brute force (all pairs, full sorts).
"""
from __future__ import annotations

import numpy as np
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import shortest_path


def hops_all(indptr, indices) -> np.ndarray:
    n = len(indptr) - 1
    A = csr_matrix((np.ones(len(indices)), np.asarray(indices), np.asarray(indptr)), shape=(n, n))
    return shortest_path(A, unweighted=True)


def sqdist(Y: np.ndarray) -> np.ndarray:
    """fp64 squared distances of the fp32 coordinates: dx*dx + dy*dy (no fused ops)."""
    X = np.asarray(Y, np.float32).astype(np.float64)
    dx = X[:, 0][:, None] - X[:, 0][None, :]
    dy = X[:, 1][:, None] - X[:, 1][None, :]
    return dx * dx + dy * dy


def neighborhood_preservation(indptr, indices, Y, r: int = 2, D=None) -> float:
    n = len(indptr) - 1
    D = hops_all(indptr, indices) if D is None else D
    S = sqdist(Y)
    tot = 0.0
    for v in range(n):
        NG = set(np.flatnonzero((D[v] <= r) & (np.arange(n) != v)).tolist())
        k = len(NG)
        if k == 0:
            tot += 1.0
            continue
        others = [w for w in range(n) if w != v]
        order = sorted(others, key=lambda w: (S[v, w], w))
        ND = set(order[:k])
        tot += len(NG & ND) / len(NG | ND)
    return tot / n


def stress(indptr, indices, Y, D=None) -> float:
    n = len(indptr) - 1
    D = hops_all(indptr, indices) if D is None else D
    assert np.all(np.isfinite(D)), "stress needs a connected graph"
    X = np.asarray(Y, np.float32).astype(np.float64)
    off = ~np.eye(n, dtype=bool)
    dist = np.sqrt(sqdist(X))[off]
    d = D[off]
    rr = dist / d
    s = rr.sum() / (rr * rr).sum()
    return float(((1.0 - s * rr) ** 2).sum() / (n * (n - 1)))
