"""O8 Pivot MDS initial layout -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Alg. 3 line 2 "Compute initial layout D of G using Pivot MDS";
tsNET* = tsNET with a PMDS initialisation.  The paper
cites PMDS (Brandes & Pich) without parameters; the readings used here (and by
the GPU) are DESIGN.md R20-R22, following SPEC.md's pivot_mds module:

  select_pivots  max-min (farthest-first) selection: the first pivot is
                 splitmix64(seed) mod n; each next pivot maximises the hop
                 distance to the chosen set, ties -> smallest id (R20);
                 unreachable vertices count as distance n (R21).
  embed          D2[i, k] = hop(i, pivot_k)^2 (n x p); double centring
                 C = -1/2 (D2 - row means - column means + grand mean);
                 top-2 right singular directions of C = top-2 eigenvectors of
                 G = C^T C by power iteration (start vectors from splitmix64,
                 <= 1000 iterations, stop when |v_new - v| < 1e-10; the second
                 on G deflated by the first and re-orthogonalised), each
                 flipped so that its largest-magnitude entry is positive;
                 Y = C [v1 v2] (rows have zero mean by construction).  If the
                 second eigenvalue is <= 1e-12 of the first (rank < 2) the
                 second coordinate is 0 (R22).

Plain fp64 numpy; the BFS is a plain queue BFS in Python (small graphs) --
no blocking or reordering beyond the definitions above.
"""
from __future__ import annotations

from collections import deque

import numpy as np

from . import splitmix64

POWER_ITERS = 1000
POWER_TOL = 1e-10
RANK_TOL = 1e-12


def hop_distances(indptr, indices, src: int) -> np.ndarray:
    """BFS hop distance from src to every vertex; unreachable -> n (R21)."""
    n = len(indptr) - 1
    d = np.full(n, -1, np.int64)
    d[src] = 0
    q = deque([src])
    while q:
        v = q.popleft()
        for w in indices[indptr[v]:indptr[v + 1]]:
            if d[w] < 0:
                d[w] = d[v] + 1
                q.append(w)
    d[d < 0] = n
    return d


def first_pivot(n: int, seed: int) -> int:
    return int(splitmix64(seed & 0xFFFFFFFFFFFFFFFF) % n)


def select_pivots(indptr, indices, p: int, seed: int = 0, first: int | None = None):
    """(pivots list, hop matrix n x p as int64): farthest-first selection (R20);
    `first` overrides the seeded first pivot (tests of SPEC's examples)."""
    n = len(indptr) - 1
    assert 1 <= p <= n
    piv = [first_pivot(n, seed) if first is None else int(first)]
    cols = [hop_distances(indptr, indices, piv[0])]
    dmin = cols[0].copy()
    while len(piv) < p:
        best = int(np.max(dmin))
        nxt = int(np.flatnonzero(dmin == best)[0])       # ties -> smallest id
        piv.append(nxt)
        cols.append(hop_distances(indptr, indices, nxt))
        dmin = np.minimum(dmin, cols[-1])
    return piv, np.stack(cols, axis=1)


def start_vector(p: int, seed: int, which: int) -> np.ndarray:
    """Deterministic start vector of the power iteration: entry k is
    u(splitmix64(seed ^ (2k + which))) - 1/2, u(x) = (x >> 11) 2^-53."""
    return np.array([(splitmix64((seed ^ (2 * k + which)) & 0xFFFFFFFFFFFFFFFF) >> 11) * 2.0 ** -53 - 0.5
                     for k in range(p)], dtype=np.float64)


def power_top(G: np.ndarray, v0: np.ndarray, ortho=None):
    """Largest eigenpair of the symmetric PSD G by power iteration from v0
    (re-orthogonalised against `ortho` every step when given)."""
    v = v0.copy()
    if ortho is not None:
        v -= (v @ ortho) * ortho
    v /= np.linalg.norm(v)
    lam = 0.0
    for _ in range(POWER_ITERS):
        w = G @ v
        if ortho is not None:
            w -= (w @ ortho) * ortho
        lam = float(np.linalg.norm(w))
        if lam == 0.0:
            return 0.0, v
        w /= lam
        done = np.linalg.norm(w - v) < POWER_TOL
        v = w
        if done:
            break
    return lam, v


def orient(v: np.ndarray) -> np.ndarray:
    """Flip so that the largest-magnitude entry (first on ties) is positive."""
    k = int(np.argmax(np.abs(v)))
    return -v if v[k] < 0 else v


def centred(hops: np.ndarray) -> np.ndarray:
    """C = -1/2 (D2 - row means - column means + grand mean), D2 = hops^2."""
    D2 = hops.astype(np.float64) ** 2
    return -0.5 * (D2 - D2.mean(axis=1, keepdims=True) - D2.mean(axis=0, keepdims=True) + D2.mean())


def embed(hops: np.ndarray, seed: int = 0):
    """Layout n x 2 (fp64) from the n x p hop matrix; also returns (l1, l2, V)."""
    C = centred(hops)
    G = C.T @ C
    p = G.shape[0]
    l1, v1 = power_top(G, start_vector(p, seed, 1))
    v1 = orient(v1)
    if p < 2:                                         # one pivot: rank 1 (R22)
        l2, v2 = 0.0, np.zeros(p)
    else:
        G2 = G - l1 * np.outer(v1, v1)
        l2, v2 = power_top(G2, start_vector(p, seed, 2), ortho=v1)
    if l2 <= RANK_TOL * l1:
        v2 = np.zeros(p)
    else:
        v2 = orient(v2)
    V = np.stack([v1, v2], axis=1)
    return C @ V, (l1, l2, V)


def pmds(indptr, indices, p: int, seed: int = 0):
    """Pivot MDS layout: dict(pivots, hops, Y (n x 2 fp64), l1, l2, V)."""
    indptr = np.asarray(indptr, np.int64)
    indices = np.asarray(indices, np.int64)
    piv, hops = select_pivots(indptr, indices, p, seed)
    Y, (l1, l2, V) = embed(hops, seed)
    return {"pivots": piv, "hops": hops, "Y": Y, "l1": l1, "l2": l2, "V": V}
