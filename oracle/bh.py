"""O9 quadtree (Barnes-Hut) gradient of BH-tsNET / FIt-tsNET -- TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).  NEXT-3.

BH-tsNET (Alg. 2): a quadtree on the drawing; for
each point a depth-first search from the root, where a node that "can be used
as a summary" stands for all its points at their centre of mass (PAPER.md:
172-173, BH-SNE); the repulsion term of Eq. 6 (with Z summed the same way) and
the entropy gradient of Eq. 7 (read as |N| (X_i - X_N) /
(eps + |X_i - X_N|^2), R2/R3) are accumulated over the summaries.  FIt-tsNET
 keeps the interpolated repulsion and takes only the
entropy from the quadtree.

Readings (R23-R24; the paper fixes no tree parameters):
  tree     the square root cell [lo_x, lo_x + S] x [lo_y, lo_y + S] of the
           bounding box (S = the larger span, as the interpolation grid, R9);
           a point's cell at depth 16 is ix = floor((x - lo_x) / S * 2^16)
           clamped to [0, 2^16 - 1] (fp64), same for y; Morton code = bits of
           ix in the even, of iy in the odd positions; a node at level l is a
           maximal run of Morton-sorted points (stable by index) sharing the
           top 2l bits; its side is S / 2^l, its centre of mass the mean of
           its points (from fp64 prefix sums of the sorted coordinates);
  summary  a node with more than one point is a summary for X_i when
           side^2 < theta^2 |X_i - com|^2 (fp64); theta = 0.5 by default;
           a one-point node is the exact pair (skipped when it is i); a
           level-16 node that is not a summary is taken point by point;
  sums     Z = sum_i sum_N |N| w(X_i, com_N); R_i = sum_N |N| w^2 (X_i - com);
           E_i = sum_N |N| (X_i - com) / (eps + |X_i - com|^2);
           g_i = 4 lkl (F_attr,i - R_i / Z) + (lc / n) X_i - (lr / n^2) E_i,
           the exact gradient's form (O4a) with the pair sums replaced.

Plain fp64 Python (small n); theta = 0 reduces it to the exact gradient.
"""
from __future__ import annotations

import numpy as np

DEPTH = 16


def morton_order(X: np.ndarray):
    """(codes sorted, permutation, lo_x, lo_y, S) of the points X (n x 2)."""
    Xf = np.asarray(X, np.float64)
    lo = Xf.min(axis=0)
    S = float(max(Xf[:, 0].max() - lo[0], Xf[:, 1].max() - lo[1]))
    if not S > 0.0:
        S = 1.0
    cells = np.floor((Xf - lo) / S * 2.0 ** DEPTH)
    cells = np.clip(cells, 0, 2 ** DEPTH - 1).astype(np.int64)
    code = np.zeros(len(Xf), np.int64)
    for b in range(DEPTH):
        code |= ((cells[:, 0] >> b) & 1) << (2 * b)
        code |= ((cells[:, 1] >> b) & 1) << (2 * b + 1)
    perm = np.argsort(code, kind="stable")
    return code[perm], perm, float(lo[0]), float(lo[1]), S


class Quadtree:
    """Levels 0..DEPTH of runs of the Morton-sorted points."""

    def __init__(self, X: np.ndarray):
        self.X = np.asarray(X, np.float64)
        self.code, self.perm, self.lo_x, self.lo_y, self.S = morton_order(self.X)
        n = len(self.X)
        Xs = self.X[self.perm]
        self.Px = np.concatenate([[0.0], np.cumsum(Xs[:, 0])])
        self.Py = np.concatenate([[0.0], np.cumsum(Xs[:, 1])])
        self.starts = []
        for lev in range(DEPTH + 1):
            pre = self.code >> (2 * (DEPTH - lev))
            s = np.flatnonzero(np.concatenate([[True], pre[1:] != pre[:-1]])) if n else np.zeros(0, np.int64)
            self.starts.append(np.append(s, n))

    def children(self, lev: int, k: int):
        """Child nodes (lev + 1, j) of node (lev, k)."""
        s, e = self.starts[lev][k], self.starts[lev][k + 1]
        nxt = self.starts[lev + 1]
        j0 = int(np.searchsorted(nxt, s))
        j1 = int(np.searchsorted(nxt, e))
        return [(lev + 1, j) for j in range(j0, j1)]

    def sums(self, i: int, theta: float, eps: float):
        """(Zpart, R_i, E_i) for point i by depth-first search from the root."""
        xi = self.X[i]
        z = 0.0
        R = np.zeros(2)
        E = np.zeros(2)
        stack = [(0, 0)] if len(self.X) else []

        def pair(xj, cnt):
            nonlocal z
            d = xi - xj
            r2 = float(d @ d)
            w = 1.0 / (1.0 + r2)
            z += cnt * w
            R[:] += cnt * w * w * d
            E[:] += cnt * d / (eps + r2)

        while stack:
            lev, k = stack.pop()
            s, e = int(self.starts[lev][k]), int(self.starts[lev][k + 1])
            cnt = e - s
            if cnt == 1:
                j = int(self.perm[s])
                if j != i:
                    pair(self.X[j], 1)
                continue
            com = np.array([(self.Px[e] - self.Px[s]) / cnt, (self.Py[e] - self.Py[s]) / cnt])
            d = xi - com
            side = self.S / 2.0 ** lev
            if side * side < theta * theta * float(d @ d):
                pair(com, cnt)
            elif lev == DEPTH:
                for t in range(s, e):
                    j = int(self.perm[t])
                    if j != i:
                        pair(self.X[j], 1)
            else:
                stack.extend(reversed(self.children(lev, k)))
        return z, R, E


def bh_gradient(X, indptr, indices, pval, lkl, lc, lr, eps=0.05, theta=0.5, repulsion=True):
    """BH-tsNET gradient (repulsion=True) or its entropy part alone for
    FIt-tsNET (repulsion=False: returns -(lr/n^2) E, to be added to the
    interpolated gradient computed with lr = 0).  Returns dict(g, Z, R, E)."""
    from . import attr_sparse
    X = np.asarray(X, np.float64)
    n = len(X)
    T = Quadtree(X)
    Z = 0.0
    R = np.zeros((n, 2))
    E = np.zeros((n, 2))
    for i in range(n):
        zi, R[i], E[i] = T.sums(i, theta, eps)
        Z += zi
    if not repulsion:
        return {"g": -(lr / (n * n)) * E, "Z": Z, "R": R, "E": E}
    Fa = attr_sparse(X, indptr, indices, pval)
    g = 4.0 * lkl * (Fa - R / Z) + (lc / n) * X - (lr / (n * n)) * E
    return {"g": g, "Z": Z, "R": R, "E": E}
