"""Seeded synthetic graph generators for the hot-path workloads.

This module is shared by the oracle (tests) and the product harness (bench.py,
runner).  It holds NONE of the method's arithmetic (no BFS-kNN, no
perplexity calibration, no gradient): it only builds undirected simple graphs
in CSR form, following the recipes of BASELINE.json `configs` and
SURVEY.md §8(d) "Synthetic inputs".  The paper's own datasets
(appendix table) are not available; these generators stand
in for its three families: meshes -> grids (configs 1, 5),
locally dense / long-diameter graphs -> RGG (2) and SBM (3), scale-free graphs
-> Chung-Lu (4).

Every graph is returned as (indptr int64[n+1], indices int32[nnz]) with
symmetric adjacency, rows sorted ascending, no self-loops, no duplicates.
"""
from __future__ import annotations

import math
import os

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components


# ---------------------------------------------------------------- CSR helpers
def edges_to_csr(n: int, u: np.ndarray, v: np.ndarray):
    """Undirected edge list -> symmetric sorted CSR (dedup, self-loops dropped)."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    keep = u != v
    u, v = u[keep], v[keep]
    rows = np.concatenate([u, v])
    cols = np.concatenate([v, u])
    m = sp.csr_matrix((np.ones(rows.shape[0], dtype=np.int8), (rows, cols)), shape=(n, n))
    m.sum_duplicates()
    m.sort_indices()
    return m.indptr.astype(np.int64), m.indices.astype(np.int32)


def largest_component(indptr: np.ndarray, indices: np.ndarray):
    """Restrict to the largest connected component, relabelling in id order."""
    n = indptr.shape[0] - 1
    a = sp.csr_matrix((np.ones(indices.shape[0], dtype=np.int8), indices, indptr), shape=(n, n))
    ncomp, labels = connected_components(a, directed=False)
    if ncomp == 1:
        return indptr, indices
    big = np.bincount(labels).argmax()
    keep = np.flatnonzero(labels == big)
    sub = a[keep][:, keep]
    sub.sort_indices()
    return sub.indptr.astype(np.int64), sub.indices.astype(np.int32)


def n_edges(indptr) -> int:
    return int(indptr[-1]) // 2


# ------------------------------------------------------------ small fixtures
def path_graph(n):
    i = np.arange(n - 1)
    return edges_to_csr(n, i, i + 1)


def cycle_graph(n):
    i = np.arange(n)
    return edges_to_csr(n, i, (i + 1) % n)


def star_graph(leaves):
    """K_{1,leaves}; vertex 0 is the centre."""
    i = np.arange(1, leaves + 1)
    return edges_to_csr(leaves + 1, np.zeros_like(i), i)


def complete_graph(n):
    u, v = np.triu_indices(n, 1)
    return edges_to_csr(n, u, v)


def random_tree(n, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    parent = np.array([rng.integers(0, i) for i in range(1, n)], dtype=np.int64)
    return edges_to_csr(n, np.arange(1, n), parent)


def erdos_renyi(n, p, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    u, v = np.triu_indices(n, 1)
    keep = rng.random(u.shape[0]) < p
    return edges_to_csr(n, u[keep], v[keep])


# --------------------------------------------------------------- generators
def grid2d(w: int, h: int):
    """4-neighbour grid, id = w*r + c (config 1: 32x32)."""
    ids = np.arange(w * h, dtype=np.int64).reshape(h, w)
    u = np.concatenate([ids[:, :-1].ravel(), ids[:-1, :].ravel()])
    v = np.concatenate([ids[:, 1:].ravel(), ids[1:, :].ravel()])
    return edges_to_csr(w * h, u, v)


def grid3d(a: int, b: int, c: int):
    """6-neighbour grid, id = (z*b + y)*a + x (config 5: 160^3)."""
    ids = np.arange(a * b * c, dtype=np.int64).reshape(c, b, a)
    u = np.concatenate([ids[:, :, :-1].ravel(), ids[:, :-1, :].ravel(), ids[:-1, :, :].ravel()])
    v = np.concatenate([ids[:, :, 1:].ravel(), ids[:, 1:, :].ravel(), ids[1:, :, :].ravel()])
    return edges_to_csr(a * b * c, u, v)


def rgg(n: int, mean_degree: float, seed: int):
    """Random geometric graph in [0,1)^2: edge iff dist < r,
    r = sqrt(mean_degree / (pi (n-1))) (config 2), then LCC."""
    from scipy.spatial import cKDTree

    rng = np.random.Generator(np.random.PCG64(seed))
    pts = rng.random((n, 2))
    r = math.sqrt(mean_degree / (math.pi * (n - 1)))
    pairs = cKDTree(pts).query_pairs(r, output_type="ndarray")
    ip, ix = edges_to_csr(n, pairs[:, 0], pairs[:, 1])
    return largest_component(ip, ix)


def _geometric_positions(rng, total: int, p: float):
    """Exact Bernoulli(p) trial positions in [0,total) by geometric skipping."""
    if p <= 0.0 or total <= 0:
        return np.empty(0, dtype=np.int64)
    if p >= 1.0:
        return np.arange(total, dtype=np.int64)
    out = []
    pos = -1
    expect = int(total * p * 1.1) + 64
    while True:
        gaps = rng.geometric(p, size=expect).astype(np.int64)
        cs = pos + np.cumsum(gaps)
        inside = cs[cs < total]
        out.append(inside)
        if inside.shape[0] < cs.shape[0]:
            break
        pos = int(cs[-1])
    return np.concatenate(out)


def _tri_index(t: np.ndarray):
    """Linear index t over pairs (i<j) ordered by j -> (i, j)."""
    j = np.floor((1.0 + np.sqrt(1.0 + 8.0 * t.astype(np.float64))) / 2.0).astype(np.int64)
    # exact correction of floating rounding
    j = np.where(j * (j - 1) // 2 > t, j - 1, j)
    j = np.where((j + 1) * j // 2 <= t, j + 1, j)
    i = t - j * (j - 1) // 2
    return i, j


def sbm(blocks: int, size: int, deg_in: float, deg_out: float, seed: int):
    """Stochastic block model with contiguous blocks (config 3):
    p_in = deg_in/(size-1), p_out = deg_out/(n-size); exact Bernoulli per block pair."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = blocks * size
    p_in = deg_in / (size - 1)
    p_out = deg_out / (n - size)
    us, vs = [], []
    for b in range(blocks):
        t = _geometric_positions(rng, size * (size - 1) // 2, p_in)
        i, j = _tri_index(t)
        us.append(b * size + i)
        vs.append(b * size + j)
    for a in range(blocks):
        for b in range(a + 1, blocks):
            t = _geometric_positions(rng, size * size, p_out)
            us.append(a * size + t // size)
            vs.append(b * size + t % size)
    ip, ix = edges_to_csr(n, np.concatenate(us), np.concatenate(vs))
    return largest_component(ip, ix)


def chung_lu(n: int, gamma: float, mean_degree: float, seed: int):
    """Chung-Lu graph (config 4): w_i ∝ (i+1)^(-1/(gamma-1)) scaled to mean
    `mean_degree`, p_ij = min(1, w_i w_j / sum w), exact O(n+m) sampling by
    sorted-weight geometric skipping (run for all u at once), then LCC."""
    rng = np.random.Generator(np.random.PCG64(seed))
    w = (np.arange(1, n + 1, dtype=np.float64)) ** (-1.0 / (gamma - 1.0))
    w *= mean_degree * n / w.sum()
    S = w.sum()
    u = np.arange(n - 1, dtype=np.int64)
    v = u + 1
    p = np.minimum(w[u] * w[v] / S, 1.0)
    eu, ev = [], []
    while u.shape[0]:
        live = (v < n) & (p > 0)
        u, v, p = u[live], v[live], p[live]
        if u.shape[0] == 0:
            break
        r = rng.random(u.shape[0])
        notone = p < 1.0
        skip = np.zeros(u.shape[0], dtype=np.int64)
        with np.errstate(divide="ignore"):
            sk = np.floor(np.log(r[notone]) / np.log1p(-p[notone]))
        skip[notone] = np.minimum(sk, n).astype(np.int64)
        v = v + skip
        ok = v < n
        u, v, p = u[ok], v[ok], p[ok]
        q = np.minimum(w[u] * w[v] / S, 1.0)
        r2 = rng.random(u.shape[0])
        acc = r2 < q / p
        eu.append(u[acc])
        ev.append(v[acc])
        p = q
        v = v + 1
    ip, ix = edges_to_csr(n, np.concatenate(eu), np.concatenate(ev))
    return largest_component(ip, ix)


# ------------------------------------------------------------ named configs
CONFIGS = {
    1: dict(name="grid2d_32x32", desc="2-D grid 32x32 (n=1024, m=1984)"),
    2: dict(name="rgg_20k_deg8", desc="RGG n=20,000 mean degree 8, LCC"),
    3: dict(name="sbm_50x4000", desc="SBM 50 blocks x 4,000, intra 10 / inter 1, LCC"),
    4: dict(name="chunglu_1M_g2.5_d6", desc="Chung-Lu n=1,000,000 gamma 2.5 mean degree 6, LCC"),
    5: dict(name="grid3d_160", desc="3-D grid 160^3 (n=4,096,000)"),
}


def _build_config(i: int):
    if i == 1:
        return grid2d(32, 32)
    if i == 2:
        return rgg(20_000, 8.0, seed=0)
    if i == 3:
        return sbm(50, 4000, 10.0, 1.0, seed=0)
    if i == 4:
        return chung_lu(1_000_000, 2.5, 6.0, seed=0)
    if i == 5:
        return grid3d(160, 160, 160)
    raise ValueError(f"unknown config {i}")


def cache_dir() -> str:
    d = os.environ.get("TSNET_CACHE", "/tmp/tsnet_cache")
    os.makedirs(d, exist_ok=True)
    return d


def config_graph(i: int, use_cache: bool = True):
    """Graph of BASELINE.json configs[i-1] as (indptr, indices)."""
    path = os.path.join(cache_dir(), f"graph_cfg{i}.npz")
    if use_cache and os.path.exists(path):
        z = np.load(path)
        return z["indptr"], z["indices"]
    ip, ix = _build_config(i)
    if use_cache:
        np.savez(path, indptr=ip, indices=ix)
    return ip, ix


def random_csr(n: int, row_lengths, seed: int = 0):
    """Seeded random sparse matrix pattern for SpMV edge cases (not a graph of
    the method): row i draws row_lengths[i] columns uniformly from [0, n) with
    replacement, keeps the distinct ones sorted (so a row has at most
    row_lengths[i] entries), values positive fp32-representable in [0.5, 1.5) / n.
    Returns (indptr int64, indices int32, values float64)."""
    rng = np.random.default_rng(seed)
    L = np.asarray(row_lengths, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), L)
    cols = rng.integers(0, n, size=len(rows), dtype=np.int64)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    keep = np.ones(len(rows), bool)
    keep[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
    rows, cols = rows[keep], cols[keep]
    indptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=indptr[1:])
    values = ((rng.random(len(cols)) + 0.5) / n).astype(np.float32).astype(np.float64)
    return indptr, cols.astype(np.int32), values
