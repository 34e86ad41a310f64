"""CPU ORACLE for the L-tsNET gradient hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import, call, link or execute anything under
`oracle/`.  The product path (paper_2509_19785_b200) never imports it and
shares no code with it: no kernels, headers, helpers, tables or constants.

Plain, slow, obviously-correct fp64 implementation written from the paper
(PAPER.md = arXiv 2509.19785).  Every function cites the passage it follows;
readings of garbled/ambiguous passages are listed in DESIGN.md ("Readings").

Layout of the oracle:
  c0.c     O1-O3  partial-BFS kNN, perplexity calibration, symmetrisation (C, fp64)
  exact.c  O4a/b  exact O(n^2) gradient and cost; exact sparse attraction (C, fp64)
  interp.py O5    FFT-accelerated Lagrange-interpolation gradient (numpy, fp64)
  update.py O6/O7 momentum/gains update and stage schedule (numpy, fp64)
  pmds.py  O8    Pivot MDS initial layout (numpy, fp64; NEXT-2)
  bh.py    O9    quadtree (Barnes-Hut) repulsion/entropy of BH-/FIt-tsNET (fp64; NEXT-3)
  quality.py O10  neighbourhood preservation and stress of a drawing (fp64; NEXT-4)

Parity status of each function is listed in DESIGN.md §"Oracle pins"; every
function here is pinned by a `-m "not gpu"` test in tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "c0.c"), os.path.join(_HERE, "exact.c")]


def build(force: bool = False) -> str:
    """Compile the C part of the oracle (gcc, fp64, no fast-math)."""
    newest = max(os.path.getmtime(s) for s in _SRC)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", tmp, *_SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64, f64, u64 = ctypes.c_int64, ctypes.c_double, ctypes.c_uint64
        _lib.oracle_splitmix64.restype = u64
        _lib.oracle_splitmix64.argtypes = [u64]
        _lib.oracle_tie_key.restype = u64
        _lib.oracle_tie_key.argtypes = [u64, i64, i64]
        _lib.oracle_knn.restype = None
        _lib.oracle_knn.argtypes = [i64, P, P, i64, u64, i64, P, P, P, P]
        _lib.oracle_calibrate_row.restype = f64
        _lib.oracle_calibrate_row.argtypes = [P, i64, f64, P]
        _lib.oracle_calibrate.restype = None
        _lib.oracle_calibrate.argtypes = [i64, i64, P, P, f64, P, P]
        _lib.oracle_symmetrize.restype = i64
        _lib.oracle_symmetrize.argtypes = [i64, i64, P, P, P, P, P, P]
        _lib.oracle_attr_sparse.restype = None
        _lib.oracle_attr_sparse.argtypes = [i64, P, P, P, P, P]
        _lib.oracle_attr_sparse_rows.restype = None
        _lib.oracle_attr_sparse_rows.argtypes = [i64, i64, P, P, P, P, P]
        _lib.oracle_exact_Z.restype = f64
        _lib.oracle_exact_Z.argtypes = [i64, P]
        _lib.oracle_exact_grad.restype = f64
        _lib.oracle_exact_grad.argtypes = [i64, P, P, P, P, f64, f64, f64, f64, P]
        _lib.oracle_exact_cost.restype = None
        _lib.oracle_exact_cost.argtypes = [i64, P, P, P, P, f64, f64, f64, f64, P]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ------------------------------------------------------------------------ C0
def resolve_k(n: int, u: float, k: int = 0) -> int:
    """k = 3u (Alg. 3 l.3; §3.1 l.272), rounded half up, capped at
    n-1 (reading R5).  An explicit k > 0 overrides 3u but is still capped."""
    if k <= 0:
        k = int(np.floor(3.0 * u + 0.5))
    return int(max(0, min(k, n - 1)))


def splitmix64(x: int) -> int:
    return int(lib().oracle_splitmix64(x & 0xFFFFFFFFFFFFFFFF))


def tie_key(seed: int, v: int, w: int) -> int:
    """key(v,w) = SplitMix64(seed ^ (v<<32 | w)) (reading R4 of PAPER.md:270)."""
    return int(lib().oracle_tie_key(seed & 0xFFFFFFFFFFFFFFFF, v, w))


def knn(indptr, indices, k: int, seed: int = 0, src=None):
    """O1 partial BFS kNN.  Returns (idx[r,k],
    hop[r,k], len[r]) for rows r = src (default all vertices); entries past
    len are -1."""
    ip = _c(indptr, np.int64)
    ix = _c(indices, np.int32)
    n = ip.shape[0] - 1
    if src is None:
        nsrc, sp = n, None
    else:
        s = _c(src, np.int64)
        nsrc, sp = s.shape[0], s
    idx = np.full((nsrc, max(k, 1)), -1, dtype=np.int32)
    hop = np.full((nsrc, max(k, 1)), -1, dtype=np.int32)
    ln = np.zeros(nsrc, dtype=np.int32)
    lib().oracle_knn(n, _p(ip), _p(ix), k, seed & 0xFFFFFFFFFFFFFFFF, nsrc,
                     _p(sp) if sp is not None else None, _p(idx), _p(hop), _p(ln))
    return idx[:, :k], hop[:, :k], ln


def calibrate_row(hops, u: float):
    """O2 for one row (Eq. 3).  Returns (p, beta)."""
    h = _c(hops, np.int32)
    p = np.zeros(max(h.shape[0], 1), dtype=np.float64)
    beta = lib().oracle_calibrate_row(_p(h), h.shape[0], float(u), _p(p))
    return p[: h.shape[0]], beta


def calibrate(hop, ln, u: float):
    """O2 for all rows.  Returns (p_cond[r,k] fp64, beta[r])."""
    hop = _c(hop, np.int32)
    ln = _c(ln, np.int32)
    r, k = hop.shape
    p = np.zeros((r, k), dtype=np.float64)
    beta = np.zeros(r, dtype=np.float64)
    lib().oracle_calibrate(r, k, _p(hop), _p(ln), float(u), _p(p), _p(beta))
    return p, beta


def symmetrize(n: int, idx, ln, p_cond):
    """O3 (Eq. 2).  Returns CSR (indptr, indices, values fp64)."""
    idx = _c(idx, np.int32)
    ln = _c(ln, np.int32)
    p_cond = _c(p_cond, np.float64)
    k = idx.shape[1]
    cap = max(2 * int(ln.sum()), 1)
    ip = np.zeros(n + 1, dtype=np.int64)
    ix = np.zeros(cap, dtype=np.int32)
    val = np.zeros(cap, dtype=np.float64)
    nnz = lib().oracle_symmetrize(n, k, _p(idx), _p(ln), _p(p_cond), _p(ip), _p(ix), _p(val))
    return ip, ix[:nnz].copy(), val[:nnz].copy()


def build_P(indptr, indices, u: float = 40.0, k: int = 0, seed: int = 0):
    """C0 end to end (Alg. 3 l.385-394)."""
    n = int(np.asarray(indptr).shape[0] - 1)
    k = resolve_k(n, u, k)
    idx, hop, ln = knn(indptr, indices, k, seed)
    p_cond, beta = calibrate(hop, ln, u)
    ip, ix, val = symmetrize(n, idx, ln, p_cond)
    return dict(n=n, k=k, knn_idx=idx, knn_hop=hop, knn_len=ln, p_cond=p_cond, beta=beta,
                indptr=ip, indices=ix, values=val)


# ------------------------------------------------------------------- exact
def attr_sparse(X, indptr, indices, pval):
    """sum_{j in row i} p_ij w_ij (X_i - X_j) (Eq. 6 term 1)."""
    X = _c(X, np.float64)
    ip, ix, pv = _c(indptr, np.int64), _c(indices, np.int32), _c(pval, np.float64)
    F = np.zeros_like(X)
    lib().oracle_attr_sparse(X.shape[0], _p(X), _p(ip), _p(ix), _p(pv), _p(F))
    return F


def attr_sparse_rows(X, indptr, indices, pval, row0: int, nrows: int):
    """attr_sparse for the rows [row0, row0 + nrows) only."""
    X = _c(X, np.float64)
    ip, ix, pv = _c(indptr, np.int64), _c(indices, np.int32), _c(pval, np.float64)
    F = np.zeros((nrows, 2))
    lib().oracle_attr_sparse_rows(row0, nrows, _p(X), _p(ip), _p(ix), _p(pv), _p(F))
    return F


def exact_Z(X):
    X = _c(X, np.float64)
    return lib().oracle_exact_Z(X.shape[0], _p(X))


def exact_grad(X, indptr, indices, pval, lkl, lc, lr, eps=0.05):
    """O4a exact gradient (Eq. 1, 6, 8).  Returns (g, Z)."""
    X = _c(X, np.float64)
    ip, ix, pv = _c(indptr, np.int64), _c(indices, np.int32), _c(pval, np.float64)
    g = np.zeros_like(X)
    Z = lib().oracle_exact_grad(X.shape[0], _p(X), _p(ip), _p(ix), _p(pv), lkl, lc, lr, eps, _p(g))
    return g, Z


def exact_cost(X, indptr, indices, pval, lkl, lc, lr, eps=0.05):
    """O4b exact cost -> array [C_KL, C_CMP, C_ENT*]."""
    X = _c(X, np.float64)
    ip, ix, pv = _c(indptr, np.int64), _c(indices, np.int32), _c(pval, np.float64)
    out = np.zeros(3, dtype=np.float64)
    lib().oracle_exact_cost(X.shape[0], _p(X), _p(ip), _p(ix), _p(pv), lkl, lc, lr, eps, _p(out))
    return out


from .interp import geometry, lagrange_weights, interp_gradient, interp_fields  # noqa: E402
from .update import update_step, stage_params, run_layout  # noqa: E402
from . import pmds  # noqa: E402,F401
from . import bh  # noqa: E402,F401
from . import quality  # noqa: E402,F401
