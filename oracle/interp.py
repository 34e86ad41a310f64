"""O5 — FFT-accelerated Lagrange-interpolation gradient (CPU ORACLE, fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain numpy, step by step
in the paper's order:

  * FIt-SNE interpolation (§2.3): "dividing the
    low-dimensional projection area into a constant number of I intervals and
    defining a constant number of P interpolant points inside each interval,
    the kernel K computed between two intervals can be approximated ... using
    the interpolant points ... accelerated using FFT".
  * Alg. 3 l.397-400: compute P interpolation points per
    interval; compute the sums for C_KL by FFT-accelerated interpolation.
  * Alg. 3 l.403-404 and Eq. 8: the entropy sums
    h1, h2, h3 with kernel K_e = 1/(eps + r^2), eps = 1/20.

Readings: R3 (h2, h3 use the summed-over point's coordinates and
Eq. 8 is x_k h1 - h2), R9 (grid policy P=3, h_max, I_min, I_max, 5-smooth I,
square cells, per-axis lo), R10 (one K1 sum for Z, three K2 sums), R11 (Z
subtracts exactly n; repulsion/entropy self terms cancel algebraically).

The oracle implements the PLAIN form (charges {1, x~, y~}); the GPU implements
the local-moment form.  `form="moment"` computes the moment form here too, in
fp64, as a self-check (the two agree to ~1e-13).
"""
from __future__ import annotations

import math

import numpy as np


# ------------------------------------------------------------- grid policy
def _is_5smooth(m: int) -> bool:
    for q in (2, 3, 5):
        while m % q == 0:
            m //= q
    return m == 1


def five_smooth_at_least(m: int) -> int:
    m = max(int(m), 1)
    while not _is_5smooth(m):
        m += 1
    return m


def five_smooth_at_most(m: int) -> int:
    m = max(int(m), 1)
    while not _is_5smooth(m):
        m -= 1
    return m


def geometry(Y, h_max: float = 0.25, I_min: int = 20, I_max: int = 1024, p: int = 3):
    """O5.1 grid geometry (R9): square cells of width h_b = S/I over the
    bounding box, S = max(span_x, span_y) floored at 1e-12, I_max = 1024 by
    default (the paper fixes I as a constant),
    I = clamp(ceil(S/h_max), I_min, I_max) rounded up to 5-smooth (down to the
    largest 5-smooth <= I_max if that exceeds I_max); p nodes per interval at
    in-box positions (t+1/2)/p ("P interpolation points for interval i",
    PAPER.md:397-398)."""
    Y = np.asarray(Y, dtype=np.float64)
    lo_x = float(Y[:, 0].min())
    lo_y = float(Y[:, 1].min())
    S = max(float(Y[:, 0].max()) - lo_x, float(Y[:, 1].max()) - lo_y)
    S = max(S, 1e-12)
    I0 = int(min(max(math.ceil(S / float(h_max)), I_min), I_max))
    I = five_smooth_at_least(I0)
    if I > I_max:
        I = five_smooth_at_most(I_max)
    h_b = S / I
    return dict(lo_x=lo_x, lo_y=lo_y, S=S, I=I, h_b=h_b, delta=h_b / p, N=p * I, p=p)


def lagrange_weights(u, p: int = 3):
    """L_t(u) = prod_{s != t} (u - s_s)/(s_t - s_s), nodes s_t = (t + 1/2)/p."""
    u = np.asarray(u, dtype=np.float64)
    s = (np.arange(p) + 0.5) / p
    L = np.ones(u.shape + (p,), dtype=np.float64)
    for t in range(p):
        for q in range(p):
            if q != t:
                L[..., t] *= (u - s[q]) / (s[t] - s[q])
    return L


def boxes(Y, geo):
    """O5.2 box b = min(floor((x - lo)/h_b), I-1), in-box coordinate u."""
    Y = np.asarray(Y, dtype=np.float64)
    rx = (Y[:, 0] - geo["lo_x"]) / geo["h_b"]
    ry = (Y[:, 1] - geo["lo_y"]) / geo["h_b"]
    bx = np.minimum(np.floor(rx), geo["I"] - 1).astype(np.int64)
    by = np.minimum(np.floor(ry), geo["I"] - 1).astype(np.int64)
    return bx, by, rx - bx, ry - by


def node_coords(geo):
    """t_g = lo + (g + 1/2) delta."""
    g = np.arange(geo["N"], dtype=np.float64)
    return geo["lo_x"] + (g + 0.5) * geo["delta"], geo["lo_y"] + (g + 0.5) * geo["delta"]


class _Interp:
    """Per-point box and tensor-product weights for one layout."""

    def __init__(self, Y, geo):
        p = geo["p"]
        self.geo = geo
        self.bx, self.by, ux, uy = boxes(Y, geo)
        self.Lx = lagrange_weights(ux, p)
        self.Ly = lagrange_weights(uy, p)
        N = geo["N"]
        self.nodes = []   # (flat node index array, weight array) for each (a, b)
        for a in range(p):
            for b in range(p):
                gx = p * self.bx + a
                gy = p * self.by + b
                self.nodes.append((gx * N + gy, self.Lx[:, a] * self.Ly[:, b], a, b))

    def spread(self, charge):
        """O5.4 W[g] = sum_i L_g(X_i) c_i."""
        N = self.geo["N"]
        W = np.zeros(N * N, dtype=np.float64)
        for flat, w, _, _ in self.nodes:
            W += np.bincount(flat, weights=w * charge, minlength=N * N)
        return W.reshape(N, N)

    def gather(self, Phi):
        """O5.6 phi(i) = sum_{a,b} L_a L_b Phi[node]."""
        f = Phi.ravel()
        out = np.zeros(self.bx.shape[0], dtype=np.float64)
        for flat, w, _, _ in self.nodes:
            out += w * f[flat]
        return out


# ------------------------------------------------------------- convolution
def _offset_table(table_fn, N: int, delta: float):
    """T[dx, dy] = table_fn(dx delta, dy delta) for dx, dy in [-(N-1), N-1]."""
    d = np.arange(-(N - 1), N, dtype=np.float64) * delta
    DX, DY = np.meshgrid(d, d, indexing="ij")
    return table_fn(DX, DY)


def convolve(W, table_fn, delta: float, method: str = "auto"):
    """O5.5 Phi[g] = sum_{g'} T(g - g') W[g'] with T(d) = table_fn(d_x delta, d_y delta).
    "direct": the N^2 x N^2 node-to-node matrix applied to W (used when
    N^2 <= 4096); "fft": zero-padded circular convolution on a 2N x 2N grid
    (numpy FFT as a library step, "accelerated using FFT")."""
    N = W.shape[0]
    if method == "auto":
        method = "direct" if N * N <= 4096 else "fft"
    if method == "direct":
        g = np.arange(N)
        GX, GY = np.meshgrid(g, g, indexing="ij")
        gx, gy = GX.ravel(), GY.ravel()
        DX = (gx[:, None] - gx[None, :]).astype(np.float64) * delta
        DY = (gy[:, None] - gy[None, :]).astype(np.float64) * delta
        A = table_fn(DX, DY)
        return (A @ W.ravel()).reshape(N, N)
    T = _offset_table(table_fn, N, delta)            # (2N-1) x (2N-1), index d + N - 1
    M = 2 * N
    Tc = np.zeros((M, M), dtype=np.float64)
    idx = np.arange(-(N - 1), N) % M
    Tc[np.ix_(idx, idx)] = T
    Wp = np.zeros((M, M), dtype=np.float64)
    Wp[:N, :N] = W
    out = np.fft.irfft2(np.fft.rfft2(Tc) * np.fft.rfft2(Wp), s=(M, M))
    return out[:N, :N]


# ------------------------------------------------------------------ kernels
def k1(r2):
    """K = (1 + r^2)^-1 (q_ij numerator)."""
    return 1.0 / (1.0 + r2)


def k2(r2):
    """K = (1 + r^2)^-2."""
    return 1.0 / (1.0 + r2) ** 2


def ke_factory(eps):
    """K_e = 1/(eps + r^2)."""
    return lambda r2: 1.0 / (eps + r2)


def interp_fields(Y, charges, kernel, geo=None, method="auto", h_max=0.25, I_min=20, I_max=1024, p=3):
    """Generic FFT-interpolated field phi_c(i) ~= sum_j K(|X_i - X_j|^2) c_j,
    INCLUDING j = i (SPEC.md:276 evaluate_field), one array per charge."""
    if geo is None:
        geo = geometry(Y, h_max, I_min, I_max, p)
    it = _Interp(Y, geo)
    tab = lambda dx, dy: kernel(dx * dx + dy * dy)  # noqa: E731
    return [it.gather(convolve(it.spread(np.asarray(c, dtype=np.float64)), tab, geo["delta"], method))
            for c in charges], geo


# -------------------------------------------------------------- the gradient
def interp_gradient(Y, indptr, indices, pval, lkl, lc, lr, eps=0.05, h_max=0.25, I_min=20,
                    I_max=1024, p=3, form="plain", method="auto", kernels=None):
    """O5: the L-tsNET gradient at layout Y (Alg. 3 l.396-404).

      Z      = sum_i phi^{K1}_1(i) - n                                 (R10, R11)
      F_rep  = (x~_i phi^{K2}_1 - phi^{K2}_x, y~_i phi^{K2}_1 - phi^{K2}_y) / Z
      g_ent  = -(1/n^2) (x~_i phi^{Ke}_1 - phi^{Ke}_x, ...)             (Eq. 8, R3)
      F_attr = sum_{j in row i} p_ij w_ij (X_i - X_j)                  (Eq. 6 term 1, exact sparse)
      g      = 4 lkl (F_attr - F_rep) + (lc/n) X + lr g_ent            (Eq. 1, 6; C_CMP PAPER.md:89)

    x~ = x - (lo_x + N delta / 2) (grid-centred coordinates).  `kernels` may
    override {"K1", "K2", "Ke"} (test hook).  Returns a dict with g, Z, parts."""
    from . import attr_sparse

    Y = np.asarray(Y, dtype=np.float64)
    n = Y.shape[0]
    geo = geometry(Y, h_max, I_min, I_max, p)
    K = dict(K1=k1, K2=k2, Ke=ke_factory(eps))
    if kernels:
        K.update(kernels)
    it = _Interp(Y, geo)
    delta = geo["delta"]
    tab = lambda kern: (lambda dx, dy: kern(dx * dx + dy * dy))  # noqa: E731

    W1 = it.spread(np.ones(n))
    phiK1 = it.gather(convolve(W1, tab(K["K1"]), delta, method))
    Z = float(phiK1.sum()) - n

    if form == "plain":
        cx = geo["lo_x"] + geo["N"] * delta / 2.0
        cy = geo["lo_y"] + geo["N"] * delta / 2.0
        xt, yt = Y[:, 0] - cx, Y[:, 1] - cy
        Wx, Wy = it.spread(xt), it.spread(yt)

        def pair_sum(kern):
            f1 = it.gather(convolve(W1, tab(kern), delta, method))
            fx = it.gather(convolve(Wx, tab(kern), delta, method))
            fy = it.gather(convolve(Wy, tab(kern), delta, method))
            return np.stack([xt * f1 - fx, yt * f1 - fy], axis=1)
    elif form == "moment":
        tx, ty = node_coords(geo)
        N = geo["N"]
        gx_all = np.repeat(tx[:, None], N, axis=1)
        gy_all = np.repeat(ty[None, :], N, axis=0)
        # M_x[g] = sum_i L_g(X_i) (t_gx - x_i): spread of per-(point,node) charges
        Mx = np.zeros(N * N)
        My = np.zeros(N * N)
        for flat, w, a, b in it.nodes:
            Mx += np.bincount(flat, weights=w * (gx_all.ravel()[flat] - Y[:, 0]), minlength=N * N)
            My += np.bincount(flat, weights=w * (gy_all.ravel()[flat] - Y[:, 1]), minlength=N * N)
        Mx, My = Mx.reshape(N, N), My.reshape(N, N)

        def pair_sum(kern):
            P0 = convolve(W1, tab(kern), delta, method)
            Qx = convolve(W1, lambda dx, dy: dx * kern(dx * dx + dy * dy), delta, method) \
                + convolve(Mx, tab(kern), delta, method)
            Qy = convolve(W1, lambda dx, dy: dy * kern(dx * dx + dy * dy), delta, method) \
                + convolve(My, tab(kern), delta, method)
            f = P0.ravel(), Qx.ravel(), Qy.ravel()
            out = np.zeros((n, 2))
            for flat, w, _, _ in it.nodes:
                out[:, 0] += w * ((Y[:, 0] - gx_all.ravel()[flat]) * f[0][flat] + f[1][flat])
                out[:, 1] += w * ((Y[:, 1] - gy_all.ravel()[flat]) * f[0][flat] + f[2][flat])
            return out
    else:
        raise ValueError(form)

    F_rep = pair_sum(K["K2"]) / Z
    g_ent = -pair_sum(K["Ke"]) / (float(n) * float(n))
    F_attr = attr_sparse(Y, indptr, indices, pval)
    g = 4.0 * lkl * (F_attr - F_rep) + (lc / n) * Y + lr * g_ent
    return dict(g=g, Z=Z, F_attr=F_attr, F_rep=F_rep, g_ent=g_ent, geo=geo)


# ------------------------------------------- the same plain form, in row blocks
# Used only by the bounded-sample CPU timing legs of bench.py: one iteration of
# O5 is split into the layout-wide part (geometry, spread, 7 convolutions, Z)
# and per-row-block parts (gather, sparse attraction, assembly).  Same
# arithmetic as interp_gradient(form="plain"); pinned equal to it by
# tests/test_oracle_interp.py::test_row_blocks_equal_full_gradient.
def field_state(Y, eps=0.05, h_max=0.25, I_min=20, I_max=1024, p=3, method="auto"):
    Y = np.asarray(Y, dtype=np.float64)
    n = Y.shape[0]
    geo = geometry(Y, h_max, I_min, I_max, p)
    it = _Interp(Y, geo)
    delta = geo["delta"]
    tab = lambda kern: (lambda dx, dy: kern(dx * dx + dy * dy))  # noqa: E731
    cx = geo["lo_x"] + geo["N"] * delta / 2.0
    cy = geo["lo_y"] + geo["N"] * delta / 2.0
    W1 = it.spread(np.ones(n))
    Wx, Wy = it.spread(Y[:, 0] - cx), it.spread(Y[:, 1] - cy)
    Phi = {}
    for name, kern in (("K2", k2), ("Ke", ke_factory(eps))):
        Phi[name] = (convolve(W1, tab(kern), delta, method), convolve(Wx, tab(kern), delta, method),
                     convolve(Wy, tab(kern), delta, method))
    Z = float(it.gather(convolve(W1, tab(k1), delta, method)).sum()) - n
    return dict(geo=geo, Phi=Phi, Z=Z, cx=cx, cy=cy, n=n)


def gradient_rows(state, Y, indptr, indices, pval, lkl, lc, lr, row0, nrows):
    """O5 gradient of the rows [row0, row0 + nrows) from a field_state of Y."""
    from . import attr_sparse_rows

    Y = np.asarray(Y, dtype=np.float64)
    n = state["n"]
    Yr = Y[row0:row0 + nrows]
    it = _Interp(Yr, state["geo"])
    xt, yt = Yr[:, 0] - state["cx"], Yr[:, 1] - state["cy"]

    def pair_sum(name):
        f1, fx, fy = (it.gather(F) for F in state["Phi"][name])
        return np.stack([xt * f1 - fx, yt * f1 - fy], axis=1)

    F_rep = pair_sum("K2") / state["Z"]
    g_ent = -pair_sum("Ke") / (float(n) * float(n))
    F_attr = attr_sparse_rows(Y, indptr, indices, pval, row0, nrows)
    return 4.0 * lkl * (F_attr - F_rep) + (lc / n) * Yr + lr * g_ent
