"""Pins of the interpolation oracle (O5) against mathematics: polynomial
reproduction (the P=3 Lagrange scheme is exact for kernels of degree <= 2 per
axis), FFT == direct node sums, h-convergence to the exact O(n^2) gradient,
linearity, translation invariance, self-term cancellation, the Z identity,
and the moment form == plain form in fp64."""
import numpy as np
import pytest

import oracle
from oracle import interp
from workloads import clustered_layout, config_graph, grid2d, uniform_layout


def direct_field(Y, c, kern):
    d = Y[:, None, :] - Y[None, :, :]
    r2 = (d ** 2).sum(-1)
    return kern(r2) @ c


@pytest.mark.parametrize("side", [0.7, 5.0, 40.0])
def test_polynomial_reproduction(side):
    """K = 1 and K = r^2 (degree <= 2 per axis) are reproduced exactly by the
    3-point-per-interval Lagrange interpolation."""
    Y = uniform_layout(300, side, 2).astype(np.float64)
    rng = np.random.default_rng(0)
    c = rng.standard_normal(300)
    for kern in (lambda r2: np.ones_like(r2), lambda r2: r2):
        (phi,), _ = interp.interp_fields(Y, [c], kern, h_max=side / 7.0, I_min=1)
        want = direct_field(Y, c, kern)
        assert np.abs(phi - want).max() <= 1e-10 * np.abs(want).max()
    # K = r^4 is NOT reproduced (degree 4): a sanity check that the test can fail
    (phi,), _ = interp.interp_fields(Y, [c], lambda r2: r2 * r2, h_max=side / 7.0, I_min=1)
    want = direct_field(Y, c, lambda r2: r2 * r2)
    assert np.abs(phi - want).max() > 1e-8 * np.abs(want).max()


def test_fft_equals_direct_convolution():
    rng = np.random.default_rng(1)
    for N in (6, 15, 36, 60):
        W = rng.standard_normal((N, N))
        for tab in (lambda dx, dy: 1 / (1 + dx * dx + dy * dy),
                    lambda dx, dy: dx / (0.05 + dx * dx + dy * dy)):
            a = interp.convolve(W, tab, 0.13, "direct")
            b = interp.convolve(W, tab, 0.13, "fft")
            assert np.abs(a - b).max() <= 1e-12 * np.abs(a).max()


def _grad_parts(Y, P, lam, h_max, **kw):
    return oracle.interp_gradient(Y, P["indptr"], P["indices"], P["values"], *lam, h_max=h_max, **kw)


@pytest.fixture(scope="module")
def grid_P():
    ip, ix = grid2d(24, 24)
    return oracle.build_P(ip, ix, 40.0)


def test_h_convergence_to_exact(grid_P):
    """As h -> 0 the interpolation gradient converges to O4a with order ~3
    (error falls ~8x per halving of h at P=3)."""
    n = grid_P["n"]
    Y = uniform_layout(n, 12.0, 5).astype(np.float64)
    lam = (1.0, 0.01, 0.6)
    ge, Ze = oracle.exact_grad(Y, grid_P["indptr"], grid_P["indices"], grid_P["values"], *lam)
    errs = []
    for h in (1.0, 0.5, 0.25, 0.125):
        r = _grad_parts(Y, grid_P, lam, h, I_min=1, I_max=1000)
        errs.append(np.linalg.norm(r["g"] - ge) / np.linalg.norm(ge))
        assert abs(r["Z"] - Ze) / Ze < 5e-2
    for a, b in zip(errs, errs[1:]):
        assert b < a / 4.0, errs
    assert errs[-1] < 1e-3


def test_z_identity_and_plain_equals_moment(grid_P):
    n = grid_P["n"]
    Y = clustered_layout(n, 15.0, 5, 1.0, 8).astype(np.float64)
    lam = (1.0, 0.01, 0.6)
    rp = _grad_parts(Y, grid_P, lam, 0.25, form="plain")
    rm = _grad_parts(Y, grid_P, lam, 0.25, form="moment")
    assert np.linalg.norm(rp["g"] - rm["g"]) <= 1e-11 * np.linalg.norm(rp["g"])
    # Z = <W1, K1 * W1> - n  (Parseval form used by the GPU) == sum_i phi(i) - n
    geo = rp["geo"]
    it = interp._Interp(Y, geo)
    W1 = it.spread(np.ones(n))
    Phi = interp.convolve(W1, lambda dx, dy: 1 / (1 + dx * dx + dy * dy), geo["delta"])
    assert abs((W1 * Phi).sum() - n - rp["Z"]) <= 1e-12 * rp["Z"]


def test_linearity_and_self_term():
    Y = uniform_layout(500, 9.0, 3).astype(np.float64)
    rng = np.random.default_rng(2)
    c1, c2 = rng.standard_normal(500), rng.standard_normal(500)
    kern = interp.k2
    (a, b, ab), _ = interp.interp_fields(Y, [c1, c2, 2.0 * c1 - 3.0 * c2], kern)
    assert np.abs(ab - (2 * a - 3 * b)).max() <= 1e-12 * np.abs(ab).max()
    # a single point feels no repulsion / entropy from itself (R11)
    Y1 = np.array([[0.3, -1.2]])
    P1 = dict(indptr=np.array([0, 0], np.int64), indices=np.zeros(0, np.int32), values=np.zeros(0))
    r = oracle.interp_gradient(Y1, P1["indptr"], P1["indices"], P1["values"], 0.0, 0.0, 1.0)
    assert np.abs(r["g"]).max() < 1e-12


def test_translation_invariance(grid_P):
    n = grid_P["n"]
    Y = uniform_layout(n, 10.0, 4).astype(np.float64)
    lam = (1.0, 0.0, 0.6)
    r1 = _grad_parts(Y, grid_P, lam, 0.25)
    r2 = _grad_parts(Y + np.array([64.0, -32.0]), grid_P, lam, 0.25)
    assert np.linalg.norm(r1["g"] - r2["g"]) <= 1e-9 * np.linalg.norm(r1["g"])


def test_interp_vs_exact_on_config1_layouts():
    """At h_max = 0.25 the interpolated gradient is within 2e-2 relL2 of the
    exact gradient (north star bar) on spread-out and clustered layouts."""
    ip, ix = config_graph(1)
    P = oracle.build_P(ip, ix, 40.0)
    lam = (1.0, 0.01, 0.6)
    for Y in (uniform_layout(1024, 25.0, 1), clustered_layout(1024, 25.0, 6, 1.5, 2)):
        Y = Y.astype(np.float64)
        r = _grad_parts(Y, P, lam, 0.25)
        ge, _ = oracle.exact_grad(Y, P["indptr"], P["indices"], P["values"], *lam)
        assert np.linalg.norm(r["g"] - ge) / np.linalg.norm(ge) < 2e-2


def test_row_blocks_equal_full_gradient(grid_P):
    """The block split used by the CPU timing legs is the same computation."""
    n = grid_P["n"]
    Y = clustered_layout(n, 15.0, 5, 1.0, 3).astype(np.float64)
    lam = (1.0, 0.01, 0.6)
    full = _grad_parts(Y, grid_P, lam, 0.25)["g"]
    st = interp.field_state(Y)
    parts = [interp.gradient_rows(st, Y, grid_P["indptr"], grid_P["indices"], grid_P["values"], *lam, r0,
                                  min(100, n - r0)) for r0 in range(0, n, 100)]
    assert np.abs(np.concatenate(parts) - full).max() <= 1e-13 * np.abs(full).max()


def test_geometry_policy():
    g = interp.geometry(np.array([[0.0, 0.0], [1.0, 0.5]]))
    assert g["I"] == 20 and g["N"] == 60                 # I_min clamp, span < 5
    g = interp.geometry(np.array([[0.0, 0.0], [30.0, 1.0]]))
    assert g["I"] == 120 and abs(g["h_b"] - 0.25) < 1e-15
    g = interp.geometry(np.array([[0.0, 0.0], [33.1, 1.0]]))
    assert g["I"] == 135                                  # ceil(132.4)=133 -> 5-smooth 135
    g = interp.geometry(np.array([[0.0, 0.0], [1000.0, 1.0]]))
    assert g["I"] == 1024                                 # I_max clamp (R9: 1024)
    g = interp.geometry(np.array([[0.0, 0.0], [1000.0, 1.0]]), I_max=250)
    assert g["I"] == 250                                  # a 5-smooth I_max is kept
    g = interp.geometry(np.array([[0.0, 0.0], [1000.0, 1.0]]), I_max=257)
    assert g["I"] == 256                                  # else the largest 5-smooth below it
    assert interp.five_smooth_at_least(97) == 100 and interp.five_smooth_at_most(97) == 96
