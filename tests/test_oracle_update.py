"""Pins of the update oracle (O6/O7): SPEC.md step examples and hand-built gains patterns."""
import numpy as np

import oracle
from oracle.update import stage_params, update_step


def test_spec_step_examples():
    Y = np.array([[1.0, 2.0], [-3.0, 0.5]])
    z = np.zeros_like(Y)
    one = np.ones_like(Y)
    # SPEC.md:440 zero gradient, zero velocity -> unchanged
    Yn, v, _ = update_step(Y, z, one, z, eta=50, mu=0.5)
    assert np.array_equal(Yn, Y) and np.array_equal(v, z)
    # SPEC.md:441 zero momentum, gradient g -> dX = -eta * gains * g (gains -> 1.2 at it 0)
    g = np.array([[0.1, -0.2], [0.0, 0.3]])
    Yn, v, gn = update_step(Y, z, one, g, eta=50, mu=0.0)
    assert np.allclose(Yn - Y, -50 * gn * g)
    assert np.allclose(gn, np.where(g != 0, 1.2, 0.8))   # at iteration 0 every gain with g != 0 -> 1.2
    # SPEC.md:442 velocity v, zero gradient -> dX = momentum * v
    v0 = np.array([[0.5, -1.0], [2.0, 0.0]])
    Yn, v, _ = update_step(Y, v0, one, z, eta=50, mu=0.8)
    assert np.allclose(Yn - Y, 0.8 * v0)


def test_gains_rule_sign_patterns():
    v = np.array([[1.0, -1.0, 1.0, 0.0, -2.0]])
    g = np.array([[1.0, 1.0, -1.0, 0.0, -0.5]])
    gains = np.array([[1.0, 1.0, 1.0, 1.0, 0.011]])
    _, _, gn = update_step(np.zeros_like(v), v, gains, g, eta=1, mu=0.5)
    # same sign -> *0.8; different sign -> +0.2; sign(0)=sign(0) -> *0.8; floor at 0.01
    assert np.allclose(gn, [[0.8, 1.2, 1.2, 0.8, 0.01]])


def test_recenter_and_schedule():
    Y = np.array([[1.0, 1.0], [3.0, -1.0]])
    Yn, _, _ = update_step(Y, np.zeros_like(Y), np.ones_like(Y), np.zeros_like(Y), recenter=True)
    assert np.allclose(Yn.mean(0), 0)
    assert stage_params(0) == (1.0, 1.2, 0.0, 0.5) and stage_params(249) == (1.0, 1.2, 0.0, 0.5)
    assert stage_params(250) == (1.0, 0.01, 0.6, 0.8)


def test_run_layout_decreases_exact_cost():
    """SPEC.md:431-style sanity: descending the exact gradient lowers the exact cost
    (small step, no momentum effects to speak of over a few iterations)."""
    from workloads import grid2d, init_layout
    ip, ix = grid2d(6, 6)
    P = oracle.build_P(ip, ix, 5.0)
    Y0 = np.random.default_rng(0).standard_normal((36, 2))
    lam = (1.0, 0.01, 0.6)
    c0 = oracle.exact_cost(Y0, P["indptr"], P["indices"], P["values"], *lam).sum()
    g, _ = oracle.exact_grad(Y0, P["indptr"], P["indices"], P["values"], *lam)
    Y1 = Y0 - 0.5 * g
    c1 = oracle.exact_cost(Y1, P["indptr"], P["indices"], P["values"], *lam).sum()
    assert c1 < c0
