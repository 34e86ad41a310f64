"""O6/O7 — position update and stage schedule (CPU ORACLE, fp64).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper says only "Move each vertex v in the direction of dC/dv"
(Alg. 3 l.405) and that the multipliers lambda_KL, lambda_c,
lambda_r vary "in different stages".  BASELINE.json's north
star asks for the momentum/gains update; reading R12 fixes it:

  gains <- max(gain_min, sign(g) != sign(v) ? gains + gain_inc : gain_dec * gains)   (sign(0) = 0)
  v     <- mu v - eta gains g
  Y     <- Y + v
  (optional, R13) Y <- Y - mean(Y)

and the two-stage schedule O7: iterations 0-249 (lkl, lc, lr) = (1, 1.2, 0),
mu = 0.5; from 250 on (1, 0.01, 0.6), mu = 0.8; eta = 50.
"""
from __future__ import annotations

import numpy as np


def update_step(Y, vel, gains, g, eta=50.0, mu=0.5, gain_inc=0.2, gain_dec=0.8, gain_min=0.01,
                recenter=False):
    """O6, per coordinate.  Returns new (Y, vel, gains) as fp64 arrays."""
    Y = np.asarray(Y, dtype=np.float64)
    vel = np.asarray(vel, dtype=np.float64)
    gains = np.asarray(gains, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    flip = np.sign(g) != np.sign(vel)
    gains = np.where(flip, gains + gain_inc, gains * gain_dec)
    gains = np.maximum(gains, gain_min)
    vel = mu * vel - eta * gains * g
    Y = Y + vel
    if recenter:
        Y = Y - Y.mean(axis=0, keepdims=True)
    return Y, vel, gains


def stage_params(it: int, stage_switch: int = 250):
    """O7 schedule -> (lkl, lc, lr, mu)."""
    if it < stage_switch:
        return 1.0, 1.2, 0.0, 0.5
    return 1.0, 0.01, 0.6, 0.8


def run_layout(Y0, indptr, indices, pval, iters, start_iter=0, vel=None, gains=None, eta=50.0,
               eps=0.05, h_max=0.25, I_min=20, I_max=1024, exact=False, fp32_state=True,
               recenter=False, callback=None):
    """Alg. 3 main loop with the O6/O7 update.

    exact=False uses the interpolation gradient O5, exact=True the exact O4a.
    fp32_state=True rounds (Y, vel, gains) to fp32 after every step, so layouts
    produced here can be handed to the fp32 GPU path bit-identically."""
    from . import exact_grad
    from .interp import interp_gradient

    Y = np.asarray(Y0, dtype=np.float64).copy()
    n = Y.shape[0]
    vel = np.zeros((n, 2)) if vel is None else np.asarray(vel, dtype=np.float64).copy()
    gains = np.ones((n, 2)) if gains is None else np.asarray(gains, dtype=np.float64).copy()
    for it in range(start_iter, start_iter + iters):
        lkl, lc, lr, mu = stage_params(it)
        if exact:
            g, _ = exact_grad(Y, indptr, indices, pval, lkl, lc, lr, eps)
        else:
            g = interp_gradient(Y, indptr, indices, pval, lkl, lc, lr, eps, h_max, I_min, I_max)["g"]
        Y, vel, gains = update_step(Y, vel, gains, g, eta, mu, recenter=recenter)
        if fp32_state:
            Y = Y.astype(np.float32).astype(np.float64)
            vel = vel.astype(np.float32).astype(np.float64)
            gains = gains.astype(np.float32).astype(np.float64)
        if callback is not None:
            callback(it, Y, vel, gains)
    return Y, vel, gains
