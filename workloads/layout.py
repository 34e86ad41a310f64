"""Seeded initial layouts (no method arithmetic).

BASELINE.json configs prescribe "layout init N(0,1e-4^2) seed 0" (SURVEY.md
§8(d), reading R15): drawn in fp64 with numpy PCG64 and rounded once to fp32,
so the GPU path and the oracle start from bit-identical positions.
"""
from __future__ import annotations

import numpy as np


def init_layout(n: int, seed: int = 0, sigma: float = 1e-4) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.standard_normal((n, 2)) * sigma).astype(np.float32)


def uniform_layout(n: int, side: float, seed: int, offset=(0.0, 0.0)) -> np.ndarray:
    """Uniform random points in a side x side square (test layouts)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    y = rng.random((n, 2)) * side + np.asarray(offset)[None, :]
    return y.astype(np.float32)


def clustered_layout(n: int, side: float, clusters: int, spread: float, seed: int) -> np.ndarray:
    """Gaussian blobs in a side x side square: a spatially very non-uniform
    layout (many points per interpolation box) for spread/gather tests."""
    rng = np.random.Generator(np.random.PCG64(seed))
    centres = rng.random((clusters, 2)) * side
    lab = rng.integers(0, clusters, size=n)
    y = centres[lab] + rng.standard_normal((n, 2)) * spread
    return y.astype(np.float32)


def random_state(n: int, seed: int, vel_scale: float = 1e-3):
    """Random optimiser state (velocity, gains) for single-step parity tests."""
    rng = np.random.Generator(np.random.PCG64(seed))
    vel = (rng.standard_normal((n, 2)) * vel_scale).astype(np.float32)
    gains = (0.01 + rng.random((n, 2)) * 3.0).astype(np.float32)
    return vel, gains
