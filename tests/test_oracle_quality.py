"""Pins of the quality-metric oracle O10 (oracle/quality.py) against values
fixed by hand: a path drawn in order on a line (NP = 1, stress = 0 for any
spacing), K4 (NP = 1 for any drawing), P4 drawn 0, 2, 1, 3 with r = 1 (NP =
2/3, enumerated below), the unit square C4 (stress = (12 - (8 + 2 sqrt 2)^2 / 10)
/ 12), scale invariance of the optimally scaled stress."""
import math

import numpy as np

from oracle import quality as Q
from workloads import complete_graph, cycle_graph, path_graph


def test_path_in_order():
    ip, ix = path_graph(9)
    Y = np.stack([0.5 * np.arange(9.0), np.zeros(9)], axis=1)      # equal spacing (r = 2 needs it)
    assert Q.neighborhood_preservation(ip, ix, Y, r=2) == 1.0
    Yg = np.stack([np.cumsum(np.arange(1, 10) * 0.5), np.zeros(9)], axis=1)
    assert Q.neighborhood_preservation(ip, ix, Yg, r=1) == 1.0      # any order-preserving spacing, r = 1
    assert abs(Q.stress(ip, ix, np.stack([np.arange(9.0), np.zeros(9)], 1))) < 1e-15
    assert abs(Q.stress(ip, ix, np.stack([10 * np.arange(9.0), np.zeros(9)], 1))) < 1e-15


def test_k4_any_drawing():
    ip, ix = complete_graph(4)
    Y = np.random.default_rng(0).normal(size=(4, 2))
    assert Q.neighborhood_preservation(ip, ix, Y, r=2) == 1.0


def test_p4_shuffled_r1():
    """P4 (0-1-2-3) drawn at x: 0 -> 0, 2 -> 1, 1 -> 2, 3 -> 3, r = 1.
    v=0: N_G {1}, nearest {2} -> 0; v=1: N_G {0,2}, distances 2 (v0), 1 (v2),
    1 (v3) -> nearest two {2,3} (tie by id) -> |{2}| / |{0,2,3}| = 1/3;
    v=2: N_G {1,3}, distances 1 (v0), 1 (v1), 2 (v3) -> {0,1} -> 1/3;
    v=3: N_G {2}, nearest: v1 at 1 -> {1} -> 0.  NP = (0 + 1/3 + 1/3 + 0) / 4."""
    ip, ix = path_graph(4)
    Y = np.array([[0.0, 0.0], [2.0, 0.0], [1.0, 0.0], [3.0, 0.0]])
    assert abs(Q.neighborhood_preservation(ip, ix, Y, r=1) - (2.0 / 3.0) / 4.0) < 1e-15


def test_c4_unit_square():
    ip, ix = cycle_graph(4)
    Y = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    s1, s2 = 8 + 4 * math.sqrt(2) / 2, 8 + 4 * 0.5
    want = (12 - s1 * s1 / s2) / 12
    assert abs(Q.stress(ip, ix, Y) - want) < 1e-15
    assert abs(Q.stress(ip, ix, 7.5 * Y) - want) < 1e-15
