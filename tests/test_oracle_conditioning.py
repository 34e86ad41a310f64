"""Pins the reading R28 (tests/parity_cases.py): which cases of the stored
oracle trajectories are cancellation residuals.  Oracle only, no GPU."""
import os

import numpy as np
import pytest

import oracle
from parity_cases import COND_LIMIT, CONDITIONED, STAGE_A, STAGE_B
from workloads import config_graph

HERE = os.path.dirname(os.path.abspath(__file__))


def scale_of(r, Y, lam):
    lkl, lc, lr = lam
    n = len(Y)
    return (np.linalg.norm(4 * lkl * r["F_attr"]) + np.linalg.norm(4 * lkl * r["F_rep"])
            + np.linalg.norm(lr * r["g_ent"]) + np.linalg.norm(lc / n * Y))


@pytest.mark.parametrize("cfg", [1, 2])
def test_conditioned_cases_are_exactly_the_listed_ones(cfg):
    ip, ix = config_graph(cfg)
    P = oracle.build_P(ip, ix, 40.0, seed=0)
    pv = P["values"].astype(np.float32).astype(np.float64)
    z = np.load(os.path.join(HERE, "golden", f"oracle_trajectory_cfg{cfg}.npz"))
    for it in (249, 260, 499):
        Y = z[f"Y{it}"].astype(np.float64)
        for lam in (STAGE_A, STAGE_B):
            r = oracle.interp_gradient(Y, P["indptr"], P["indices"], pv, *lam)
            ratio = np.linalg.norm(r["g"]) / scale_of(r, Y, lam)
            key = (cfg, it, lam)
            if key in CONDITIONED:
                assert ratio < COND_LIMIT
                assert abs(np.log10(ratio) - np.log10(CONDITIONED[key])) < 0.5, (key, ratio)
            else:
                assert ratio >= 1e-2, (key, ratio)
