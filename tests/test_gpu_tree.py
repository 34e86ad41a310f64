"""Quadtree (Barnes-Hut) gradients of BH-tsNET and FIt-tsNET (NEXT-3;
tsnet_grad_tree, tree.cu) against the oracle O9 (oracle/bh.py).  Both sides
build the same tree (fp64 Morton cells of the same fp32 points, stable order)
and take the same summary decisions (fp64 criterion), so BH-tsNET agrees to
fp32 output rounding (relL2 <= 1e-6) and Z to 1e-12; theta = 0 is the exact
gradient; FIt-tsNET = the interpolated gradient with lambda_r = 0 (bar 1e-4,
as tsnet_grad) plus the quadtree entropy."""
import numpy as np
import pytest
import torch

import oracle
from oracle import bh as B
from paper_2509_19785_b200 import CSR, GradParams, alloc_workspace, tsnet_grad, tsnet_grad_tree
from paper_2509_19785_b200 import tsnet as T
from workloads import clustered_layout, config_graph, grid2d, uniform_layout

pytestmark = pytest.mark.gpu

LAM = (1.0, 0.01, 0.6)


def relL2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def dev(P):
    return CSR(torch.from_numpy(P["indptr"]).cuda(), torch.from_numpy(P["indices"]).cuda(),
               torch.from_numpy(P["values"].astype(np.float32)).cuda())


_P = {}


def Pcfg(cfg):
    if cfg not in _P:
        ip, ix = config_graph(cfg)
        _P[cfg] = oracle.build_P(ip, ix, 40.0, seed=0)
    return _P[cfg]


def gpu(P, Y, theta, variant, lam=LAM):
    Pd = dev(P)
    gp = GradParams(*lam)
    ws = alloc_workspace(P["n"], Pd.nnz, gp)
    g, Z = tsnet_grad_tree(Pd, torch.from_numpy(Y).cuda(), gp, ws, theta=theta, variant=variant)
    torch.cuda.synchronize()
    return g.cpu().numpy().astype(np.float64), float(Z.item())


@pytest.mark.parametrize("theta", [0.5, 0.3])
@pytest.mark.parametrize("lay", ["clustered", "uniform"])
def test_bh_tsnet_config1(theta, lay):
    P = Pcfg(1)
    n = P["n"]
    Y = clustered_layout(n, 20.0, 5, 1.5, 7) if lay == "clustered" else uniform_layout(n, 3.0, 4)
    g, Z = gpu(P, Y, theta, 0)
    r = B.bh_gradient(Y.astype(np.float64), P["indptr"], P["indices"], P["values"].astype(np.float32).astype(np.float64),
                      *LAM, eps=0.05, theta=theta)
    assert abs(Z - r["Z"]) <= 1e-12 * r["Z"]
    assert relL2(g, r["g"]) <= 1e-6


def test_theta_zero_is_exact():
    ip, ix = grid2d(20, 17)
    P = oracle.build_P(ip, ix, 10.0, seed=0)
    Y = clustered_layout(P["n"], 10.0, 4, 1.0, 3)
    g, Z = gpu(P, Y, 0.0, 0)
    ge, Ze = oracle.exact_grad(Y.astype(np.float64), P["indptr"], P["indices"],
                               P["values"].astype(np.float32).astype(np.float64), *LAM, eps=0.05)
    assert abs(Z - Ze) <= 1e-12 * Ze
    assert relL2(g, ge) <= 1e-6


def test_fit_tsnet_config1():
    P = Pcfg(1)
    n = P["n"]
    Y = clustered_layout(n, 20.0, 5, 1.5, 7)
    g, _ = gpu(P, Y, 0.5, 1)
    pv = P["values"].astype(np.float32).astype(np.float64)
    gi = oracle.interp_gradient(Y.astype(np.float64), P["indptr"], P["indices"], pv, LAM[0], LAM[1], 0.0,
                                eps=0.05)["g"]
    ge = B.bh_gradient(Y.astype(np.float64), P["indptr"], P["indices"], pv, *LAM, eps=0.05, theta=0.5,
                       repulsion=False)["g"]
    assert relL2(g, gi + ge) <= 1e-4


def test_bh_config3_sampled_points():
    """n = 0.2M: sampled points' gradients against the oracle's walk of the
    same tree (with the GPU's Z, checked separately against the exact Z)."""
    P = Pcfg(3)
    n = P["n"]
    Y = clustered_layout(n, 30.0, 40, 2.0, 5)
    g, Z = gpu(P, Y, 0.5, 0)
    Yd = Y.astype(np.float64)
    T_ = B.Quadtree(Yd)
    pv = P["values"].astype(np.float32).astype(np.float64)
    rows = np.random.default_rng(0).choice(n, 40, replace=False)
    for i in rows:
        _, R, E = T_.sums(int(i), 0.5, 0.05)
        fa = oracle.attr_sparse_rows(Yd, P["indptr"], P["indices"], pv, int(i), 1)[0]
        want = 4.0 * LAM[0] * (fa - R / Z) + (LAM[1] / n) * Yd[i] - (LAM[2] / n ** 2) * E
        assert np.linalg.norm(g[i] - want) <= 1e-5 * np.linalg.norm(want) + 1e-30
    # Z against the interpolated Z (tsnet_grad, ~1e-4 accurate), within the BH error
    Pd = dev(P)
    gp = GradParams(*LAM)
    _, Zi = tsnet_grad(Pd, torch.from_numpy(Y).cuda(), gp, alloc_workspace(n, Pd.nnz, gp))
    Zi = float(Zi.item())
    assert abs(Z - Zi) <= 2e-2 * Zi


def test_arguments():
    P = Pcfg(1)
    with pytest.raises(T.TsnetError):
        gpu(P, uniform_layout(P["n"], 3.0, 1), 0.9, 0)
    with pytest.raises(T.TsnetError):
        gpu(P, uniform_layout(P["n"], 3.0, 1), 0.5, 2)
