"""The paper's four algorithms run through the same schedule (Alg. 1-3;
SURVEY §8(f) NEXT-3/4): tsNET (the exact gradient, here the quadtree walk with
theta = 0, which is the exact O(n^2) sum), BH-tsNET and FIt-tsNET
(tsnet_grad_tree) and L-tsNET (tsnet_step).  Every step runs in libtsnet's
kernels; this module only sequences the calls (stage A / stage B multipliers
and momentum of runner.stage_params) for the Hypothesis-4 quality comparison
("very similar quality metrics")."""
from __future__ import annotations

import torch

from .runner import stage_of, stage_params
from .tsnet import CSR, alloc_workspace, lib, tsnet_grad_tree, tsnet_move, tsnet_step

METHODS = ("tsnet", "bh", "fit", "linear")


def run_method(P: CSR, Y0: torch.Tensor, method: str, iters: int = 500, theta: float = 0.5, stream=None,
               start: int = 0, state=None):
    """Layout after iterations start .. start + iters of `method` from Y0
    (device n x 2 fp32); `state` = (vel, gains) to continue a run (updated in
    place), else zero velocity and unit gains."""
    assert method in METHODS
    Y = Y0.clone()
    vel, gains = state if state is not None else (torch.zeros_like(Y), torch.ones_like(Y))
    params = [stage_params(0), stage_params(1)]
    ws = alloc_workspace(P.n, P.nnz, params[0][0], device=Y.device)
    tws = None
    if method != "linear":
        tws = torch.empty(max(int(lib().tsnet_tree_workspace_bytes(P.n)), 1), dtype=torch.uint8, device=Y.device)
    grad = torch.empty_like(Y)
    for it in range(start, start + iters):
        gp, sp = params[stage_of(it)]
        if method == "linear":
            tsnet_step(P, Y, vel, gains, gp, sp, ws, stream=stream)
            continue
        th = 0.0 if method == "tsnet" else theta
        variant = 1 if method == "fit" else 0
        tsnet_grad_tree(P, Y, gp, ws, theta=th, variant=variant, tree_ws=tws, grad=grad, stream=stream)
        tsnet_move(Y, vel, gains, grad, sp, stream=stream)
    return Y
