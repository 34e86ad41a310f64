"""Experiment: does a spatial (Morton of the layout) renumbering of the
vertices make the attractive SpMV's Y[j] gathers local?  Runs the layout
(250 stage-A + K stage-B iterations, as bench.py), permutes P and Y by the
Morton order of the layout, and times tsnet_attr on both.
    python scripts/reorder_probe.py [cfg] [stageB_iters]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_19785_b200 import CSR, Layout, tsnet_attr, tsnet_build_P  # noqa: E402
from workloads import config_graph, init_layout  # noqa: E402


def timed(P, Y, reps=30):
    F = torch.empty_like(Y)
    for _ in range(3):
        tsnet_attr(P, Y, F)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        tsnet_attr(P, Y, F)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, F


def morton(Y):
    lo = Y.min(0).values
    span = (Y.max(0).values - lo).max().clamp_min(1e-12)
    q = ((Y - lo) / span * 65535).long().clamp(0, 65535)
    def spread(v):
        v = (v | (v << 8)) & 0x00FF00FF
        v = (v | (v << 4)) & 0x0F0F0F0F
        v = (v | (v << 2)) & 0x33333333
        v = (v | (v << 1)) & 0x55555555
        return v
    return spread(q[:, 0]) | (spread(q[:, 1]) << 1)


def permute(P, perm):
    """P' = Pi P Pi^T with new index = position in perm."""
    n = P.n
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(n, device=perm.device)
    rows = torch.repeat_interleave(torch.arange(n, device=perm.device), P.indptr[1:] - P.indptr[:-1])
    r2 = inv[rows]
    c2 = inv[P.indices.long()]
    key = r2 * n + c2
    order = torch.argsort(key)
    r2, c2, v2 = r2[order], c2[order], P.values[order]
    ip = torch.zeros(n + 1, dtype=torch.int64, device=perm.device)
    ip[1:] = torch.cumsum(torch.bincount(r2, minlength=n), 0)
    return CSR(ip, c2.int().contiguous(), v2.contiguous())


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    kb = int(sys.argv[2]) if len(sys.argv) > 2 else 500
    ip, ix = config_graph(cfg)
    P = tsnet_build_P(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), u=40.0, seed=0)["P"]
    lay = Layout(P, torch.from_numpy(init_layout(P.n, 0)).cuda()).run(250 + kb)
    lay.sync()
    Y = lay.Y.clone()
    t0, F0 = timed(P, Y)
    perm = torch.argsort(morton(Y))
    P2 = permute(P, perm)
    Y2 = Y[perm].contiguous()
    t1, F1 = timed(P2, Y2)
    err = float((F1 - F0[perm]).norm() / F0.norm())
    span = float((Y.max(0).values - Y.min(0).values).max())
    print(f"cfg{cfg} after {250 + kb} its (span {span:.2f}): SpMV original {t0:.3f} ms, Morton-renumbered {t1:.3f} ms,"
          f" relL2 {err:.1e}", flush=True)


if __name__ == "__main__":
    main()
