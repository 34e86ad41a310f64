"""Time the quadtree gradients (BH-tsNET, FIt-tsNET) against the L-tsNET
gradient on a config graph at a converged-like layout.   python scripts/tree_probe.py [cfg]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2509_19785_b200 import GradParams, alloc_workspace, tsnet_build_P, tsnet_grad, tsnet_grad_tree  # noqa: E402
from paper_2509_19785_b200 import tsnet as T  # noqa: E402
from workloads import clustered_layout, config_graph  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    ip, ix = config_graph(cfg)
    P = tsnet_build_P(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), u=40.0, seed=0)["P"]
    n = P.n
    Y = torch.from_numpy(clustered_layout(n, 10.0, 40, 2.0, 5)).cuda()
    gp = GradParams(1.0, 0.01, 0.6)
    ws = alloc_workspace(n, P.nnz, gp)
    tws = torch.empty(int(T.lib().tsnet_tree_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
    t_l = timed(lambda: tsnet_grad(P, Y, gp, ws))
    t_bh = timed(lambda: tsnet_grad_tree(P, Y, gp, ws, theta=0.5, variant=0, tree_ws=tws), 3)
    t_fit = timed(lambda: tsnet_grad_tree(P, Y, gp, ws, theta=0.5, variant=1, tree_ws=tws), 3)
    print(f"cfg{cfg} n={n}: gradient L-tsNET {t_l:.3f} ms, BH-tsNET (theta 0.5) {t_bh:.1f} ms, "
          f"FIt-tsNET {t_fit:.1f} ms", flush=True)


if __name__ == "__main__":
    main()
