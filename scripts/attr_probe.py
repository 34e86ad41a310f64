"""Time the attractive SpMV alone (CSR kernel vs column-blocked plan) on one
config; the CB consumer-warp count comes from TSNET_CB_WARPS.
    python scripts/attr_probe.py [cfg] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2509_19785_b200 import tsnet_attr, tsnet_build_P, tsnet_plan_build  # noqa: E402
from workloads import clustered_layout, config_graph  # noqa: E402


def timed(P, Y, F, reps):
    s = torch.cuda.current_stream()
    for _ in range(3):
        tsnet_attr(P, Y, F)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        tsnet_attr(P, Y, F)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    ip, ix = config_graph(cfg)
    got = tsnet_build_P(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), u=40.0, seed=0)
    P = got["P"]
    n, nnz = P.n, P.nnz
    Y = torch.from_numpy(clustered_layout(n, 10.0, 40, 2.0, 5)).cuda()
    F = torch.empty_like(Y)
    t_csr = timed(P.without_plan(), Y, F, reps)
    t0 = time.perf_counter()
    tsnet_plan_build(P)
    torch.cuda.synchronize()
    tp = time.perf_counter() - t0
    F2 = torch.empty_like(Y)
    t_cb = timed(P, Y, F2, reps)
    err = float((F2 - F).norm() / F.norm())
    b = 8 * nnz + 8 * (n + 1) + 16 * n
    print(f"cfg{cfg} n={n} nnz={nnz} W={os.environ.get('TSNET_CB_WARPS', 'default')} csr {t_csr:.3f} ms "
          f"({b / t_csr / 1e6:.0f} GB/s)  cb {t_cb:.3f} ms ({b / t_cb / 1e6:.0f} GB/s)  plan {tp:.2f}s  "
          f"relL2(cb,csr) {err:.2e}", flush=True)


if __name__ == "__main__":
    main()
