"""Time the attractive SpMV alone (CSR kernel vs column-blocked plan) on one
config; the CB consumer-warp count comes from TSNET_CB_WARPS.
    python scripts/attr_probe.py [cfg] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2509_19785_b200 import tsnet_attr, tsnet_build_P, tsnet_plan_build, tsnet_sell_build, tsnet_sell_query  # noqa: E402
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
    sell = "sell skipped"
    Ps = P.without_plan()
    _, ratio = tsnet_sell_query(Ps)
    if ratio <= 3.0 or os.environ.get("SELL_ALWAYS"):
        t0 = time.perf_counter()
        tsnet_sell_build(Ps)
        torch.cuda.synchronize()
        ts_build = time.perf_counter() - t0
        F3 = torch.empty_like(Y)
        t_sell = timed(Ps, Y, F3, reps)
        e3 = float((F3 - F).norm() / F.norm())
        sell = (f"sell {t_sell:.3f} ms ({b / t_sell / 1e6:.0f} GB/s) build {ts_build:.2f}s relL2(sell,csr) {e3:.2e}")
    print(f"cfg{cfg} n={n} nnz={nnz} W={os.environ.get('TSNET_CB_WARPS', 'default')} csr {t_csr:.3f} ms "
          f"({b / t_csr / 1e6:.0f} GB/s)  cb {t_cb:.3f} ms ({b / t_cb / 1e6:.0f} GB/s)  plan {tp:.2f}s  "
          f"relL2(cb,csr) {err:.2e}  sell slots/nnz {ratio:.3f}  {sell}", flush=True)


if __name__ == "__main__":
    main()
