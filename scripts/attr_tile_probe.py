"""Time the attractive SpMV (tsnet_attr) on a config with the CSR kernel and
with the column-blocked (tiled) plan; check the plan against the CSR result on
all rows.  python scripts/attr_tile_probe.py [cfg] [reps]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_19785_b200 import tsnet_attr, tsnet_build_P  # noqa: E402
from paper_2509_19785_b200 import tsnet as T  # noqa: E402
from workloads import clustered_layout, config_graph  # noqa: E402


def timeit(P, Y, F, reps):
    for _ in range(3):
        tsnet_attr(P, Y, F)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        tsnet_attr(P, Y, F)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    ip, ix = config_graph(cfg)
    P = tsnet_build_P(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), u=40.0, seed=0)["P"]
    n, nnz = P.n, P.nnz
    Y = torch.from_numpy(clustered_layout(n, 30.0, 40, 2.0, 5)).cuda()
    F0 = torch.empty_like(Y)
    t_csr = timeit(P, Y, F0, reps)
    t0 = time.perf_counter()
    Q = T.tsnet_plan_build(P.without_plan())
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    F1 = torch.full_like(Y, float("nan"))
    t_cb = timeit(Q, Y, F1, reps)
    a, b = F1.double(), F0.double()
    rel = float((a - b).norm() / b.norm())
    byts = 8 * nnz + 8 * (n + 1) + 16 * n
    out = {"cfg": cfg, "n": n, "nnz": nnz, "csr_ms": t_csr, "cb_ms": t_cb, "cb_build_s": build_s,
           "plan_bytes": int(Q.plan.numel()), "relL2_cb_vs_csr": rel, "nan": bool(torch.isnan(F1).any()),
           "csr_frac": byts / (t_csr * 1e-3) / 6537.3e9, "cb_frac": byts / (t_cb * 1e-3) / 6537.3e9}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
