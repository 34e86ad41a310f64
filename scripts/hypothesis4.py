"""Hypothesis 4 on synthetic graphs: NP (r = 2) and stress
of the drawings of tsNET (exact gradient), BH-tsNET, FIt-tsNET and L-tsNET
from the same PMDS start, and the time per iteration of each.
    python scripts/hypothesis4.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2509_19785_b200 import tsnet_build_P, tsnet_pmds, tsnet_quality  # noqa: E402
from paper_2509_19785_b200.variants import run_method  # noqa: E402
from workloads import config_graph, cycle_graph, grid2d  # noqa: E402

GRAPHS = {"grid 32x32 (cfg 1)": lambda: config_graph(1), "cycle 500": lambda: cycle_graph(500),
          "grid 100x100": lambda: grid2d(100, 100), "RGG n=20k (cfg 2)": lambda: config_graph(2)}


def main():
    out = []
    for name, make in GRAPHS.items():
        ip, ix = make()
        ipd, ixd = torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda()
        P = tsnet_build_P(ipd, ixd, u=40.0, seed=0)["P"]
        Y0 = tsnet_pmds(ipd, ixd, 250, 0)["Y"]
        Y0 = Y0 * (1e-4 / float(Y0.std()))
        row = {"graph": name, "n": P.n}
        for m in ("tsnet", "bh", "fit", "linear"):
            if m == "tsnet" and P.n > 12000:
                continue
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            Y = run_method(P, Y0, m, iters=500)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / 500 * 1e3
            npv, st = tsnet_quality(ipd, ixd, Y, 2)
            row[m] = {"np": round(npv, 4), "stress": round(st, 4), "ms_per_iter": round(dt, 3)}
        print(json.dumps(row), flush=True)
        out.append(row)


if __name__ == "__main__":
    main()
