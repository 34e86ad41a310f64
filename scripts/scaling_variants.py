"""Per-iteration time of tsNET (exact), BH-tsNET, FIt-tsNET and L-tsNET on
square grid graphs of growing n (SPEC acceptance 5/6: log-log slopes and the
ordering linear < fit < bh < exact; PAPER.md Theorems 1-3 and Fig. 2's
"93.5%, 96%, and 98.6% faster").  Times iterations 250..500 of the schedule
from a PMDS start, CUDA events around the whole loop.
    python scripts/scaling_variants.py"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_19785_b200 import tsnet_build_P, tsnet_pmds  # noqa: E402
from paper_2509_19785_b200.variants import run_method  # noqa: E402
from workloads import grid2d  # noqa: E402

SIDES = (32, 64, 128, 181)          # n = 1024, 4096, 16384, 32761
EXACT_MAX_N = 5000


def per_iter_ms(P, Y0, m):
    st = (torch.zeros_like(Y0), torch.ones_like(Y0))
    Y = run_method(P, Y0, m, iters=250, state=st)                      # stage A, untimed
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    run_method(P, Y, m, iters=250, start=250, state=st)                # stage B, timed
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 250


def main():
    rows = []
    for a in SIDES:
        ip, ix = grid2d(a, a)
        ipd, ixd = torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda()
        P = tsnet_build_P(ipd, ixd, u=40.0, seed=0)["P"]
        Y0 = tsnet_pmds(ipd, ixd, 250, 0)["Y"]
        Y0 = Y0 * (1e-4 / float(Y0.std()))
        row = {"n": P.n}
        for m in ("tsnet", "bh", "fit", "linear"):
            if m == "tsnet" and P.n > EXACT_MAX_N:
                continue
            row[m] = round(per_iter_ms(P, Y0, m), 4)
        print(json.dumps(row), flush=True)
        rows.append(row)
    for m in ("tsnet", "bh", "fit", "linear"):
        pts = [(r["n"], r[m]) for r in rows if m in r]
        if len(pts) >= 2:
            x = np.log([p[0] for p in pts])
            y = np.log([p[1] for p in pts])
            print(json.dumps({"method": m, "loglog_slope": round(float(np.polyfit(x, y, 1)[0]), 3)}), flush=True)


if __name__ == "__main__":
    main()
