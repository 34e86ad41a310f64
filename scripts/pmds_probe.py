"""Time tsnet_pmds (set-up) on a config graph.   python scripts/pmds_probe.py [cfg] [pivots]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2509_19785_b200 import tsnet_pmds  # noqa: E402
from workloads import config_graph  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 250
    ip, ix = config_graph(cfg)
    ipd, ixd = torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda()
    tsnet_pmds(ipd, ixd, 4, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = tsnet_pmds(ipd, ixd, p, 0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    Y = r["Y"]
    print(f"cfg{cfg} n={len(ip) - 1} m={len(ix) // 2} pivots={p}: {dt:.3f} s  eig={r['eig'].cpu().tolist()}  "
          f"span=({float(Y[:, 0].max() - Y[:, 0].min()):.3g}, {float(Y[:, 1].max() - Y[:, 1].min()):.3g})", flush=True)


if __name__ == "__main__":
    main()
