"""Dump the structure of a few panels of a config's P (local rows in ascending
order, their global columns) for offline study of the tiled SpMV's entry
schedule: python scripts/dump_panel.py cfg out.npz [panels...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_19785_b200 import tsnet as T  # noqa: E402
from workloads import config_graph  # noqa: E402


def main():
    cfg, out = int(sys.argv[1]), sys.argv[2]
    panels = [int(a) for a in sys.argv[3:]] or [0]
    ip, ix = config_graph(cfg)
    P = T.tsnet_build_P(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), u=40.0, seed=0)["P"]
    pip = P.indptr.cpu().numpy().astype(np.int64)
    pix = P.indices.cpu().numpy()
    n = len(pip) - 1
    Pn, row_panel, row_local, panel_off, panel_rows = T.tsnet_plan_partition(pip, 0, n, 148, 6464)
    d = {"n": n, "P": Pn}
    for p in panels:
        rows = panel_rows[panel_off[p]:panel_off[p + 1]]
        lens = pip[rows + 1] - pip[rows]
        d[f"rows{p}"] = rows
        d[f"ptr{p}"] = np.concatenate([[0], np.cumsum(lens)])
        d[f"cols{p}"] = np.concatenate([pix[pip[r]:pip[r + 1]] for r in rows]).astype(np.int32)
    np.savez_compressed(out, **d)
    print(n, Pn, [len(d[f"cols{p}"]) for p in panels])


if __name__ == "__main__":
    main()
