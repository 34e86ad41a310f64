"""SpMV (a6) probe: how much of k_spmv's time is the random Y[j] gathers?

Times tsnet_attr (CUDA events, 50 launches) on the config's P and on variants
with the same row structure but different column patterns:
  real      the P built by tsnet_build_P
  self      every column replaced by the row id (gathers hit one address / row)
  rcm       P of the graph relabelled by reverse Cuthill-McKee (locality of ids)
Prints one JSON line per variant: ms, algorithmic GB/s, fraction of measured peak.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_19785_b200 import CSR, tsnet_attr, tsnet_build_P  # noqa: E402
from workloads import clustered_layout, config_graph  # noqa: E402


def time_attr(P, Y, reps=50):
    F = torch.empty_like(Y)
    for _ in range(3):
        tsnet_attr(P, Y, F)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        tsnet_attr(P, Y, F)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    ip, ix = config_graph(cfg)
    n = len(ip) - 1
    dev = torch.device("cuda")
    P = tsnet_build_P(torch.from_numpy(ip).to(dev), torch.from_numpy(ix).to(dev), u=40.0)["P"]
    Y = torch.from_numpy(clustered_layout(n, 30.0, 40, 2.0, 5)).to(dev)
    nnz = P.nnz
    byts = 8 * nnz + 24 * n + 8

    def rep(name, PP, YY):
        ms = time_attr(PP, YY)
        gbs = byts / (ms * 1e-3) / 1e9
        print(json.dumps({"variant": name, "cfg": cfg, "n": n, "nnz": nnz, "ms": ms, "GBps": gbs,
                          "frac": gbs / peak}), flush=True)

    rep("real", P, Y)
    rows = torch.repeat_interleave(torch.arange(n, device=dev, dtype=torch.int32),
                                   (P.indptr[1:] - P.indptr[:-1]))
    rep("self", CSR(P.indptr, rows, P.values), Y)
    del rows
    import scipy.sparse as sp
    from scipy.sparse.csgraph import reverse_cuthill_mckee
    A = sp.csr_matrix((np.ones(len(ix), np.int8), ix, ip), shape=(n, n))
    perm = reverse_cuthill_mckee(A, symmetric_mode=True).astype(np.int64)
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    B = A[perm][:, perm]
    B.sort_indices()
    P2 = tsnet_build_P(torch.from_numpy(B.indptr.astype(np.int64)).to(dev),
                       torch.from_numpy(B.indices.astype(np.int32)).to(dev), u=40.0)["P"]
    rep("rcm", P2, Y[torch.from_numpy(perm).to(dev)].contiguous())


if __name__ == "__main__":
    main()
