"""Grid geometry along a full L-tsNET run (SURVEY §8 "spans at
n = 0.2M-4M are unmeasured"): span S, intervals I, nodes N = 3I and the
per-iteration time of 50-iteration windows, for configs given on the command
line, from the seeded init through iteration 999 (stage A 0-249, stage B after).

    python scripts/spans.py 3 4 5 > gpurun_out/spans.jsonl
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2509_19785_b200 import Layout, attach_plan, tsnet_build_P, tsnet_read_stats  # noqa: E402
from workloads import config_graph, init_layout  # noqa: E402


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [3, 4, 5]
    iters = int(os.environ.get("SPAN_ITERS", "1000"))
    dev = torch.device("cuda", 0)
    for cfg in cfgs:
        ip, ix = config_graph(cfg)
        P = tsnet_build_P(torch.from_numpy(ip).to(dev), torch.from_numpy(ix).to(dev), u=40.0, seed=0)["P"]
        attach_plan(P, "auto")
        lay = Layout(P, torch.from_numpy(init_layout(P.n, 0)).to(dev), use_graphs=True)
        rec = []
        w = 50
        for it0 in range(0, iters, w):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            Ns = []
            e0.record(lay.stream)
            for it in range(it0, min(iters, it0 + w)):
                lay.step(it)
            e1.record(lay.stream)
            lay.sync()
            st = tsnet_read_stats(lay.ws, stream=lay.stream)
            ms = e0.elapsed_time(e1) / (min(iters, it0 + w) - it0)
            rec.append({"it_end": min(iters, it0 + w) - 1, "S": st["S"], "I": st["I"], "N": st["N"],
                        "ms_per_iter": ms, "nonfinite": st["nonfinite"]})
        print(json.dumps({"cfg": cfg, "n": P.n, "nnz": P.nnz, "windows": rec}), flush=True)
        del lay, P
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
