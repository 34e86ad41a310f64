"""Time L-tsNET steps of a probe build (paper_2509_19785_b200/build/variants,
scripts/tile_variants.sh) after `start` iterations on a config:
    python scripts/step_variant_probe.py cfg start name [steps] [eager|graph] [spread]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2509_19785_b200 import tsnet as T  # noqa: E402

cfg, start, name = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
eager = len(sys.argv) > 5 and sys.argv[5] == "eager"
spread = int(sys.argv[6]) if len(sys.argv) > 6 else 0
if name != "product":
    T.LIB_PATH = os.path.join(ROOT, "paper_2509_19785_b200", "build", "variants", f"libtsnet_{name}.so")
from paper_2509_19785_b200 import GradParams, Layout, tsnet_build_P, tsnet_read_stats  # noqa: E402
from workloads import config_graph, init_layout  # noqa: E402
from bench import choose_plan  # noqa: E402

ip, ix = config_graph(cfg)
P = tsnet_build_P(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), u=40.0, seed=0)["P"]
Pk, info = choose_plan(P, None, torch.cuda.Stream())
lay = Layout(Pk, torch.from_numpy(init_layout(P.n, 0)).cuda(), base=GradParams(spread=spread), use_graphs=True)
lay.run(start, start=0)
lay.sync()
lay.use_graphs = not eager
lay.run(3, start=start)
lay.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(lay.stream):
    e0.record()
lay.run(steps, start=start)
with torch.cuda.stream(lay.stream):
    e1.record()
lay.sync()
st = tsnet_read_stats(lay.ws, stream=lay.stream)
print(json.dumps({"cfg": cfg, "variant": name, "eager": eager, "spread_req": spread, "spread": st.get("spread"), "start": start, "ms_per_step": e0.elapsed_time(e1) / steps, "N": st["N"],
                  "span": st["S"], "nonfinite": st.get("nonfinite")}), flush=True)
