"""Per-kernel device times of L-tsNET iterations late in stage B (iteration
~990, grid N ~ 162 on cfg 4), for an ncu launch list:
    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
        python scripts/late_window_launches.py 4 990 3
The profiled region (cudaProfilerStart/Stop) holds `reps` eager iterations."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2509_19785_b200 import tsnet as T  # noqa: E402
if os.environ.get("PROBE_LIB"):      # a probe build (scripts/tile_variants.sh): build/variants/libtsnet_<name>.so
    T.LIB_PATH = os.path.join(ROOT, "paper_2509_19785_b200", "build", "variants", f"libtsnet_{os.environ['PROBE_LIB']}.so")
from paper_2509_19785_b200 import Layout, tsnet_build_P, tsnet_read_stats  # noqa: E402
from workloads import config_graph, init_layout  # noqa: E402

sys.path.insert(0, ROOT)
from bench import choose_plan  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
start = int(sys.argv[2]) if len(sys.argv) > 2 else 990
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ip, ix = config_graph(cfg)
P = tsnet_build_P(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), u=40.0, seed=0)["P"]
Pk, info = choose_plan(P, None, torch.cuda.Stream())
lay = Layout(Pk, torch.from_numpy(init_layout(P.n, 0)).cuda(), use_graphs=True)
lay.run(start, start=0)
lay.sync()
st = tsnet_read_stats(lay.ws, stream=lay.stream)
print("plan", info, "N", st["N"], "span", st["S"], flush=True)
lay.use_graphs = False
torch.cuda.profiler.start()
for r in range(reps):
    lay.run(1, start=start + r)
    if len(sys.argv) > 4:      # per-iteration spread path and its measure
        st = tsnet_read_stats(lay.ws, stream=lay.stream)
        print("iter", start + r, "spread", st["spread"], "points", st["spread_points"], "flushes",
              st["spread_flushes"], "N", st["N"], flush=True)
lay.sync()
torch.cuda.profiler.stop()
