"""Per-CTA / per-warp cycle counts of the tiled SpMV (probe builds TILE_DIAG=3 -> libtsnet_timing.so,
TILE_DIAG=4 -> libtsnet_timing4.so: also the cycles each warp waits at the per-block barrier).
    python scripts/tile_timing_probe.py cfg [timing|timing4]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_19785_b200 import tsnet as T  # noqa: E402
from workloads import clustered_layout, config_graph  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
lib = sys.argv[2] if len(sys.argv) > 2 else "timing"
T.LIB_PATH = os.path.join(ROOT, "paper_2509_19785_b200", "build", "variants", f"libtsnet_{lib}.so")
ip, ix = config_graph(cfg)
P = T.tsnet_build_P(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), u=40.0, seed=0)["P"]
Y = torch.from_numpy(clustered_layout(P.n, 30.0, 40, 2.0, 5)).cuda()
Q = T.tsnet_plan_build(P.without_plan())
F = torch.empty_like(Y)
for _ in range(3):
    T.tsnet_attr(Q, Y, F)
torch.cuda.synchronize()
W = 15
if lib == "timing4":
    t4 = F[:2 * 148 * W].cpu().numpy().reshape(148, W, 2, 2)
    tot, wait, bar = t4[..., 0, 0], t4[..., 0, 1], t4[..., 1, 0]
    print(json.dumps({"cfg": cfg, "cta_max_cycles": float(tot.max()), "cta_mean_cycles": float(tot.max(1).mean()),
                      "ring_wait_frac_mean": float((wait / tot).mean()), "barrier_wait_frac_mean": float((bar / tot).mean()),
                      "barrier_wait_frac_min_warp": float((bar / tot).min()),
                      "barrier_wait_frac_max_warp": float((bar / tot).max()),
                      "barrier_wait_frac_by_warp": (bar / tot).mean(0).round(4).tolist()}))
    np.save(os.path.join(ROOT, "gpurun_out", f"tile_timing4_cfg{cfg}.npy"), t4)
    sys.exit(0)
t = F[:148 * W].cpu().numpy().reshape(148, W, 2)
tot, wait = t[..., 0], t[..., 1]
ip_h = P.indptr.cpu().numpy()
out = {"cta_max_cycles": float(tot.max()), "cta_mean_cycles": float(tot.max(1).mean()),
       "cta_min_cycles": float(tot.max(1).min()), "warp_wait_frac_mean": float((wait / tot).mean()),
       "slowest_ctas": np.argsort(-tot.max(1))[:5].tolist(), "slowest_cta_wait_frac": float((wait / tot)[np.argmax(tot.max(1))].mean())}
print(json.dumps(out))
np.save(os.path.join(ROOT, "gpurun_out", f"tile_timing_cfg{cfg}.npy"), t)
