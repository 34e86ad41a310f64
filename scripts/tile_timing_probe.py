"""Per-CTA / per-warp cycle counts of the tiled SpMV (probe build TILE_DIAG=3)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_19785_b200 import tsnet as T  # noqa: E402
from workloads import clustered_layout, config_graph  # noqa: E402

T.LIB_PATH = os.path.join(ROOT, "paper_2509_19785_b200", "build", "variants", "libtsnet_timing.so")
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ip, ix = config_graph(cfg)
P = T.tsnet_build_P(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), u=40.0, seed=0)["P"]
Y = torch.from_numpy(clustered_layout(P.n, 30.0, 40, 2.0, 5)).cuda()
Q = T.tsnet_plan_build(P.without_plan())
F = torch.empty_like(Y)
for _ in range(3):
    T.tsnet_attr(Q, Y, F)
torch.cuda.synchronize()
W = 15
t = F[:148 * W].cpu().numpy().reshape(148, W, 2)
tot, wait = t[..., 0], t[..., 1]
ip_h = P.indptr.cpu().numpy()
out = {"cta_max_cycles": float(tot.max()), "cta_mean_cycles": float(tot.max(1).mean()),
       "cta_min_cycles": float(tot.max(1).min()), "warp_wait_frac_mean": float((wait / tot).mean()),
       "slowest_ctas": np.argsort(-tot.max(1))[:5].tolist(), "slowest_cta_wait_frac": float((wait / tot)[np.argmax(tot.max(1))].mean())}
print(json.dumps(out))
np.save(os.path.join(ROOT, "gpurun_out", f"tile_timing_cfg{cfg}.npy"), t)
