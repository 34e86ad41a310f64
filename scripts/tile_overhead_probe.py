"""Time the tiled SpMV on synthetic CSRs with n = 947,974 rows and d uniformly
random columns per row (d = 1 .. 256): the time at small d is the per-tile floor
(every (panel, block) tile still runs), the slope the per-entry cost.
    python scripts/tile_overhead_probe.py [lib-variant]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2509_19785_b200 import tsnet as T  # noqa: E402

if len(sys.argv) > 1:
    T.LIB_PATH = os.path.join(ROOT, "paper_2509_19785_b200", "build", "variants", f"libtsnet_{sys.argv[1]}.so")
n = 947974
g = torch.Generator(device="cuda").manual_seed(0)
Y = torch.randn(n, 2, device="cuda", generator=g) * 5
for d in (1, 4, 16, 64, 128, 217):
    cols = torch.randint(0, n, (n, d), device="cuda", generator=g, dtype=torch.int64)
    cols, _ = torch.sort(cols, dim=1)
    indptr = torch.arange(0, n * d + 1, d, device="cuda", dtype=torch.int64)
    P = T.CSR(indptr, cols.reshape(-1).to(torch.int32).contiguous(),
              torch.rand(n * d, device="cuda", generator=g) * 1e-6 + 1e-9)
    F0 = T.tsnet_attr(P, Y)
    Q = T.tsnet_plan_build(P)
    F = torch.empty_like(Y)
    for _ in range(3):
        T.tsnet_attr(Q, Y, F)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        T.tsnet_attr(Q, Y, F)
    e1.record()
    torch.cuda.synchronize()
    rel = float((F.double() - F0.double()).norm() / F0.double().norm())
    print(json.dumps({"d": d, "nnz": n * d, "ms": e0.elapsed_time(e1) / 20, "relL2_vs_csr": rel}), flush=True)
    del P, Q, cols, F0, F
    torch.cuda.empty_cache()
