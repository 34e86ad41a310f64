"""Time the tiled SpMV of every probe build in paper_2509_19785_b200/build/variants
(scripts/tile_variants.sh) on a config: python scripts/tile_variant_probe.py cfg name..."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2509_19785_b200 import tsnet as T  # noqa: E402
from workloads import clustered_layout, config_graph  # noqa: E402


def main():
    cfg = int(sys.argv[1])
    name = sys.argv[2]
    if name != "product":
        T.LIB_PATH = os.path.join(ROOT, "paper_2509_19785_b200", "build", "variants", f"libtsnet_{name}.so")
    ip, ix = config_graph(cfg)
    P = T.tsnet_build_P(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), u=40.0, seed=0)["P"]
    Y = torch.from_numpy(clustered_layout(P.n, 30.0, 40, 2.0, 5)).cuda()
    F0 = T.tsnet_attr(P, Y)
    Q = T.tsnet_plan_build(P.without_plan())
    F = torch.empty_like(Y)
    for _ in range(3):
        T.tsnet_attr(Q, Y, F)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30):
        T.tsnet_attr(Q, Y, F)
    e1.record()
    torch.cuda.synchronize()
    rel = float((F.double() - F0.double()).norm() / F0.double().norm())
    print(json.dumps({"cfg": cfg, "variant": name, "ms": e0.elapsed_time(e1) / 30, "relL2_vs_csr": rel}), flush=True)


if __name__ == "__main__":
    main()
