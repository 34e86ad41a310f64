"""Experiment: where the end-to-end (host buffers) iteration time goes on cfg 4.
Times with CUDA events: the host<->device copies alone, the device step alone,
and tsnet_step_host (wall clock, blocking) for the chunk count of this process
(TSNET_HOST_CHUNKS).
    TSNET_HOST_CHUNKS=8 python scripts/e2e_probe.py [cfg]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_19785_b200 import GradParams, StepParams, alloc_workspace, tsnet_build_P, tsnet_step, tsnet_step_host  # noqa: E402
from workloads import config_graph, init_layout  # noqa: E402


def ev_time(fn, reps, stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    ip, ix = config_graph(cfg)
    P = tsnet_build_P(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), u=40.0, seed=0)["P"]
    n = P.n
    gp, sp = GradParams(1.0, 0.01, 0.6), StepParams(eta=50.0, momentum=0.8)
    ws = alloc_workspace(n, P.nnz, gp)
    Y = torch.from_numpy(init_layout(n, 0) * 1e4).cuda()
    V, G = torch.zeros_like(Y), torch.ones_like(Y)
    s = torch.cuda.Stream()
    Yh, Vh, Gh = Y.cpu().pin_memory(), V.cpu().pin_memory(), G.cpu().pin_memory()
    b = Y.numel() * 4
    with torch.cuda.stream(s):
        h2d1 = ev_time(lambda: Y.copy_(Yh, non_blocking=True), 20, s)
        h2d3 = ev_time(lambda: (Y.copy_(Yh, non_blocking=True), V.copy_(Vh, non_blocking=True),
                                G.copy_(Gh, non_blocking=True)), 20, s)
        d2h3 = ev_time(lambda: (Yh.copy_(Y, non_blocking=True), Vh.copy_(V, non_blocking=True),
                                Gh.copy_(G, non_blocking=True)), 20, s)
        h2dV = ev_time(lambda: V.copy_(Vh, non_blocking=True), 20, s)
        h2dG = ev_time(lambda: G.copy_(Gh, non_blocking=True), 20, s)
        h2dYYY = ev_time(lambda: (Y.copy_(Yh, non_blocking=True), Y.copy_(Yh, non_blocking=True),
                                  Y.copy_(Yh, non_blocking=True)), 20, s)
        big_h = torch.empty(3 * Y.numel(), dtype=torch.float32).pin_memory()
        big_d = torch.empty(3 * Y.numel(), dtype=torch.float32, device="cuda")
        h2dbig = ev_time(lambda: big_d.copy_(big_h, non_blocking=True), 20, s)
        print(f"H2D V {h2dV:.3f}  H2D G {h2dG:.3f}  H2D Y x3 {h2dYYY:.3f}  H2D one 3n buffer {h2dbig:.3f} ms", flush=True)
        dev = ev_time(lambda: tsnet_step(P, Y, V, G, gp, sp, ws, stream=s), 50, s)
    # the device step while another stream streams D2H / H2D copies (DMA interference)
    s2 = torch.cuda.Stream()
    D = [torch.empty_like(Y) for _ in range(3)]
    H = [torch.empty(Y.shape, dtype=torch.float32).pin_memory() for _ in range(3)]

    def with_dma(direction):
        def fn():
            with torch.cuda.stream(s2):
                for d, h in zip(D, H):
                    if direction == "d2h":
                        h.copy_(d, non_blocking=True)
                    else:
                        d.copy_(h, non_blocking=True)
            tsnet_step(P, Y, V, G, gp, sp, ws, stream=s)
            s.wait_stream(s2)
        return fn
    with torch.cuda.stream(s):
        dev_d2h = ev_time(with_dma("d2h"), 30, s)
        dev_h2d = ev_time(with_dma("h2d"), 30, s)
    print(f"device step {dev:.3f} ms; with concurrent 3 x {b / 1e6:.1f} MB D2H {dev_d2h:.3f}, H2D {dev_h2d:.3f} "
          f"(copies alone: D2H {d2h3:.3f}, H2D {h2d3:.3f})", flush=True)
    Yh.copy_(Y.cpu()), Vh.copy_(V.cpu()), Gh.copy_(G.cpu())
    tsnet_step_host(P, Yh, Vh, Gh, gp, sp, ws, stream=s)
    ts = []
    for _ in range(60):
        t0 = time.perf_counter()
        tsnet_step_host(P, Yh, Vh, Gh, gp, sp, ws, stream=s)
        ts.append(time.perf_counter() - t0)
    ts = np.array(ts[10:]) * 1e3
    print(f"cfg{cfg} n={n} chunks={os.environ.get('TSNET_HOST_CHUNKS', 'default')}  H2D Y {h2d1:.3f} ms "
          f"({b / h2d1 / 1e6:.1f} GB/s)  H2D Y,V,G {h2d3:.3f}  D2H Y,V,G {d2h3:.3f} ({3 * b / d2h3 / 1e6:.1f} GB/s)  "
          f"device step {dev:.3f}  step_host mean {ts.mean():.3f} min {ts.min():.3f} max {ts.max():.3f} ms",
          flush=True)


if __name__ == "__main__":
    main()
