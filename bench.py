#!/usr/bin/env python
"""bench.py -- tsNET gradient iterations/s on B200 (BASELINE.json `metric`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

A step is one L-tsNET iteration (Alg. 3 l.396-405) over the
whole workload: box sort + spread + FFT convolution + attractive SpMV + gather
+ momentum/gains move, all in libtsnet's CUDA kernels (one CUDA graph replay).
Default workload: BASELINE.json configs[3], Chung-Lu n = 1e6 (LCC), u = 40,
with P built on the GPU (C0, untimed); 250 stage-A iterations run untimed
first so the timed window sits in stage B (all terms active, steady grid).

One JSON line on rank 0.  `roofline` is for the dominant kernel (the
attractive SpMV, timed alone with CUDA events on its stream); `cpu_baseline`
is the fp64 oracle (test infrastructure) timed on this host on a bounded
sample; `e2e` is the same metric through tsnet_step_host with host buffers.
`--impl reference` times the oracle (the reference arm of this tier) instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "tsNET gradient iterations/sec at n=1M (1/2/4/8 B200); % of HBM roofline"
UNIT = "iterations/s"
KERNELS_PER_STEP = 11   # kernels tsnet_step launches: field.cu 8 (bbox, the box sort's 3, which exit at
                        # once on the runs path, the run pass, 3 FFT passes), attractive SpMV 1, the move 2
                        # (the shared-memory and the L1 variant; the one not matching the grid size exits at once)
CONFIG_DESC = {
    1: "cfg1 2-D grid 32x32 (n=1024), u=40",
    2: "cfg2 RGG n=20,000 mean degree 8 (LCC), u=40",
    3: "cfg3 SBM 50x4000 intra 10 / inter 1 (LCC), u=40",
    4: "cfg4 Chung-Lu n=1,000,000 gamma=2.5 mean degree 6 (LCC), u=40",
    5: "cfg5 3-D grid 160^3 (n=4,096,000), u=40",
}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons every 100 ms with a timestamp per
    sample; start() well before the timed region (nvidia-smi needs ~1 s to
    produce its first line), stop(t0, t1) keeps the samples taken inside the
    timed wall-clock window [t0, t1] (widened to the nearest samples when the
    window is shorter than the sampling period)."""
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        if self.proc is not None:
            import atexit
            atexit.register(self._kill)      # never leave the sampler running (error paths)

    def _kill(self):
        if self.proc is not None and self.proc.poll() is None:
            self.proc.kill()

    def stop(self, t0: float | None = None, t1: float | None = None):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        import datetime
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        with open(self.path) as f:
            for ln in f:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                    rows.append((ts, float(parts[1]), float(parts[2]),
                                 {nm for nm, v in zip(names, parts[5:9]) if v.lower().startswith("active")}))
                except ValueError:
                    continue
        os.unlink(self.path)
        if t0 is not None and t1 is not None and rows:
            inside = [r for r in rows if t0 <= r[0] <= t1]
            if not inside:                      # window shorter than the period: the nearest samples
                inside = sorted(rows, key=lambda r: min(abs(r[0] - t0), abs(r[0] - t1)))[:2]
            rows = inside
        sm = [r[1] for r in rows]
        reasons = set().union(*[r[3] for r in rows]) if rows else set()
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(r[2] for r in rows) if rows else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------- CPU legs
def oracle_P(cfg: int):
    """Oracle C0 for the workload (untimed)."""
    import oracle
    from workloads import config_graph
    ip, ix = config_graph(cfg)
    t0 = time.perf_counter()
    P = oracle.build_P(ip, ix, 40.0, seed=0)
    return P, time.perf_counter() - t0


def oracle_stepper(P, Y):
    """Full oracle iterations (O5 interpolation gradient + O6 move, stage-B
    multipliers and momentum, fp64) from the layout Y with v = 0, gains = 1."""
    import oracle
    state = {"Y": np.asarray(Y, np.float64).copy(), "vel": np.zeros((P["n"], 2)), "gains": np.ones((P["n"], 2))}

    def step():
        g = oracle.interp_gradient(state["Y"], P["indptr"], P["indices"], P["values"], 1.0, 0.01, 0.6)["g"]
        state["Y"], state["vel"], state["gains"] = oracle.update_step(state["Y"], state["vel"], state["gains"], g,
                                                                      eta=50.0, mu=0.8)
    return step


def cpu_baseline(cfg: int, Y, where: str, budget_s: float = 12.0):
    """The oracle as it stands, on the GPU arm's own layout (bounded sample)."""
    P, setup_s = oracle_P(cfg)
    step = oracle_stepper(P, Y)
    step()                                  # warm-up iteration
    t0 = time.perf_counter()
    iters = 0
    while True:
        step()
        iters += 1
        el = time.perf_counter() - t0
        if el >= budget_s or iters >= 50:
            break
    return {"value": iters / el, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"{iters} full O5 iterations (fp64 interpolation gradient + O6 move, stage-B multipliers) "
                      f"of the {CONFIG_DESC[cfg]} workload (n={P['n']}, nnz={len(P['values'])}) from the GPU arm's "
                      f"own layout {where}; OpenMP C parts on all {os.cpu_count()} host threads, numpy parts 1 "
                      f"thread; oracle C0 set-up {setup_s:.0f}s untimed"}


REF_SPAN = 8.0     # synthetic stage-B-like layout of the reference arm (GPU windows span 0.5-13 on cfg 4)


def run_reference(args, rank):
    """The reference arm of this tier: the oracle, whole O5 iterations (the
    layout-wide field step included in every step)."""
    if rank != 0:
        return
    from workloads import clustered_layout
    P, setup_s = oracle_P(args.config)
    n = P["n"]
    Y = clustered_layout(n, REF_SPAN, 40, REF_SPAN / 15.0, 5)
    step = oracle_stepper(P, Y)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    value = args.steps / el
    sample = (f"each step = one full fp64 oracle O5 iteration (field + gradient + move, stage-B multipliers) of the "
              f"{CONFIG_DESC[args.config]} workload (n={n}) from a synthetic clustered layout of span {REF_SPAN} "
              f"(the span of the GPU arm's stage-B windows); OpenMP C parts on all {os.cpu_count()} host threads; "
              f"oracle C0 set-up {setup_s:.0f}s untimed")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(args.config, n, len(P["values"])),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(cfg, n, nnz):
    """The workload (identical on both arms; run-specific figures go to "run")."""
    return {"workload": CONFIG_DESC[cfg], "n": int(n), "nnz": int(nnz), "perplexity": 40,
            "window": "stage B (iterations 250-999; lambda = (1, 0.01, 0.6), momentum 0.8, eta 50)",
            "l2": "inputs larger than L2 (CSR >> 126 MB)" if 8 * nnz > 126e6 else "CSR fits in L2 (small config)"}


# -------------------------------------------------------------- our arm
N_WINDOWS = 5       # the paper averages 5 runs; here 5 timed windows over stage B
STAGE_B_END = 1000  # configs 3-5 run 1000 iterations (BASELINE.json)


def window_starts(pre: int, warmup: int, steps: int):
    """Start iterations of the timed windows: N_WINDOWS windows of `steps`
    iterations spread evenly over stage B (after the warm-up), or as many as fit."""
    first = pre + warmup
    avail = STAGE_B_END - first
    nwin = max(1, min(N_WINDOWS, avail // max(steps, 1)))
    if nwin == 1:
        return [first]
    stride = (avail - steps) // (nwin - 1)
    return [first + i * stride for i in range(nwin)]


def choose_plan(P, shard, stream):
    """attach_plan("auto") plus a measured choice between the row-wise CSR kernel
    and the column-blocked plan where the sliced ELL pads too much: a few
    launches of each on a synthetic layout (set-up, untimed)."""
    import torch
    from paper_2509_19785_b200 import attach_plan, tsnet_attr
    from paper_2509_19785_b200.tsnet import PLAN_SELL, tsnet_plan_build
    Q = attach_plan(P, "auto", shard, stream)
    if Q.plan is not None and Q.plan_kind == PLAN_SELL:
        return Q, {"choice": "sliced ELL (pads <= 1.3 slots per entry)"}
    Y = torch.randn((P.n, 2), device=P.indptr.device) * 3.0
    F = tsnet_attr(Q, Y, shard=shard, stream=stream)      # this rank's rows

    def t(Pk):
        for _ in range(2):
            tsnet_attr(Pk, Y, F, shard=shard, stream=stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            tsnet_attr(Pk, Y, F, shard=shard, stream=stream)
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / 5
    t_csr = t(Q)
    C = tsnet_plan_build(P.without_plan(), shard, stream)
    t_cb = t(C)
    if t_cb < t_csr:
        return C, {"choice": "column-blocked plan", "csr_ms": t_csr, "cb_ms": t_cb}
    del C
    return Q, {"choice": "CSR", "csr_ms": t_csr, "cb_ms": t_cb}


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2509_19785_b200 import Layout, attach_plan, tsnet_attr, tsnet_build_P, tsnet_read_stats, tsnet_step_host
    from paper_2509_19785_b200.tsnet import PLAN_CB, PLAN_SELL
    from workloads import config_graph, init_layout

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    clocks = ClockSampler(local_rank)          # started early: nvidia-smi's first sample takes ~1 s
    clocks.start()
    ip, ix = config_graph(args.config)
    t0 = time.perf_counter()
    built = tsnet_build_P(torch.from_numpy(ip).to(dev), torch.from_numpy(ix).to(dev), u=40.0, seed=0)
    torch.cuda.synchronize()
    c0_s = time.perf_counter() - t0
    P = built["P"]
    n, nnz = P.n, P.nnz
    Y0 = torch.from_numpy(init_layout(n, 0)).to(dev)
    t0 = time.perf_counter()
    plan_info = None
    if world > 1 or args.sharded:
        # row shards + NCCL communicator (+ the plan of the own rows) (set-up, untimed)
        from paper_2509_19785_b200.distributed import ShardedLayout
        if args.plan == "auto":      # the same timed choice as one GPU, on this rank's rows
            def pick(Pc, sh, st):
                nonlocal plan_info
                Pk, plan_info = choose_plan(Pc, sh, st)
                return Pk
            lay = ShardedLayout(P, Y0, rank, world, plan=pick)
        else:
            lay = ShardedLayout(P, Y0, rank, world, plan=args.plan)
        shard = lay.shard
        rb, re = lay.rows
    else:
        setup_stream = torch.cuda.Stream(device=dev)
        if args.plan == "auto":
            Pk, plan_info = choose_plan(P, None, setup_stream)
        else:
            Pk = attach_plan(P.without_plan(), args.plan)
        torch.cuda.synchronize()
        lay = Layout(Pk, Y0, use_graphs=True)
        shard, rb, re = None, 0, n
    torch.cuda.synchronize()
    plan_s = time.perf_counter() - t0
    nnz_l = int(P.indptr[re].item() - P.indptr[rb].item())
    nl = re - rb
    # stage A (untimed for `value`; its rate is reported separately): the first
    # step captures the graph, the rest are replays between events
    lay.run(1, start=0)
    a0 = torch.cuda.Event(enable_timing=True)
    a1 = torch.cuda.Event(enable_timing=True)
    a0.record(lay.stream)
    lay.run(args.pre_iters - 1, start=1)
    a1.record(lay.stream)
    lay.sync()
    stage_a_ms = a0.elapsed_time(a1) / max(1, args.pre_iters - 1)
    it = args.pre_iters
    starts = window_starts(args.pre_iters, args.warmup, args.steps)
    windows = []
    Y_med = None
    med_idx = len(starts) // 2
    w_t0 = w_t1 = None
    for wi, st in enumerate(starts):
        lay.run(st - it, start=it)           # warm-up (first window) / untimed fast-forward
        it = st
        lay.sync()
        g0 = tsnet_read_stats(lay.ws, stream=lay.stream)
        if wi == med_idx and rank == 0 and world == 1:
            Y_med = lay.Y.cpu().numpy().copy()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if w_t0 is None:
            w_t0 = time.time()
        e0.record(lay.stream)
        lay.run(args.steps, start=it)
        e1.record(lay.stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        w_t1 = time.time()
        ms = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        it += args.steps
        g1 = tsnet_read_stats(lay.ws, stream=lay.stream)
        windows.append({"start": st, "ms_per_step": ms / args.steps, "grid_N_start": g0["N"], "grid_N_end": g1["N"],
                        "span_start": round(g0["S"], 3), "span_end": round(g1["S"], 3),
                        "nonfinite": g1["nonfinite"]})
    clk = clocks.stop(w_t0, w_t1)
    order = sorted(range(len(windows)), key=lambda i: windows[i]["ms_per_step"])
    mid = windows[order[len(order) // 2]]
    step_ms = mid["ms_per_step"]
    Ns = [w[k] for w in windows for k in ("grid_N_start", "grid_N_end")]

    # dominant kernel: the attractive SpMV alone (own rows), CUDA events on its stream
    Pk = lay.P
    reps = max(10, min(args.steps, 200))
    fa = torch.empty((nl, 2), dtype=torch.float32, device=dev)
    with torch.cuda.stream(lay.stream):
        for _ in range(3):
            tsnet_attr(Pk, lay.Y, fa, shard=shard, stream=lay.stream)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(lay.stream)
        for _ in range(reps):
            tsnet_attr(Pk, lay.Y, fa, shard=shard, stream=lay.stream)
        s1.record(lay.stream)
    torch.cuda.synchronize()
    spmv_ms = s0.elapsed_time(s1) / reps
    peak, peak_src = measured_peak()
    spmv_bytes = 8 * nnz_l + 8 * (nl + 1) + 16 * nl        # col+val, indptr, Y_i read, F_i write
    achieved = spmv_bytes / (spmv_ms * 1e-3) / 1e9
    # SURVEY §8(d) B_g: CSR + state of the own rows + the all-gather payload landing in HBM
    step_bytes = 8 * nnz_l + 8 * (nl + 1) + 48 * nl + 8 * (n - nl)
    layout = {PLAN_CB: "cb", PLAN_SELL: "sell"}.get(Pk.plan_kind, "csr") if Pk.plan is not None else "csr"
    kname = {"cb": "k_attr_tile", "sell": "k_attr_sell_g"}.get(layout, "k_spmv2")
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"{kname}_dram_bytes_cfg{args.config}.json")
    if os.path.exists(tp) and world == 1:
        with open(tp) as f:
            rec = json.load(f)
        traffic = float(rec["dram_bytes_per_launch"]) * (nnz / rec["nnz"])

    # end to end through the host-buffer API (H2D + step + D2H every step)
    e2e = None
    if not args.no_e2e:
        gp, sp = lay.params[1]
        Yh = lay.Y.cpu().pin_memory()
        Vh = lay.vel.cpu().pin_memory()
        Gh = lay.gains.cpu().pin_memory()
        ne = max(3, min(args.steps, 50))
        tsnet_step_host(Pk, Yh, Vh, Gh, gp, sp, lay.ws, shard=shard, stream=lay.stream)
        if world > 1:
            dist.barrier()
        h0 = time.perf_counter()
        for _ in range(ne):
            tsnet_step_host(Pk, Yh, Vh, Gh, gp, sp, lay.ws, shard=shard, stream=lay.stream)
        h1 = time.perf_counter()
        el = h1 - h0
        if world > 1:
            tt = torch.tensor([el], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            el = float(tt.item())
        e2e = {"value": ne / el, "unit": UNIT, "h2d_bytes_per_step": 24 * n, "d2h_bytes_per_step": 24 * n,
               "steps": ne}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and Y_med is not None:
        cpu = cpu_baseline(args.config, Y_med, f"at iteration {starts[med_idx]} (the median timed window)",
                           args.cpu_budget)

    if rank == 0:
        value = 1e3 / step_ms                  # whole-job iterations/s: every rank takes part in each iteration
        par = ("single GPU" if (world == 1 and not args.sharded) else
               f"{world} row shards (nnz-balanced), NCCL all-reduce of the charge grid + all-gather of Y")
        run = {"windows": windows, "value_from": "median window (ms/step) of the timed windows",
               "grid_N": {"min": min(Ns), "median": float(np.median(Ns)), "max": max(Ns)},
               "pre_iters": args.pre_iters, "stage_a_iters_per_s": round(1e3 / stage_a_ms, 1),
               "c0_gpu_s": round(c0_s, 3), "parallelism": par,
               "attr_layout": {"cb": "column-blocked plan", "sell": "sliced-ELL plan"}.get(layout, "CSR"),
               "plan_choice": plan_info, "plan_build_s": round(plan_s, 3)}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": config_dict(args.config, n, nnz), "run": run,
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic, "kernel": f"{kname} (tsnet_attr)",
                             "kernel_ms": spmv_ms, "algorithmic_bytes": spmv_bytes, "peak_source": peak_src,
                             "share_of_step": spmv_ms / step_ms, "rank": 0},
                "step_roofline": {"achieved": step_bytes / (step_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                                  "frac": step_bytes / (step_ms * 1e-3) / 1e9 / peak, "algorithmic_bytes": step_bytes},
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": KERNELS_PER_STEP * args.steps * len(windows),
                "clocks": clk, "nonfinite": max(w["nonfinite"] for w in windows)}
        print(json.dumps(line), flush=True)
    if world > 1 or args.sharded:
        lay.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--pre-iters", type=int, default=250)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--plan", default="auto", choices=["auto", "csr", "cb", "sell"],
                    help="SpMV layout of P: auto (default: sliced ELL when it pads <= 1.3 slots per entry, else "
                         "the faster of CSR and the column-blocked plan, timed at set-up), csr, cb, sell")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU (NCCL) path even on one rank (needs torchrun / a process group)")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    assert args.warmup >= 3, "at least 3 warm-up steps"

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torch.distributed.run
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1 or args.sharded:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    run_ours(args, rank, world, local_rank)
    if world > 1 or args.sharded:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
