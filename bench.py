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
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "tsNET gradient iterations/sec at n=1M (1/2/4/8 B200); % of HBM roofline"
UNIT = "iterations/s"
KERNELS_PER_STEP = 11   # kernels tsnet_step launches (field.cu 9, attr 1, update 1; recenter off)
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
def oracle_setup(cfg: int):
    """Oracle C0 for the workload (untimed) and a synthetic stage-B-like layout."""
    import oracle
    from workloads import clustered_layout, config_graph
    ip, ix = config_graph(cfg)
    t0 = time.perf_counter()
    P = oracle.build_P(ip, ix, 40.0, seed=0)
    n = P["n"]
    Y = clustered_layout(n, 30.0, 40, 2.0, 5).astype(np.float64)
    return P, Y, time.perf_counter() - t0


def oracle_block_stepper(P, Y, blocks: int):
    """One oracle O5 iteration split into `blocks` bounded steps: step 0 of a
    cycle computes the layout-wide part (geometry, spread, convolutions, Z),
    every step computes gradient + move for one row block (stage-B multipliers).
    `blocks` consecutive steps = exactly one full oracle iteration."""
    import oracle
    from oracle import interp
    n = P["n"]
    bs = (n + blocks - 1) // blocks
    state = {"Y": Y.copy(), "vel": np.zeros_like(Y), "gains": np.ones_like(Y), "Ynext": Y.copy(), "fs": None, "b": 0}

    def step():
        b = state["b"]
        if b == 0:
            state["fs"] = interp.field_state(state["Y"])
        r0 = b * bs
        nr = min(bs, n - r0)
        if nr > 0:
            g = interp.gradient_rows(state["fs"], state["Y"], P["indptr"], P["indices"], P["values"], 1.0, 0.01,
                                     0.6, r0, nr)
            Yn, V, G = oracle.update_step(state["Y"][r0:r0 + nr], state["vel"][r0:r0 + nr],
                                          state["gains"][r0:r0 + nr], g, eta=50.0, mu=0.8)
            state["Ynext"][r0:r0 + nr], state["vel"][r0:r0 + nr], state["gains"][r0:r0 + nr] = Yn, V, G
        state["b"] = b + 1
        if state["b"] == blocks:
            state["b"] = 0
            state["Y"] = state["Ynext"].copy()

    return step


def cpu_baseline(cfg: int, budget_s: float = 12.0):
    P, Y, setup_s = oracle_setup(cfg)
    step = oracle_block_stepper(P, Y, 1)
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
                      f"of the {CONFIG_DESC[cfg]} workload (n={P['n']}, nnz={len(P['values'])}) at a synthetic "
                      f"span-30 layout; OpenMP C parts on all {os.cpu_count()} host threads, numpy parts 1 thread; "
                      f"oracle C0 set-up {setup_s:.0f}s untimed"}


def run_reference(args, rank):
    if rank != 0:
        return
    P, Y, setup_s = oracle_setup(args.config)
    n = P["n"]
    blocks = max(1, (n + 16383) // 16384)
    step = oracle_block_stepper(P, Y, blocks)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    value = (args.steps / blocks) / el
    sample = (f"each step = one {min(16384, n)}-row block of an fp64 oracle O5 iteration (layout-wide spread + "
              f"convolutions once per {blocks} steps); {blocks} steps = 1 iteration of the {CONFIG_DESC[args.config]}"
              f" workload (n={n}); oracle C0 set-up {setup_s:.0f}s untimed")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(args.config, n, len(P["values"]), None),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(cfg, n, nnz, extra):
    d = {"workload": CONFIG_DESC[cfg], "n": int(n), "nnz": int(nnz), "perplexity": 40,
         "window": "stage B (iterations 250+; lambda = (1, 0.01, 0.6), momentum 0.8, eta 50)",
         "l2": "inputs larger than L2 (CSR >> 126 MB)"
         if 8 * nnz > 126e6 else "CSR fits in L2 (small config)"}
    if extra:
        d.update(extra)
    return d


# -------------------------------------------------------------- our arm
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
    plan_s = None
    t0 = time.perf_counter()
    if world > 1 or args.sharded:
        # row shards + NCCL communicator (+ the plan of the own rows) (set-up, untimed)
        from paper_2509_19785_b200.distributed import ShardedLayout
        lay = ShardedLayout(P, Y0, rank, world, plan=args.plan)
        shard = lay.shard
        rb, re = lay.rows
    else:
        attach_plan(P, args.plan)             # SpMV layout of P (set-up, untimed)
        lay = Layout(P, Y0, use_graphs=True)
        shard, rb, re = None, 0, n
    torch.cuda.synchronize()
    if world > 1 or P.plan is not None or args.sharded:
        plan_s = time.perf_counter() - t0
    nnz_l = int(P.indptr[re].item() - P.indptr[rb].item())
    nl = re - rb
    it = 0
    # stage A (untimed for `value`; its rate is reported separately): the first
    # step captures the graph, the rest are replays between events
    stage_a_ms = None
    if args.pre_iters >= 2:
        lay.run(1, start=0)
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(lay.stream)
        lay.run(args.pre_iters - 1, start=1)
        a1.record(lay.stream)
        lay.sync()
        stage_a_ms = a0.elapsed_time(a1) / (args.pre_iters - 1)
    else:
        lay.run(args.pre_iters, start=0)
    it += args.pre_iters
    lay.sync()
    grid_start = tsnet_read_stats(lay.ws, stream=lay.stream)
    lay.run(args.warmup, start=it)
    it += args.warmup
    lay.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    e0.record(lay.stream)
    lay.run(args.steps, start=it)
    e1.record(lay.stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop(w0, time.time())
    ms = e0.elapsed_time(e1)
    it += args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    stats = tsnet_read_stats(lay.ws, stream=lay.stream)

    # dominant kernel: the attractive SpMV alone (own rows), CUDA events on its stream
    Pk = lay.P
    reps = max(10, min(args.steps, 200))
    fa = torch.empty_like(lay.Y)
    with torch.cuda.stream(lay.stream):
        for _ in range(3):
            tsnet_attr(Pk, lay.Y, fa, stream=lay.stream)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(lay.stream)
        for _ in range(reps):
            tsnet_attr(Pk, lay.Y, fa, stream=lay.stream)
        s1.record(lay.stream)
    torch.cuda.synchronize()
    spmv_ms = s0.elapsed_time(s1) / reps
    peak, peak_src = measured_peak()
    spmv_bytes = 8 * nnz_l + 8 * (nl + 1) + 16 * nl        # col+val, indptr, Y_i read, F_i write
    achieved = spmv_bytes / (spmv_ms * 1e-3) / 1e9
    step_ms = ms / args.steps
    # SURVEY §8(d) B_g: CSR + state of the own rows + the all-gather payload landing in HBM
    step_bytes = 8 * nnz_l + 8 * (nl + 1) + 48 * nl + 8 * (n - nl)
    traffic = None
    limiter = None
    layout = {PLAN_CB: "cb", PLAN_SELL: "sell"}.get(lay.P.plan_kind, "csr") if lay.P.plan is not None else "csr"
    kname = {"cb": "k_attr_cb", "sell": "k_attr_sell_g"}.get(layout, "k_spmv2")
    tp = os.path.join(ROOT, "profiles", f"{kname}_dram_bytes_cfg{args.config}.json")
    if os.path.exists(tp) and world == 1:
        with open(tp) as f:
            rec = json.load(f)
        traffic = float(rec["dram_bytes_per_launch"]) * (nnz / rec["nnz"])
        limiter = rec.get("limiter")
        if "l2_request_path_utilization" in rec:
            limiter = {"what": limiter, "l1tex_to_l2_request_path_util": rec["l2_request_path_utilization"],
                       "lts_tag_request_util": rec["lts_tag_request_utilization"], "source": rec["source"]}
    gc = os.path.join(ROOT, "profiles", "gather_ceiling_b200.json")
    if os.path.exists(gc) and layout == "csr":
        with open(gc) as f:
            ceil = float(json.load(f)["global_gathers_per_s"])
        # one Y[j] gather per stored entry; the measured random-gather ceiling bounds the SpMV
        # at nnz / ceiling whatever the HBM bandwidth
        g = {"gathers_per_s": nnz_l / (spmv_ms * 1e-3), "ceiling_gathers_per_s": ceil,
             "frac": nnz_l / (spmv_ms * 1e-3) / ceil, "hbm_frac_at_ceiling": spmv_bytes * ceil / nnz_l / 1e9 / peak,
             "source": "profiles/gather_ceiling_b200.json"}
        limiter = {"what": limiter, "gather_ceiling": g} if not isinstance(limiter, dict) else {**limiter, "gather_ceiling": g}

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
            t = torch.tensor([el], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": ne / el, "unit": UNIT, "h2d_bytes_per_step": 24 * n, "d2h_bytes_per_step": 24 * n,
               "steps": ne}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, args.cpu_budget)

    if rank == 0:
        value = args.steps / (ms * 1e-3)       # whole-job iterations/s: every rank takes part in each iteration
        par = ("single GPU" if (world == 1 and not args.sharded) else
               f"{world} row shards (nnz-balanced), NCCL all-reduce of the charge grid + all-gather of Y")
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": config_dict(args.config, n, nnz,
                                      {"grid_I": stats["I"], "grid_N": stats["N"], "fft_M": stats["M"],
                                       "span": round(stats["S"], 3), "pre_iters": args.pre_iters,
                                       "grid_N_window_start": grid_start["N"], "span_window_start":
                                       round(grid_start["S"], 3), "stage_a_iters_per_s": None if stage_a_ms is None else round(1e3 / stage_a_ms, 1),
                                       "c0_gpu_s": round(c0_s, 3), "parallelism": par,
                                       "attr_layout": {"cb": "column-blocked plan", "sell": "sliced-ELL plan"}.get(
                                           layout, "CSR"),
                                       "plan_build_s": None if plan_s is None else round(plan_s, 3)}),
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic, "kernel": f"{kname} (tsnet_attr)",
                             "kernel_ms": spmv_ms, "algorithmic_bytes": spmv_bytes, "peak_source": peak_src,
                             "share_of_step": spmv_ms / step_ms, "rank": 0, "limiter": limiter},
                "step_roofline": {"achieved": step_bytes / (step_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                                  "frac": step_bytes / (step_ms * 1e-3) / 1e9 / peak, "algorithmic_bytes": step_bytes},
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": KERNELS_PER_STEP * args.steps,
                "clocks": clk, "nonfinite": stats["nonfinite"]}
        print(json.dumps(line), flush=True)
    if world > 1 or args.sharded:
        lay.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--pre-iters", type=int, default=250)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--plan", nargs="?", const="cb", default="auto", choices=["auto", "csr", "cb", "sell"],
                    help="SpMV layout of P: auto (default: sliced ELL when it pads <= 1.6 slots per entry, else "
                         "CSR), csr, cb (column-blocked; a bare --plan), sell (sliced ELL)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU (NCCL) path even on one rank (needs torchrun / a process group)")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    assert args.warmup >= 3, "at least 3 warm-up steps"

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
