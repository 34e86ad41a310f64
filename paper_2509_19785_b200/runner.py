"""L-tsNET iteration driver over the C-ABI (Alg. 3 main loop).

Holds the device state (Y, velocity, gains), the workspace and P, applies the
two-stage multiplier schedule of reading R12/O7 (the paper only
says multipliers change "in different stages") and replays one
captured CUDA graph per stage so the ~12 kernels of an iteration launch as one
graph (launch-latency-bound at small n).
"""
from __future__ import annotations

import torch

from .tsnet import CSR, GradParams, StepParams, alloc_workspace, tsnet_read_stats, tsnet_step

STAGE_SWITCH = 250


def stage_of(it: int, stage_switch: int = STAGE_SWITCH) -> int:
    return 0 if it < stage_switch else 1


def stage_params(stage: int, base: GradParams | None = None, eta: float = 50.0):
    """O7: stage A (lkl, lc, lr) = (1, 1.2, 0), momentum 0.5; stage B (1, 0.01, 0.6), momentum 0.8."""
    b = base or GradParams()
    if stage == 0:
        gp = GradParams(1.0, 1.2, 0.0, b.eps, b.interp_P, b.h_max, b.I_min, b.I_max, b.spread)
        sp = StepParams(eta=eta, momentum=0.5)
    else:
        gp = GradParams(1.0, 0.01, 0.6, b.eps, b.interp_P, b.h_max, b.I_min, b.I_max, b.spread)
        sp = StepParams(eta=eta, momentum=0.8)
    return gp, sp


class Layout:
    def __init__(self, P: CSR, Y0: torch.Tensor, base: GradParams | None = None, use_graphs: bool = True,
                 eta: float = 50.0, stage_switch: int = STAGE_SWITCH, stream: torch.cuda.Stream | None = None):
        assert Y0.is_cuda and Y0.dtype == torch.float32 and Y0.shape == (P.n, 2)
        self.P = P
        self.Y = Y0.clone()
        self.vel = torch.zeros_like(self.Y)
        self.gains = torch.ones_like(self.Y)
        self.params = [stage_params(0, base, eta), stage_params(1, base, eta)]
        self.ws = alloc_workspace(P.n, P.nnz, self.params[0][0], device=Y0.device)
        self.stage_switch = stage_switch
        self.use_graphs = use_graphs
        self.stream = stream or torch.cuda.Stream(device=Y0.device)
        # the state above was written on the caller's stream; every later step runs on self.stream
        self.stream.wait_stream(torch.cuda.current_stream(Y0.device))
        self.graphs = [None, None]

    def _raw_step(self, stage: int):
        gp, sp = self.params[stage]
        tsnet_step(self.P, self.Y, self.vel, self.gains, gp, sp, self.ws, stream=self.stream)

    def _graph(self, stage: int):
        if self.graphs[stage] is None:
            # warm-up outside capture, then restore the state so the captured
            # iteration does not advance the real layout.  Snapshot and restore run
            # on self.stream, ordered after every step already enqueued there.
            with torch.cuda.stream(self.stream):
                saved = (self.Y.clone(), self.vel.clone(), self.gains.clone())
                self._raw_step(stage)
            self.stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                self._raw_step(stage)
            with torch.cuda.stream(self.stream):
                self.Y.copy_(saved[0])
                self.vel.copy_(saved[1])
                self.gains.copy_(saved[2])
            self.stream.synchronize()
            self.graphs[stage] = g
        return self.graphs[stage]

    def step(self, it: int):
        stage = stage_of(it, self.stage_switch)
        if self.use_graphs:
            g = self._graph(stage)
            with torch.cuda.stream(self.stream):
                g.replay()
        else:
            with torch.cuda.stream(self.stream):
                self._raw_step(stage)

    def run(self, iters: int, start: int = 0):
        for it in range(start, start + iters):
            self.step(it)
        return self

    def sync(self):
        self.stream.synchronize()

    def stats(self):
        self.sync()
        return tsnet_read_stats(self.ws, stream=self.stream)
