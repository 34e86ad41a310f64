"""Multi-GPU L-tsNET iterations: one process per GPU.

Rank r owns the contiguous rows bounds[r]:bounds[r+1] of P (nnz + rows
balanced, tsnet_shard_rows), holds the full replicated layout Y, and runs
tsnet_step with its shard: geometry from the full Y, spread of its own points,
NCCL all-reduce of the charge grid, replicated FFT convolution, attractive
SpMV + gather + move of its own rows, exchange of Y.  The NCCL
communicator is created inside libtsnet (tsnet_comm_init); torch.distributed
only carries its 128-byte id from rank 0 to the others.  The charge-grid sum is
a peer-memory all-reduce of the live grid (tsnet_comm_init maps every peer's
exchange buffer).  Y lives in the communicator's own IPC-shared buffer
(tsnet_comm_layout) when every peer can map it: the move then stores the new
positions straight into every rank's copy over NVLink; otherwise Y is
all-gathered in equal padded slices.
"""
from __future__ import annotations

import torch

from .runner import STAGE_SWITCH, stage_of, stage_params
from .tsnet import (CSR, GradParams, Shard, attach_plan, alloc_workspace, tsnet_comm_destroy, tsnet_comm_init,
                    tsnet_comm_layout, tsnet_comm_layout_push, tsnet_comm_layout_sync, tsnet_comm_unique_id,
                    tsnet_read_stats, tsnet_shard_rows, tsnet_step)


def shard_bounds(indptr_host, world: int):
    """Row bounds of the `world` shards (host; identical on every rank)."""
    return tsnet_shard_rows(indptr_host, world)


def share_comm_id(rank: int, group=None) -> bytes:
    """NCCL unique id made on rank 0 and broadcast over torch.distributed."""
    import torch.distributed as dist
    obj = [tsnet_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class ShardedLayout:
    """Sharded counterpart of runner.Layout (same schedule, same state layout:
    Y, vel, gains are full n x 2 tensors; vel/gains are only meaningful on the
    own rows)."""

    def __init__(self, P: CSR, Y0: torch.Tensor, rank: int, world: int, base: GradParams | None = None,
                 use_graphs: bool = True, eta: float = 50.0, stage_switch: int = STAGE_SWITCH, group=None,
                 plan: bool | str = False):
        assert Y0.is_cuda and Y0.shape == (P.n, 2)
        self.rank, self.world = rank, world
        bounds = shard_bounds(P.indptr.cpu().numpy(), world)
        uid = share_comm_id(rank, group)
        self.params = [stage_params(0, base, eta), stage_params(1, base, eta)]
        self.comm = tsnet_comm_init(uid, world, rank, self.params[0][0].I_max)
        self.shard = Shard(rank, world, bounds, self.comm)
        self.stream = torch.cuda.Stream(device=Y0.device)
        self.stream.wait_stream(torch.cuda.current_stream(Y0.device))
        # the attractive SpMV reads the own rows of P (CSR), or a plan of them
        # (attach_plan: "csr", "cb", "sell", "auto"; or a callable
        # (P, shard, stream) -> P with a plan, e.g. bench.choose_plan) attached
        # to a shallow copy, so the caller's P keeps its own plan
        if callable(plan):
            self.P = plan(P.without_plan(), self.shard, self.stream)
        else:
            self.P = attach_plan(P.without_plan(), plan, self.shard)
        # the replicated layout: the communicator's buffer when the move can push
        # into every peer's copy (collective call on every rank), else a tensor
        # of our own and the all-gather
        Yc = tsnet_comm_layout(self.comm, P.n, device=Y0.device)
        self.push = tsnet_comm_layout_push(self.comm)
        if self.push:
            self.Y = Yc
            with torch.cuda.stream(self.stream):
                self.Y.copy_(Y0)
        else:
            self.Y = Y0.clone()
        self.vel = torch.zeros_like(Y0)
        self.gains = torch.ones_like(Y0)
        self.ws = alloc_workspace(P.n, P.nnz, self.params[0][0], device=Y0.device)
        self.stage_switch = stage_switch
        self.use_graphs = use_graphs
        self.graphs = [None, None]

    @property
    def rows(self):
        return self.shard.row_begin, self.shard.row_end

    def _raw_step(self, stage: int):
        gp, sp = self.params[stage]
        tsnet_step(self.P, self.Y, self.vel, self.gains, gp, sp, self.ws, shard=self.shard, stream=self.stream)

    def _graph(self, stage: int):
        if self.graphs[stage] is None:
            # capture without advancing the state (snapshot/restore on self.stream);
            # every rank captures at the same iteration, so the collectives match
            with torch.cuda.stream(self.stream):
                self._layout_sync()
                saved = (self.Y.clone(), self.vel.clone(), self.gains.clone())
                self._raw_step(stage)
            self.stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                self._raw_step(stage)
            with torch.cuda.stream(self.stream):
                self._layout_sync()          # every peer's push of the eager step has landed
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

    def _layout_sync(self):
        if self.push and self.comm:
            tsnet_comm_layout_sync(self.comm, self.stream)

    def sync(self):
        """Wait for this rank's work and, with the layout push, for every peer's
        moves into this rank's Y (so Y is complete when read)."""
        self._layout_sync()
        self.stream.synchronize()

    def stats(self):
        self.sync()
        return tsnet_read_stats(self.ws, stream=self.stream)

    def close(self):
        self.sync()
        self.graphs = [None, None]
        if self.push:
            self.Y = self.Y.clone()    # the communicator's buffer is freed with it
            self.push = False
        if self.comm:
            tsnet_comm_destroy(self.comm)
            self.comm = None
