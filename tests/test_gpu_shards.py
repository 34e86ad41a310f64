"""Sharded iteration on one GPU.

Only one GPU is available to the tests, so the ranks are emulated the way the
profiling guide prescribes (no kernels that wait on each other): G virtual
shards run tsnet_field_local one after the other, their live charge grids are
summed by tsnet_grids_sum (the reduction of the peer all-reduce, over pointers
on one device), tsnet_step_finish runs per shard on its own replicated copy of
Y, and the own rows are assembled (the all-gather).  The result must equal the
unsharded tsnet_step (same arithmetic up to fp32 summation order) and the
oracle's step.  The communicator itself runs with one rank through tsnet_step:
the peer all-reduce's publish / flag handshake / reduce kernels (1 peer), the
NCCL all-gather path, eagerly and in a captured CUDA graph.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2509_19785_b200 import CSR, GradParams, StepParams, alloc_workspace, tsnet_step
from paper_2509_19785_b200 import tsnet as T
from workloads import clustered_layout, config_graph, random_state

pytestmark = pytest.mark.gpu


def relL2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


_P = {}


def oracle_P(cfg):
    if cfg not in _P:
        ip, ix = config_graph(cfg)
        _P[cfg] = oracle.build_P(ip, ix, 40.0, seed=0)
    return _P[cfg]


def dev(P):
    return CSR(torch.from_numpy(P["indptr"]).cuda(), torch.from_numpy(P["indices"]).cuda(),
               torch.from_numpy(P["values"].astype(np.float32)).cuda())


def with_plan(P, plan, shard=None):
    """P without a plan ("csr"), or with its column-blocked ("cb") / sliced-ELL ("sell") plan."""
    Q = P.without_plan()
    if plan == "cb":
        return T.tsnet_plan_build(Q, shard)
    if plan == "sell":
        return T.tsnet_sell_build(Q, shard)
    return Q


def emulated_step(P, Y, vel, gains, gp, sp, world, plan="cb"):
    n = P.n
    bounds = T.tsnet_shard_rows(P.indptr.cpu().numpy(), world)
    shards = [T.Shard(r, world, bounds) for r in range(world)]
    Ps, wss, Ys = [], [], []
    for sh in shards:
        Pr = with_plan(P, plan, sh)
        ws = alloc_workspace(n, P.nnz, gp)
        Yr = Y.clone()
        T.tsnet_field_local(Pr, Yr, gp, ws, shard=sh)
        Ps.append(Pr), wss.append(ws), Ys.append(Yr)
    T.tsnet_grids_sum(wss, n, P.nnz, gp)                 # the all-reduce (live N x N cells)
    Yout, Vout, Gout = Y.clone(), vel.clone(), gains.clone()
    for sh, Pr, ws, Yr in zip(shards, Ps, wss, Ys):
        V, G = vel.clone(), gains.clone()
        T.tsnet_step_finish(Pr, Yr, V, G, gp, sp, ws, shard=sh)
        a, b = sh.row_begin, sh.row_end                 # the all-gather of the own rows
        Yout[a:b], Vout[a:b], Gout[a:b] = Yr[a:b], V[a:b], G[a:b]
    torch.cuda.synchronize()
    return Yout, Vout, Gout, bounds


@pytest.mark.parametrize("plan", ["csr", "cb", "sell"])
@pytest.mark.parametrize("cfg,world", [(1, 2), (2, 3), (2, 8), (3, 4)])
@pytest.mark.parametrize("stage", [0, 1])
def test_emulated_shards_equal_one_gpu_and_oracle(cfg, world, stage, plan):
    P = oracle_P(cfg)
    n = P["n"]
    Y = clustered_layout(n, 20.0, 5, 1.5, 7)
    vel, gains = random_state(n, 3)
    lam = ((1.0, 1.2, 0.0), 0.5) if stage == 0 else ((1.0, 0.01, 0.6), 0.8)
    gp, sp = GradParams(*lam[0]), StepParams(eta=50.0, momentum=lam[1])
    Pd = dev(P)
    Yd, Vd, Gd = (torch.from_numpy(a.copy()).cuda() for a in (Y, vel, gains))
    Ys, Vs, Gs, bounds = emulated_step(Pd, Yd, Vd, Gd, gp, sp, world, plan)
    assert len(bounds) == world + 1 and bounds[0] == 0 and bounds[-1] == n
    # unsharded, same attractive kernel
    P1 = with_plan(Pd, plan)
    ws = alloc_workspace(n, Pd.nnz, gp)
    Y1, V1, G1 = Yd.clone(), Vd.clone(), Gd.clone()
    tsnet_step(P1, Y1, V1, G1, gp, sp, ws)
    torch.cuda.synchronize()
    assert relL2(Vs.cpu().numpy(), V1.cpu().numpy()) <= 1e-5
    assert relL2(Ys.cpu().numpy(), Y1.cpu().numpy()) <= 1e-6
    # oracle
    r = oracle.interp_gradient(Y.astype(np.float64), P["indptr"], P["indices"],
                               P["values"].astype(np.float32).astype(np.float64), *lam[0])
    _, Vo, _ = oracle.update_step(Y, vel, gains, r["g"], eta=50.0, mu=lam[1])
    assert relL2(Vs.cpu().numpy(), Vo) <= 1e-4


def test_nccl_one_rank_communicator_step():
    """tsnet_step with a real (1-rank) NCCL communicator: grid all-reduce and Y
    all-gather run through NCCL, also inside a captured CUDA graph."""
    P = oracle_P(2)
    n = P["n"]
    Y = clustered_layout(n, 20.0, 5, 1.5, 7)
    vel, gains = random_state(n, 3)
    gp, sp = GradParams(1.0, 0.01, 0.6), StepParams(eta=50.0, momentum=0.8)
    Pd = dev(P)
    uid = T.tsnet_comm_unique_id()
    comm = T.tsnet_comm_init(uid, 1, 0, gp.I_max)
    try:
        assert T.tsnet_comm_peer_reduce(comm)      # one rank: its own exchange buffer, peer path
        sh = T.Shard(0, 1, [0, n], comm)
        ws = alloc_workspace(n, Pd.nnz, gp)
        Yd, Vd, Gd = (torch.from_numpy(a.copy()).cuda() for a in (Y, vel, gains))
        Y1, V1, G1 = Yd.clone(), Vd.clone(), Gd.clone()
        tsnet_step(Pd, Yd, Vd, Gd, gp, sp, ws, shard=sh)
        tsnet_step(Pd, Y1, V1, G1, gp, sp, alloc_workspace(n, Pd.nnz, gp))
        torch.cuda.synchronize()
        assert relL2(Vd.cpu().numpy(), V1.cpu().numpy()) <= 1e-6
        # graph capture of the communicating step
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            tsnet_step(Pd, Yd, Vd, Gd, gp, sp, ws, shard=sh, stream=s)
        with torch.cuda.stream(s):
            g.replay()
        tsnet_step(Pd, Y1, V1, G1, gp, sp, alloc_workspace(n, Pd.nnz, gp))
        torch.cuda.synchronize()
        assert relL2(Vd.cpu().numpy(), V1.cpu().numpy()) <= 1e-5
        # several replays: the iteration counter and the grid parity advance on the device
        for _ in range(3):
            with torch.cuda.stream(s):
                g.replay()
            tsnet_step(Pd, Y1, V1, G1, gp, sp, alloc_workspace(n, Pd.nnz, gp))
        torch.cuda.synchronize()
        assert relL2(Yd.cpu().numpy(), Y1.cpu().numpy()) <= 1e-5
    finally:
        T.tsnet_comm_destroy(comm)


def test_shard_argument_errors():
    P = oracle_P(1)
    n = P["n"]
    gp, sp = GradParams(), StepParams()
    ws = alloc_workspace(n, P["indptr"][-1], gp)
    Yd = torch.zeros((n, 2), device="cuda")
    V, G = torch.zeros_like(Yd), torch.ones_like(Yd)
    Pp = T.tsnet_plan_build(dev(P), T.Shard(0, 2, [0, n // 2, n]))
    with pytest.raises(T.TsnetError):      # world > 1 without a communicator
        tsnet_step(Pp, Yd, V, G, gp, sp, ws, shard=T.Shard(0, 2, [0, n // 2, n]))
    with pytest.raises(T.TsnetError):      # recentring across ranks
        T.tsnet_step_finish(Pp, Yd, V, G, gp, StepParams(recenter=1), ws, shard=T.Shard(0, 2, [0, n // 2, n]))


def test_layout_push_one_rank_communicator():
    """The fused move + Y push (tsnet_comm_layout): with a 1-rank communicator
    the step on the communicator's own layout buffer takes the push path (its
    read-done / moved handshake, the move's last-block ticket and iteration
    counter), eagerly, in a captured CUDA graph and over several replays, and
    equals the unsharded step; tsnet_comm_layout_sync waits on the counters."""
    P = oracle_P(2)
    n = P["n"]
    Y = clustered_layout(n, 20.0, 5, 1.5, 7)
    vel, gains = random_state(n, 3)
    gp, sp = GradParams(1.0, 0.01, 0.6), StepParams(eta=50.0, momentum=0.8)
    Pd = dev(P)
    comm = T.tsnet_comm_init(T.tsnet_comm_unique_id(), 1, 0, gp.I_max)
    try:
        Yc = T.tsnet_comm_layout(comm, n)
        assert T.tsnet_comm_layout_push(comm)
        assert T.tsnet_comm_layout(comm, n).data_ptr() == Yc.data_ptr()
        with pytest.raises(T.TsnetError):
            T.tsnet_comm_layout(comm, n + 1)
        Yc.copy_(torch.from_numpy(Y))
        sh = T.Shard(0, 1, [0, n], comm)
        ws = alloc_workspace(n, Pd.nnz, gp)
        Vd, Gd = (torch.from_numpy(a.copy()).cuda() for a in (vel, gains))
        Y1, V1, G1 = (torch.from_numpy(a.copy()).cuda() for a in (Y, vel, gains))
        ws1 = alloc_workspace(n, Pd.nnz, gp)
        tsnet_step(Pd, Yc, Vd, Gd, gp, sp, ws, shard=sh)
        tsnet_step(Pd, Y1, V1, G1, gp, sp, ws1)
        T.tsnet_comm_layout_sync(comm)
        torch.cuda.synchronize()
        assert relL2(Yc.cpu().numpy(), Y1.cpu().numpy()) <= 1e-6
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            tsnet_step(Pd, Yc, Vd, Gd, gp, sp, ws, shard=sh, stream=s)
        for _ in range(4):
            with torch.cuda.stream(s):
                g.replay()
            tsnet_step(Pd, Y1, V1, G1, gp, sp, ws1)
        T.tsnet_comm_layout_sync(comm, stream=s)
        torch.cuda.synchronize()
        assert relL2(Yc.cpu().numpy(), Y1.cpu().numpy()) <= 1e-5
        assert relL2(Vd.cpu().numpy(), V1.cpu().numpy()) <= 1e-5
        # another Y than the communicator's: the all-gather path
        Y2 = Yc.clone()
        tsnet_step(Pd, Y2, Vd.clone(), Gd.clone(), gp, sp, alloc_workspace(n, Pd.nnz, gp), shard=sh)
        torch.cuda.synchronize()
    finally:
        T.tsnet_comm_destroy(comm)
