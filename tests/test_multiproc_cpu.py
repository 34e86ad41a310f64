"""N > 1 host logic on CPU: two processes over torch.distributed `gloo`.

What runs here without a GPU:
  * the row shards (tsnet_shard_rows, libtsnet host code) agree on every rank
    and tile [0, n);
  * the NCCL id travels from rank 0 to the others (distributed.share_comm_id,
    the code ShardedLayout uses);
  * the communication schedule of a sharded iteration (SURVEY.md §8(e),
    DESIGN.md §9), executed with the oracle's arithmetic: geometry from the
    replicated Y, spread of the own points, all-reduce (sum) of the charge
    grids, replicated convolution and Z from the grid, gradient + move of the
    own rows, all-gather of Y -- reproduces the unsharded oracle iteration.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def sharded_oracle_step(Y, P, bounds, rank, world, lam, mu, dist):
    """One iteration in the sharded schedule, oracle arithmetic (test infrastructure)."""
    from oracle import interp
    from oracle import attr_sparse_rows, update_step
    lkl, lc, lr = lam
    n = Y.shape[0]
    rb, re = int(bounds[rank]), int(bounds[rank + 1])
    geo = interp.geometry(Y)                                   # replicated Y -> same grid everywhere
    it = interp._Interp(Y[rb:re], geo)
    delta = geo["delta"]
    cx = geo["lo_x"] + geo["N"] * delta / 2.0
    cy = geo["lo_y"] + geo["N"] * delta / 2.0
    Yr = Y[rb:re]
    xt, yt = Yr[:, 0] - cx, Yr[:, 1] - cy
    import torch
    W = torch.from_numpy(np.stack([it.spread(np.ones(re - rb)), it.spread(xt), it.spread(yt)]))
    dist.all_reduce(W)                                         # the charge-grid all-reduce (live N x N cells)
    W1, Wx, Wy = W.numpy()
    tab = lambda kern: (lambda dx, dy: kern(dx * dx + dy * dy))  # noqa: E731
    Z = float((W1 * interp.convolve(W1, tab(interp.k1), delta)).sum()) - n   # grid dot, replicated

    def pair_sum(kern):
        f1, fx, fy = (it.gather(interp.convolve(Wc, tab(kern), delta)) for Wc in (W1, Wx, Wy))
        return np.stack([xt * f1 - fx, yt * f1 - fy], axis=1)

    F_rep = pair_sum(interp.k2) / Z
    g_ent = -pair_sum(interp.ke_factory(0.05)) / (float(n) * float(n))
    F_attr = attr_sparse_rows(Y, P["indptr"], P["indices"], P["values"], rb, re - rb)
    g = 4.0 * lkl * (F_attr - F_rep) + (lc / n) * Yr + lr * g_ent
    vel, gains = np.zeros_like(Yr), np.ones_like(Yr)
    Yn, _, _ = update_step(Yr, vel, gains, g, eta=50.0, mu=mu)
    # the Y all-gather as libtsnet does it (comm.cu): own rows padded to an equal
    # slice of max_r(rows_r), one all-gather, each rank's valid rows back by bounds
    slice_ = int(max(bounds[r + 1] - bounds[r] for r in range(world)))
    stage = torch.zeros((slice_, 2), dtype=torch.float64)
    stage[:re - rb] = torch.from_numpy(Yn)
    parts = [torch.empty_like(stage) for _ in range(world)]
    dist.all_gather(parts, stage)
    out = np.empty_like(Y)
    for r in range(world):
        a, b = int(bounds[r]), int(bounds[r + 1])
        out[a:b] = parts[r][:b - a].numpy()
    return out


def worker(rank, world, port, errq):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_2509_19785_b200.distributed import shard_bounds, share_comm_id
        from workloads import clustered_layout, config_graph

        ip, ix = config_graph(1)
        P = oracle.build_P(ip, ix, 40.0, seed=0)
        P["values"] = P["values"].astype(np.float32).astype(np.float64)
        n = P["n"]
        bounds = shard_bounds(P["indptr"], world)
        allb = [None] * world
        dist.all_gather_object(allb, bounds.tolist())
        assert all(b == allb[0] for b in allb)
        assert bounds[0] == 0 and bounds[-1] == n and np.all(np.diff(bounds) >= 0)
        uid = share_comm_id(rank)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert len(uid) == 128 and all(u == ids[0] for u in ids)
        Y = clustered_layout(n, 20.0, 5, 1.5, 7).astype(np.float64)
        for lam, mu in (((1.0, 1.2, 0.0), 0.5), ((1.0, 0.01, 0.6), 0.8)):
            got = sharded_oracle_step(Y, P, bounds, rank, world, lam, mu, dist)
            r = oracle.interp_gradient(Y, P["indptr"], P["indices"], P["values"], *lam)
            want, _, _ = oracle.update_step(Y, np.zeros_like(Y), np.ones_like(Y), r["g"], eta=50.0, mu=mu)
            err = np.linalg.norm(got - want) / np.linalg.norm(want)
            assert err <= 1e-12, err
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback
        errq.put((rank, traceback.format_exc()))
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_schedule_gloo(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
