"""Attractive SpMV kernels vs the oracle: the column-blocked plan kernel
(attr_cb.cu, tsnet_plan_build), the sliced-ELL plan kernel (attr_sell.cu,
tsnet_sell_build) and the row-wise CSR kernel (iterate.cu, used when P has no
plan).

F_attr,i = sum_j p_ij w_ij (X_i - X_j) (Eq. 6 first term) is
computed by oracle.attr_sparse in fp64 from the same fp32 P and fp32 Y.
Bar: relL2 <= 1e-5 over all rows (fp32 per-entry arithmetic, fp32 sums in
another order), and per row |f - f_oracle| <= 1e-5 * sum_j |p_ij w_ij Delta_ij|
(the row's own term scale), so no row can hide behind the global norm.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2509_19785_b200 import CSR, tsnet_attr
from paper_2509_19785_b200 import tsnet as T
from workloads import clustered_layout, config_graph, random_csr, uniform_layout

pytestmark = pytest.mark.gpu

TOL = 1e-5


def relL2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def row_scale(Y, ip, ix, pv, rows):
    """sum_j |p_ij w_ij Delta_ij| per row (L1 of the row's terms)."""
    out = np.zeros(len(rows))
    for t, i in enumerate(rows):
        cols = ix[ip[i]:ip[i + 1]]
        d = Y[i] - Y[cols]
        w = 1.0 / (1.0 + (d * d).sum(1))
        out[t] = (np.abs(pv[ip[i]:ip[i + 1]] * w)[:, None] * np.abs(d)).sum()
    return out


def dev_csr(ip, ix, pv):
    return CSR(torch.from_numpy(np.asarray(ip, np.int64)).cuda(), torch.from_numpy(np.asarray(ix, np.int32)).cuda(),
               torch.from_numpy(np.asarray(pv, np.float32)).cuda())


def attach(P, plan, shard=None):
    if plan in (True, "cb"):
        T.tsnet_plan_build(P, shard=shard)
    elif plan == "sell":
        T.tsnet_sell_build(P, shard=shard)
    return P


def check(ip, ix, pv, Y, shard=None, y_offset_rows=0, plan="cb"):
    """Plan kernel ("cb", "sell") or the CSR kernel ("csr") vs oracle on rows [rb, re)."""
    n = len(ip) - 1
    pv32 = np.asarray(pv, np.float32).astype(np.float64)
    P = attach(dev_csr(ip, ix, pv32), plan, shard)
    rb, re = (0, n) if shard is None else (shard.row_begin, shard.row_end)
    # optionally place Y at an 8-byte (not 16-byte) aligned address -> non-TMA copy path
    base = torch.zeros((n + y_offset_rows, 2), dtype=torch.float32, device="cuda")
    base[y_offset_rows:] = torch.from_numpy(Y)
    Yd = base[y_offset_rows:]
    F = torch.full((n, 2), float("nan"), dtype=torch.float32, device="cuda")
    tsnet_attr(P, Yd, F, shard=shard)
    torch.cuda.synchronize()
    got = F.cpu().numpy()[: re - rb].astype(np.float64)
    want = oracle.attr_sparse(Y.astype(np.float64), ip, ix, pv32)[rb:re]
    assert np.all(np.isfinite(got))
    if re > rb and np.linalg.norm(want) > 0:
        assert relL2(got, want) <= TOL, relL2(got, want)
    rows = np.arange(rb, re)
    if len(rows) > 4000:
        rows = np.unique(np.concatenate([rows[:1000], rows[-1000:], np.random.default_rng(1).choice(rows, 2000)]))
    sc = row_scale(Y.astype(np.float64), ip, ix, pv32, rows)
    err = np.abs(got[rows - rb] - want[rows - rb]).sum(1)
    assert np.all(err <= TOL * sc + 1e-30), float((err / np.maximum(sc, 1e-300)).max())
    return P


@pytest.mark.parametrize("plan", ["cb", "sell", "csr"])
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_configs(cfg, plan):
    ip, ix = config_graph(cfg)
    P = oracle.build_P(ip, ix, 40.0, seed=0)
    n = P["n"]
    for Y in (clustered_layout(n, 25.0, 7, 1.2, 2), uniform_layout(n, 3.0, 4)):
        check(P["indptr"], P["indices"], P["values"], Y, plan=plan)


@pytest.mark.parametrize("plan", ["cb", "sell", "csr"])
@pytest.mark.parametrize("n,kind", [(1, "single"), (7, "tiny"), (4095, "one_block_minus"), (4096, "one_block"),
                                    (4097, "block_plus_one"), (7167, "tile_block_minus"), (7168, "tile_block"),
                                    (7169, "tile_block_plus"), (7999, "y_block_minus"), (8000, "y_block"),
                                    (8001, "y_block_plus"), (8191, "two_blocks_minus"), (8192, "two_blocks"),
                                    (8193, "block_plus_one"), (24577, "odd_tail"), (20011, "hub_and_empty"),
                                    (50000, "short_rows"), (30011, "many_empty")])
def test_edge_patterns(n, kind, plan):
    rng = np.random.default_rng(n)
    L = rng.integers(0, 40, n)
    if kind == "hub_and_empty":
        L[::7] = 0                      # empty rows
        L[5] = n                        # a row touching every column (every block)
        L[6] = 3000
    if kind == "single":
        L[:] = 1
    if kind == "short_rows":            # > 32 row ends per 128 entries (window overflow path)
        L = rng.integers(0, 4, n)
    if kind == "many_empty":
        L[rng.random(n) < 0.8] = 0
    if kind in ("one_block", "two_blocks", "tile_block", "y_block"):
        L[0] = n                        # one row filling whole tiles: a run over many lanes (atomic pieces)
    ip, ix, pv = random_csr(n, L, seed=n)
    Y = uniform_layout(n, 10.0, 9)
    check(ip, ix, pv, Y, plan=plan)


def test_unaligned_Y_uses_copy_path():
    n = 9000
    ip, ix, pv = random_csr(n, np.random.default_rng(0).integers(1, 60, n), seed=3)
    check(ip, ix, pv, uniform_layout(n, 5.0, 1), y_offset_rows=1)


@pytest.mark.parametrize("plan", ["cb", "sell", "csr"])
def test_long_rows_many_tasks(plan):
    """Rows longer than a sweep and more than one wave of tasks (rows > 148 * 11264)."""
    n = 148 * 11264 + 5000
    L = np.full(n, 3)
    L[:200] = 2000
    ip, ix, pv = random_csr(n, L, seed=11)
    check(ip, ix, pv, uniform_layout(n, 20.0, 2), plan=plan)


@pytest.mark.parametrize("plan", ["cb", "sell"])
def test_shards_partition_the_rows(plan):
    ip, ix = config_graph(2)
    P = oracle.build_P(ip, ix, 40.0, seed=0)
    n = P["n"]
    Y = clustered_layout(n, 25.0, 7, 1.2, 2)
    for rb, re in ((0, n // 3), (n // 3, n // 3 + 1), (n // 3 + 1, n), (n, n), (33, 97)):
        check(P["indptr"], P["indices"], P["values"], Y, shard=T.tsnet_shard(0, 1, rb, re), plan=plan)


@pytest.mark.parametrize("plan", ["cb", "csr"])
def test_config4_full_size_sampled_rows(plan):
    """The bench workload (n ~ 0.95M, nnz ~ 2.06e8), GPU C0 output."""
    from paper_2509_19785_b200 import tsnet_build_P
    ip, ix = config_graph(4)
    got = tsnet_build_P(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), u=40.0, seed=0)
    P = got["P"]
    n = P.n
    Y = clustered_layout(n, 30.0, 40, 2.0, 5)
    Yd = torch.from_numpy(Y).cuda()
    attach(P, plan)
    F = tsnet_attr(P, Yd)
    torch.cuda.synchronize()
    pip, pix = P.indptr.cpu().numpy(), P.indices.cpu().numpy()
    pv = P.values.cpu().numpy().astype(np.float64)
    deg = np.diff(pip)
    rows = np.unique(np.concatenate([np.random.default_rng(0).choice(n, 3000, replace=False),
                                     np.argsort(deg)[-50:], [0, n - 1]]))
    want = np.stack([oracle.attr_sparse_rows(Y.astype(np.float64), pip, pix, pv, int(i), 1)[0] for i in rows])
    got = F.cpu().numpy()[rows].astype(np.float64)
    sc = row_scale(Y.astype(np.float64), pip, pix, pv, rows)
    err = np.abs(got - want).sum(1)
    assert np.all(err <= TOL * sc), float((err / sc).max())


def test_sell_config5_full_size():
    """Sliced ELL on the 3-D mesh at full size (n = 4.1M, nnz ~ 5.3e8, GPU C0):
    padding is small (slots per entry), sampled rows match the oracle, and all
    rows match the CSR kernel."""
    from paper_2509_19785_b200 import tsnet_build_P
    ip, ix = config_graph(5)
    P = tsnet_build_P(torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda(), u=40.0, seed=0)["P"]
    n = P.n
    Y = clustered_layout(n, 30.0, 40, 2.0, 5)
    Yd = torch.from_numpy(Y).cuda()
    F_csr = tsnet_attr(P, Yd)
    _, ratio = T.tsnet_sell_query(P)
    assert 1.0 <= ratio <= 1.3
    T.tsnet_sell_build(P)
    F = tsnet_attr(P, Yd)
    torch.cuda.synchronize()
    assert relL2(F.cpu().numpy(), F_csr.cpu().numpy()) <= 1e-6
    pip, pix = P.indptr.cpu().numpy(), P.indices.cpu().numpy()
    pv = P.values.cpu().numpy().astype(np.float64)
    rows = np.unique(np.concatenate([np.random.default_rng(0).choice(n, 2000, replace=False), [0, 31, 32, n - 1]]))
    want = np.stack([oracle.attr_sparse_rows(Y.astype(np.float64), pip, pix, pv, int(i), 1)[0] for i in rows])
    got = F.cpu().numpy()[rows].astype(np.float64)
    sc = row_scale(Y.astype(np.float64), pip, pix, pv, rows)
    assert np.all(np.abs(got - want).sum(1) <= TOL * sc), "sampled rows"
