"""Pivot MDS initial layout (NEXT-2; tsnet_pmds, pmds.cu) against the oracle
O8 (oracle/pmds.py).  Integer work bit-exact: the pivot sequence and the hop
matrix.  Floating point: the two eigenvalues within 1e-9 relative; the layout
within 1e-5 relative L2 where the top-2 eigenvectors are unique (a gap between
the second and third eigenvalue and between the first and second), and
otherwise through what is unique -- the pairwise distances of the layout,
which do not depend on the basis chosen inside a degenerate eigenspace."""
import numpy as np
import pytest
import torch
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import shortest_path

import oracle
from oracle import pmds as O
from paper_2509_19785_b200 import tsnet_pmds
from paper_2509_19785_b200 import tsnet as T
from workloads import config_graph, cycle_graph, erdos_renyi, grid2d, path_graph, random_tree, star_graph

pytestmark = pytest.mark.gpu


def relL2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run_gpu(ip, ix, p, seed):
    r = tsnet_pmds(torch.from_numpy(np.asarray(ip, np.int64)).cuda(),
                   torch.from_numpy(np.asarray(ix, np.int32)).cuda(), p, seed, hops=True)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in r.items()}


def pairwise(Y, idx):
    Z = Y[idx].astype(np.float64)
    return np.linalg.norm(Z[:, None, :] - Z[None, :, :], axis=2)


def check_layout(got, want, p):
    """Eigenvalues; then the layout elementwise when its basis is unique,
    else its pairwise distances."""
    l1, l2 = want["l1"], want["l2"]
    assert abs(got["eig"][0] - l1) <= 1e-9 * l1
    assert abs(got["eig"][1] - l2) <= 1e-9 * l1
    Yg, Yo = got["Y"], want["Y"]
    assert np.abs(Yg.astype(np.float64).mean(axis=0)).max() <= 1e-5 * np.abs(Yo).max()
    C = O.centred(want["hops"])
    ev = np.linalg.eigvalsh(C.T @ C)[::-1]
    third = ev[2] if p > 2 else 0.0
    unique = (l1 - l2 > 1e-6 * l1) and (l2 <= 1e-12 * l1 or l2 - third > 1e-6 * l1)
    if unique:
        assert relL2(Yg, Yo) <= 1e-5, relL2(Yg, Yo)
    else:
        idx = np.random.default_rng(0).choice(len(Yo), min(len(Yo), 400), replace=False)
        assert relL2(pairwise(Yg, idx), pairwise(Yo, idx)) <= 1e-5
    return unique


@pytest.mark.parametrize("cfg,p", [(1, 50), (1, 250), (2, 60)])
@pytest.mark.parametrize("seed", [0, 5])
def test_configs(cfg, p, seed):
    ip, ix = config_graph(cfg)
    want = O.pmds(ip, ix, p, seed)
    got = run_gpu(ip, ix, p, seed)
    assert list(got["pivots"]) == want["pivots"]
    assert np.array_equal(got["hops"], want["hops"].T.astype(np.int32))
    check_layout(got, want, p)


@pytest.mark.parametrize("make,p", [(lambda: path_graph(2), 2), (lambda: path_graph(37), 37),
                                    (lambda: cycle_graph(4), 4), (lambda: cycle_graph(31), 12),
                                    (lambda: star_graph(40), 10), (lambda: random_tree(300, 3), 40),
                                    (lambda: erdos_renyi(200, 0.006, 4), 30),     # disconnected: unreachable = n
                                    (lambda: grid2d(13, 11), 143), (lambda: path_graph(1), 1)])
def test_edge_graphs(make, p):
    ip, ix = make()
    want = O.pmds(ip, ix, p, 3)
    got = run_gpu(ip, ix, p, 3)
    assert list(got["pivots"]) == want["pivots"]
    assert np.array_equal(got["hops"], want["hops"].T.astype(np.int32))
    if len(ip) - 1 >= 2:
        check_layout(got, want, p)


def test_config4_full_size_16_pivots():
    """n = 0.95M: every hop column equals a library BFS (scipy) from its
    pivot, the pivot chain obeys the max-min rule on those columns, and the
    layout equals the oracle's embedding of the same hop matrix."""
    ip, ix = config_graph(4)
    n, p = len(ip) - 1, 16
    got = run_gpu(ip, ix, p, 0)
    piv = [int(v) for v in got["pivots"]]
    assert piv[0] == O.first_pivot(n, 0)
    A = csr_matrix((np.ones(len(ix)), ix, ip), shape=(n, n))
    D = shortest_path(A, unweighted=True, indices=piv)
    D[~np.isfinite(D)] = n
    assert np.array_equal(got["hops"], D.astype(np.int32))
    dmin = D[0].copy()
    for t in range(1, p):
        assert piv[t] == int(np.flatnonzero(dmin == dmin.max())[0])
        dmin = np.minimum(dmin, D[t])
    Y, (l1, l2, V) = O.embed(D.T.astype(np.int64), 0)
    check_layout(got, {"Y": Y, "l1": l1, "l2": l2, "hops": D.T.astype(np.int64)}, p)


def test_argument_errors():
    ip, ix = path_graph(5)
    with pytest.raises(T.TsnetError):
        tsnet_pmds(torch.from_numpy(ip).cuda(), torch.from_numpy(ix.astype(np.int32)).cuda(), 0, 0)
