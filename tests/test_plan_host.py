"""Host logic of the column-blocked plan (tsnet_plan_partition, pure host code
in libtsnet): the cut of rows into units (rows, or pieces of long rows) and of
units into mini-tasks used by the attractive SpMV.  No GPU."""
import numpy as np
import pytest

from workloads import config_graph, random_csr


@pytest.fixture(scope="module")
def T():
    from paper_2509_19785_b200 import build
    build.build()
    from paper_2509_19785_b200 import tsnet
    return tsnet


def check_cut(ip, rb, re, W, RM, base, cut):
    G, row_mt, row_K, mt_r0, mt_info = cut
    nr = re - rb
    L = np.diff(ip[rb:re + 1])
    nnz = int(L.sum())
    cap = max(256, nnz // (base * W) // 2)
    T = G * W
    assert G % base == 0 and G >= base and len(mt_r0) == T
    assert np.array_equal(row_K, np.where(L > cap, -(-L // cap), 1))     # long rows split into pieces
    covered = np.zeros(nr, np.int64)
    for t in range(T):
        r0, info = int(mt_r0[t]), int(mt_info[t])
        if info < 0:                                     # a piece of one split row
            assert row_K[r0] > 1 and row_mt[r0] <= t < row_mt[r0] + row_K[r0]
            covered[r0] += 1
        elif info > 0:                                   # a run of whole rows
            assert info <= RM
            rows = np.arange(r0, r0 + info)
            assert np.all(row_K[rows] == 1) and np.all(row_mt[rows] == t)
            covered[rows] += 1
    assert np.array_equal(covered, row_K)                 # every row exactly once (pieces: K times)
    # runs in row order
    firsts = [int(mt_r0[t]) for t in range(T) if mt_info[t] != 0]
    assert firsts == sorted(firsts)
    # balance of runs on (entries + rows): none exceeds the mean by more than one row
    runs = [(int(mt_r0[t]), int(mt_info[t])) for t in range(T) if mt_info[t] > 0]
    if runs:
        w = [int(L[r0:r0 + k].sum()) + k for r0, k in runs]
        tot = sum(int(L[q]) + 1 for q in range(nr) if row_K[q] == 1)
        n_pieces = int(row_K[row_K > 1].sum())
        n_split = int((row_K > 1).sum())
        assert max(w) <= tot / max(1, T - n_pieces - n_split) + cap + 1
    return T


@pytest.mark.parametrize("base", [1, 7, 148])
def test_cut_covers_rows_balanced(T, base):
    ip, _ = config_graph(2)
    n = len(ip) - 1
    check_cut(ip, 0, n, 16, 704, base, T.tsnet_plan_partition(ip, 0, n, 16, 704, base))


def test_row_cap_forces_more_groups(T):
    n = 100_000
    ip = np.arange(n + 1, dtype=np.int64) * 3
    cut = T.tsnet_plan_partition(ip, 0, n, 4, 100, 148)
    check_cut(ip, 0, n, 4, 100, 148, cut)
    assert cut[0] == 148 * 2     # 592 mini-tasks cannot hold 100k rows at <= 100 each; 1184 can


def test_long_rows_are_split(T):
    L = np.full(5000, 3)
    L[10] = 4000                 # a hub row: far above the piece cap
    ip, _, _ = random_csr(5000, L, seed=2)
    cut = T.tsnet_plan_partition(ip, 0, 5000, 4, 64, 2)
    check_cut(ip, 0, 5000, 4, 64, 2, cut)
    assert cut[2][10] > 1


def test_shard_and_empty_ranges(T):
    ip, _, _ = random_csr(5000, np.random.default_rng(0).integers(0, 30, 5000), seed=1)
    check_cut(ip, 1234, 4321, 8, 64, 8, T.tsnet_plan_partition(ip, 1234, 4321, 8, 64, 8))
    cut = T.tsnet_plan_partition(ip, 77, 77, 8, 64, 8)
    assert len(cut[1]) == 0 and np.all(cut[4] == 0)


def test_trailing_and_leading_empty_rows(T):
    """Rows with no entries at either end are covered (an earlier cut looped
    forever when the last rows were empty)."""
    L = np.zeros(30011, np.int64)
    L[100:20000] = 5
    ip = np.zeros(len(L) + 1, np.int64)
    np.cumsum(L, out=ip[1:])
    check_cut(ip, 0, len(L), 16, 704, 148, T.tsnet_plan_partition(ip, 0, len(L), 16, 704, 148))
    z = np.zeros(501, np.int64)                                      # no entries at all
    check_cut(z, 0, 500, 4, 64, 4, T.tsnet_plan_partition(z, 0, 500, 4, 64, 4))


def test_bad_arguments(T):
    ip = np.arange(11, dtype=np.int64)
    with pytest.raises(Exception):
        T.tsnet_plan_partition(ip, 5, 3, 16, 704, 1)
