"""Host logic of the column-blocked plan (tsnet_plan_partition, pure host code
in libtsnet): the task cut of rows used by the attractive SpMV.
No GPU needed."""
import numpy as np
import pytest

from workloads import config_graph, random_csr


@pytest.fixture(scope="module")
def T():
    from paper_2509_19785_b200 import build
    build.build()
    from paper_2509_19785_b200 import tsnet
    return tsnet


def check_cut(ip, rb, re, rows_max, base, r0, rr):
    T_ = len(r0)
    assert T_ % base == 0 and T_ >= base
    assert r0[0] == rb and np.all(rr >= 0) and np.all(rr <= rows_max)
    assert np.array_equal(r0[1:], r0[:-1] + rr[:-1])       # contiguous, in order
    assert r0[-1] + rr[-1] == re                          # covers [rb, re)
    return T_


@pytest.mark.parametrize("base", [1, 7, 148])
def test_cut_covers_rows_balanced(T, base):
    ip, ix = config_graph(2)
    n = len(ip) - 1
    r0, rr = T.tsnet_plan_partition(ip, 0, n, 11264, base)
    Tn = check_cut(ip, 0, n, 11264, base, r0, rr)
    wgt = np.array([ip[a + b] - ip[a] + b for a, b in zip(r0, rr)])
    # greedy cut at multiples of (nnz + rows)/T: each task within one row of the target
    assert wgt.max() <= (ip[-1] + n) / Tn + np.diff(ip).max() + 1


def test_row_cap_forces_more_tasks(T):
    n = 100_000
    ip = np.arange(n + 1, dtype=np.int64) * 3
    r0, rr = T.tsnet_plan_partition(ip, 0, n, 500, 148)
    Tn = check_cut(ip, 0, n, 500, 148, r0, rr)
    assert Tn == 148 * 2          # 148 tasks cannot hold 100k rows at <= 500 each; 296 can


def test_shard_and_empty_ranges(T):
    ip, _, _ = random_csr(5000, np.random.default_rng(0).integers(0, 30, 5000), seed=1)
    r0, rr = T.tsnet_plan_partition(ip, 1234, 4321, 64, 8)
    check_cut(ip, 1234, 4321, 64, 8, r0, rr)
    r0, rr = T.tsnet_plan_partition(ip, 77, 77, 64, 8)
    assert len(r0) == 1 and rr[0] == 0 and r0[0] == 77


def test_hub_row_alone(T):
    L = np.full(1000, 2)
    L[500] = 1000
    ip, _, _ = random_csr(1000, L, seed=2)
    r0, rr = T.tsnet_plan_partition(ip, 0, 1000, 11264, 4)
    check_cut(ip, 0, 1000, 11264, 4, r0, rr)


def test_bad_arguments(T):
    ip = np.arange(11, dtype=np.int64)
    with pytest.raises(Exception):
        T.tsnet_plan_partition(ip, 5, 3, 10, 1)


def test_trailing_and_leading_empty_rows(T):
    """Rows with no entries at either end must still be covered (the cut used
    to loop forever when the last rows were empty)."""
    L = np.zeros(30011, np.int64)
    L[100:20000] = 5
    ip = np.zeros(len(L) + 1, np.int64)
    np.cumsum(L, out=ip[1:])
    r0, rr = T.tsnet_plan_partition(ip, 0, len(L), 11264, 148)
    check_cut(ip, 0, len(L), 11264, 148, r0, rr)
    r0, rr = T.tsnet_plan_partition(np.zeros(501, np.int64), 0, 500, 64, 4)   # no entries at all
    check_cut(np.zeros(501, np.int64), 0, 500, 64, 4, r0, rr)
