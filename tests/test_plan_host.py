"""Host logic of the column-blocked plan (tsnet_plan_partition, pure host code
in libtsnet): the deal of rows into panels (one CTA each) used by the tiled
attractive SpMV.  No GPU."""
import numpy as np
import pytest

from workloads import config_graph, random_csr


@pytest.fixture(scope="module")
def T():
    from paper_2509_19785_b200 import build
    build.build()
    from paper_2509_19785_b200 import tsnet
    return tsnet


# the deal's row weight (attr_cb.cu, tile_row_weight): entries + 8, and rows of
# >= HUB_MIN entries weigh HUB_PM per mille more
HUB_MIN, HUB_PM = 32768, 600


def row_weight(L):
    return L + 8 + np.where(L >= HUB_MIN, L * HUB_PM // 1000, 0)


def check_cut(ip, rb, re, G, cap, cut):
    P, row_panel, row_local, panel_off, panel_rows = cut
    nr = re - rb
    L = np.diff(ip[rb:re + 1]).astype(np.int64)
    # panel count: G * ceil(nr / (G cap)), at most nr, at least 1
    want_P = max(1, min(G * -(-nr // (G * cap)), max(nr, 1)))
    assert P == want_P
    assert panel_off[0] == 0 and panel_off[-1] == nr and np.all(np.diff(panel_off) >= 0)
    sizes = np.diff(panel_off)
    assert sizes.max(initial=0) <= cap
    # every row exactly once; local index = position inside its panel; rows ascending in a panel
    assert np.array_equal(np.sort(panel_rows), np.arange(nr))
    for p in range(P):
        rows = panel_rows[panel_off[p]:panel_off[p + 1]]
        assert np.all(np.diff(rows) > 0)
        assert np.all(row_panel[rows] == p)
        assert np.array_equal(row_local[rows], np.arange(len(rows)))
    # LPT balance on the row weight: no panel exceeds the mean by more than the
    # largest single row weight (the textbook LPT bound); with a cap that binds,
    # only panels below the cap are compared
    if nr:
        w = row_weight(L)
        wts = np.bincount(row_panel, weights=w, minlength=P)
        open_ = sizes < cap
        if open_.any():
            assert wts[open_].max() <= wts.sum() / P + w.max() + 1e-9
    return P


@pytest.mark.parametrize("G", [1, 7, 148])
def test_cut_covers_rows_balanced(T, G):
    ip, _ = config_graph(2)
    n = len(ip) - 1
    check_cut(ip, 0, n, G, 8192, T.tsnet_plan_partition(ip, 0, n, G, 8192))


def test_row_cap_forces_more_panels(T):
    ip, _ = config_graph(2)
    n = len(ip) - 1
    cut = T.tsnet_plan_partition(ip, 0, n, 4, 100)
    P = check_cut(ip, 0, n, 4, 100, cut)
    assert P == 4 * -(-n // 400) and np.diff(cut[3]).max() <= 100


def test_power_law_rows_balanced(T):
    """Hub rows (a few rows hold a large share of the entries) spread over the
    panels: entries per panel within one hub row of the mean."""
    rng = np.random.default_rng(3)
    L = np.minimum((rng.pareto(1.5, 20000) * 60 + 120).astype(np.int64), 20000)
    ip = np.concatenate([[0], np.cumsum(L)])
    P = check_cut(ip, 0, len(L), 148, 8192, T.tsnet_plan_partition(ip, 0, len(L), 148, 8192))
    assert P == 148


def test_shard_rows_and_empty(T):
    ip, _ = config_graph(1)
    check_cut(ip, 100, 900, 8, 64, T.tsnet_plan_partition(ip, 100, 900, 8, 64))
    P, rp, rl, po, pr = T.tsnet_plan_partition(ip, 77, 77, 8, 64)
    assert P == 1 and len(rp) == 0 and list(po) == [0, 0]
    # fewer rows than groups: one row per panel
    P, rp, rl, po, pr = T.tsnet_plan_partition(ip, 0, 5, 148, 8192)
    assert P == 5 and np.array_equal(np.sort(rp), np.arange(5))


def test_empty_rows_and_bad_args(T):
    ip = np.concatenate([[0], np.cumsum(np.array([0, 3, 0, 0, 5, 1, 0] * 50))])
    check_cut(ip, 0, 350, 4, 64, T.tsnet_plan_partition(ip, 0, 350, 4, 64))
    z = np.zeros(501, np.int64)
    check_cut(z, 0, 500, 4, 64, T.tsnet_plan_partition(z, 0, 500, 4, 64))
    ip2, _, _ = random_csr(1000, np.full(1000, 5), 1)
    check_cut(ip2, 0, 1000, 3, 2000, T.tsnet_plan_partition(ip2, 0, 1000, 3, 2000))
    with pytest.raises(Exception):
        T.tsnet_plan_partition(ip, 5, 3, 16, 704)


def test_hub_rows_weigh_more(T):
    """Rows of >= HUB_MIN entries carry the hub penalty in the deal: the panels
    holding them get fewer entries than the others (their runs are split between
    warps in every block: DESIGN §5.1), and the LPT bound holds on the weight."""
    rng = np.random.default_rng(3)
    L = np.concatenate([[100000, 70000, 50000, 40000], rng.integers(5, 50, 20000)]).astype(np.int64)
    rng.shuffle(L)
    ip = np.concatenate([[0], np.cumsum(L)]).astype(np.int64)
    G = 8
    P, row_panel, _, _, _ = cut = T.tsnet_plan_partition(ip, 0, len(L), G, 8192)
    check_cut(ip, 0, len(L), G, 8192, cut)
    ent = np.bincount(row_panel, weights=L, minlength=P)
    hubp = np.unique(row_panel[L >= HUB_MIN])
    rest = np.setdiff1d(np.arange(P), hubp)
    assert len(rest) > 0 and ent[hubp].max() < ent[rest].min(), (ent[hubp], ent[rest])
