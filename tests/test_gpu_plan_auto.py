"""attach_plan(P, "auto"): sliced ELL on a mesh (padding
<= 1.3 slots per entry), CSR on a block model and on a power-law graph; and
the hot-column L1 policy of the CSR SpMV gives the same forces whether it is
on or off (it only changes cache hints)."""
import numpy as np
import pytest
import torch

from paper_2509_19785_b200 import CSR, attach_plan, tsnet_attr, tsnet_build_P
from paper_2509_19785_b200 import tsnet as T
from workloads import chung_lu, config_graph, grid2d, clustered_layout

pytestmark = pytest.mark.gpu


def build(ip, ix):
    return tsnet_build_P(torch.from_numpy(np.asarray(ip, np.int64)).cuda(),
                         torch.from_numpy(np.asarray(ix, np.int32)).cuda(), u=40.0, seed=0)["P"]


def test_auto_choices():
    mesh = build(*grid2d(200, 150))
    attach_plan(mesh, "auto")
    assert mesh.plan is not None and mesh.plan_kind == T.PLAN_SELL
    sbm = build(*config_graph(3))
    attach_plan(sbm, "auto")
    assert sbm.plan is None
    pl = build(*chung_lu(60000, 2.5, 6.0, 3))
    attach_plan(pl, "auto")
    assert pl.plan is None


def test_hot_column_policy_same_forces():
    """Chung-Lu numbers vertices by weight, so the policy switches on; the
    forces must equal those of a copy whose index array is shifted by nothing
    but evaluated with the policy off (a CSR whose first columns are cold:
    the same P with its vertices reversed)."""
    ip, ix = chung_lu(400000, 2.5, 6.0, 3)     # first 8192 columns: > 4x their share of P (policy on)
    P = build(ip, ix)
    n = P.n
    pip = P.indptr.cpu().numpy()
    assert (pip[8192] - pip[0]) / pip[n] >= 4.0 * 8192 / n
    Y = torch.from_numpy(clustered_layout(n, 10.0, 10, 1.5, 2)).cuda()
    F = tsnet_attr(P, Y)
    # reversed numbering: the hubs are last, the policy stays off
    perm = torch.arange(n - 1, -1, -1, device="cuda")
    ipr = P.indptr.cpu().numpy()
    ixr = P.indices.cpu().numpy()
    vr = P.values.cpu().numpy()
    rows = []
    for r in range(n - 1, -1, -1):
        a, b = ipr[r], ipr[r + 1]
        c = (n - 1 - ixr[a:b])[::-1]
        rows.append((c, vr[a:b][::-1]))
    ind = np.concatenate([c for c, _ in rows]).astype(np.int32)
    val = np.concatenate([v for _, v in rows]).astype(np.float32)
    ptr = np.zeros(n + 1, np.int64)
    ptr[1:] = np.cumsum([len(c) for c, _ in rows])
    Pr = CSR(torch.from_numpy(ptr).cuda(), torch.from_numpy(ind).cuda(), torch.from_numpy(val).cuda())
    Fr = tsnet_attr(Pr, Y[perm].contiguous())
    torch.cuda.synchronize()
    a = F.cpu().numpy().astype(np.float64)
    b = Fr.cpu().numpy()[::-1].astype(np.float64)
    assert np.linalg.norm(a - b) <= 1e-6 * np.linalg.norm(a)
