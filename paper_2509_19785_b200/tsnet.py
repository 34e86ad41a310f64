"""Thin ctypes binding of libtsnet.so (include/tsnet.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C-ABI.  PyTorch provides device memory and the stream.
Names follow the C-ABI (tsnet_build_P, tsnet_grad, tsnet_grad_parts,
tsnet_step, tsnet_step_host, tsnet_cost, tsnet_workspace_bytes,
tsnet_read_stats, tsnet_last_error).  There is no CPU fallback: if the
library is missing or fails, these functions raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtsnet.so")

c_i32, c_i64, c_f32, c_f64, c_sz, c_vp, c_u64 = (ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double,
                                                 ctypes.c_size_t, ctypes.c_void_p, ctypes.c_uint64)

TSNET_OK, TSNET_E_ARG, TSNET_E_CAPACITY, TSNET_E_CUDA, TSNET_E_NCCL, TSNET_E_NONFINITE, TSNET_W_PERPLEXITY = range(7)
TSNET_I_MAX_LIMIT = 1024
PLAN_CB, PLAN_SELL = 1, 2     # tsnet_csr.plan_kind (include/tsnet.h)


class tsnet_graph(ctypes.Structure):
    _fields_ = [("n", c_i64), ("indptr", c_vp), ("indices", c_vp)]


class tsnet_csr(ctypes.Structure):
    _fields_ = [("n", c_i64), ("nnz", c_i64), ("capacity", c_i64), ("indptr", c_vp), ("indices", c_vp),
                ("values", c_vp), ("plan", c_vp), ("plan_kind", c_i32), ("plan_row_begin", c_i64),
                ("plan_row_end", c_i64)]


class tsnet_grad_params(ctypes.Structure):
    _fields_ = [("lambda_kl", c_f32), ("lambda_c", c_f32), ("lambda_r", c_f32), ("eps", c_f32),
                ("interp_P", c_i32), ("h_max", c_f32), ("I_min", c_i32), ("I_max", c_i32), ("spread", c_i32)]


class tsnet_step_params(ctypes.Structure):
    _fields_ = [("eta", c_f32), ("momentum", c_f32), ("gain_inc", c_f32), ("gain_dec", c_f32),
                ("gain_min", c_f32), ("recenter", c_i32)]


class tsnet_shard(ctypes.Structure):
    _fields_ = [("rank", c_i32), ("world", c_i32), ("row_begin", c_i64), ("row_end", c_i64), ("comm", c_vp),
                ("bounds", ctypes.POINTER(c_i64))]


class tsnet_stats(ctypes.Structure):
    _fields_ = [("Z", c_f64), ("lo_x", c_f64), ("lo_y", c_f64), ("S", c_f64), ("h_b", c_f64), ("I", c_i32),
                ("N", c_i32), ("M", c_i32), ("nonfinite", c_i32), ("spread", c_i32), ("spread_points", c_i64),
                ("spread_flushes", c_i64)]


_lib = None

# (name, restype, argtypes) of every C-ABI entry point
SIGNATURES = [
    ("tsnet_resolve_k", c_i32, [c_i64, c_f64, c_i32]),
    ("tsnet_build_P_workspace_bytes", c_sz, [c_i64, c_i32]),
    ("tsnet_build_P", ctypes.c_int, [ctypes.POINTER(tsnet_graph), c_f64, c_i32, c_u64, ctypes.POINTER(tsnet_csr),
                                     c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    ("tsnet_workspace_bytes", c_sz, [c_i64, c_i64, ctypes.POINTER(tsnet_grad_params), ctypes.POINTER(tsnet_shard)]),
    ("tsnet_grad", ctypes.c_int, [ctypes.POINTER(tsnet_csr), c_vp, ctypes.POINTER(tsnet_grad_params),
                                  ctypes.POINTER(tsnet_shard), c_vp, c_vp, c_vp, c_sz, c_vp]),
    ("tsnet_attr", ctypes.c_int, [ctypes.POINTER(tsnet_csr), c_vp, ctypes.POINTER(tsnet_shard), c_vp, c_vp]),
    ("tsnet_grad_parts", ctypes.c_int, [ctypes.POINTER(tsnet_csr), c_vp, ctypes.POINTER(tsnet_grad_params),
                                        ctypes.POINTER(tsnet_shard), c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    ("tsnet_step", ctypes.c_int, [ctypes.POINTER(tsnet_csr), c_vp, c_vp, c_vp, ctypes.POINTER(tsnet_grad_params),
                                  ctypes.POINTER(tsnet_step_params), ctypes.POINTER(tsnet_shard), c_vp, c_sz, c_vp]),
    ("tsnet_step_host", ctypes.c_int, [ctypes.POINTER(tsnet_csr), c_vp, c_vp, c_vp,
                                       ctypes.POINTER(tsnet_grad_params), ctypes.POINTER(tsnet_step_params),
                                       ctypes.POINTER(tsnet_shard), c_vp, c_sz, c_vp]),
    ("tsnet_cost", ctypes.c_int, [ctypes.POINTER(tsnet_csr), c_vp, ctypes.POINTER(tsnet_grad_params), c_i32,
                                  ctypes.POINTER(tsnet_shard), c_vp, c_vp, c_sz, c_vp]),
    ("tsnet_plan_query", ctypes.c_int, [ctypes.POINTER(tsnet_csr), ctypes.POINTER(tsnet_shard),
                                        ctypes.POINTER(c_sz), ctypes.POINTER(c_sz), c_vp]),
    ("tsnet_plan_build", ctypes.c_int, [ctypes.POINTER(tsnet_csr), ctypes.POINTER(tsnet_shard), c_vp, c_sz, c_vp,
                                        c_sz, c_vp]),
    ("tsnet_pmds_workspace_bytes", c_sz, [c_i64, c_i32]),
    ("tsnet_pmds", ctypes.c_int, [ctypes.POINTER(tsnet_graph), c_i32, ctypes.c_uint64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                  c_sz, c_vp]),
    ("tsnet_tree_workspace_bytes", c_sz, [c_i64]),
    ("tsnet_grad_tree", ctypes.c_int, [ctypes.POINTER(tsnet_csr), c_vp, ctypes.POINTER(tsnet_grad_params),
                                       ctypes.c_double, c_i32, c_vp, c_vp, c_vp, c_sz, c_vp, c_sz, c_vp]),
    ("tsnet_quality_workspace_bytes", c_sz, [c_i64]),
    ("tsnet_quality", ctypes.c_int, [ctypes.POINTER(tsnet_graph), c_vp, c_i32, c_vp, c_vp, c_sz, c_vp]),
    ("tsnet_move", ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, ctypes.POINTER(tsnet_step_params), c_vp]),
    ("tsnet_sell_query", ctypes.c_int, [ctypes.POINTER(tsnet_csr), ctypes.POINTER(tsnet_shard), ctypes.POINTER(c_sz),
                                        ctypes.POINTER(ctypes.c_double), c_vp]),
    ("tsnet_sell_build", ctypes.c_int, [ctypes.POINTER(tsnet_csr), ctypes.POINTER(tsnet_shard), c_vp, c_sz, c_vp]),
    ("tsnet_plan_partition", c_i32, [c_vp, c_i64, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_i64]),
    ("tsnet_comm_unique_id", ctypes.c_int, [c_vp]),
    ("tsnet_comm_init", ctypes.c_int, [c_vp, c_i32, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    ("tsnet_comm_peer_reduce", ctypes.c_int, [c_vp]),
    ("tsnet_comm_layout", ctypes.c_int, [c_vp, c_i64, ctypes.POINTER(c_vp)]),
    ("tsnet_comm_layout_push", ctypes.c_int, [c_vp]),
    ("tsnet_comm_layout_sync", ctypes.c_int, [c_vp, c_vp]),
    ("tsnet_grids_sum", ctypes.c_int, [c_i32, ctypes.POINTER(c_vp), c_sz, c_i64, c_i64,
                                       ctypes.POINTER(tsnet_grad_params), c_vp]),
    ("tsnet_comm_destroy", ctypes.c_int, [c_vp]),
    ("tsnet_shard_rows", c_i32, [c_vp, c_i64, c_i32, c_vp]),
    ("tsnet_field_local", ctypes.c_int, [ctypes.POINTER(tsnet_csr), c_vp, ctypes.POINTER(tsnet_grad_params),
                                         ctypes.POINTER(tsnet_shard), c_vp, c_sz, c_vp]),
    ("tsnet_ws_grid", ctypes.c_int, [c_i64, c_i64, ctypes.POINTER(tsnet_grad_params), ctypes.POINTER(c_sz),
                                     ctypes.POINTER(c_sz)]),
    ("tsnet_step_finish", ctypes.c_int, [ctypes.POINTER(tsnet_csr), c_vp, c_vp, c_vp,
                                         ctypes.POINTER(tsnet_grad_params), ctypes.POINTER(tsnet_step_params),
                                         ctypes.POINTER(tsnet_shard), c_vp, c_sz, c_vp]),
    ("tsnet_read_stats", ctypes.c_int, [c_vp, ctypes.POINTER(tsnet_stats), c_vp]),
    ("tsnet_last_error", ctypes.c_char_p, []),
]


def lib():
    """Load libtsnet.so (fails loudly if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2509_19785_b200.build` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class TsnetError(RuntimeError):
    def __init__(self, fn, status):
        msg = lib().tsnet_last_error().decode(errors="replace")
        super().__init__(f"{fn} failed with status {status}: {msg}")
        self.status = status


def _check(fn, st, ok=(TSNET_OK,)):
    if st not in ok:
        raise TsnetError(fn, st)
    return st


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("tensor must be on the CUDA device (no CPU fallback)")


# ----------------------------------------------------------------- params
@dataclass
class GradParams:
    lambda_kl: float = 1.0
    lambda_c: float = 0.01
    lambda_r: float = 0.6
    eps: float = 0.05
    interp_P: int = 3
    h_max: float = 0.25
    I_min: int = 20
    I_max: int = TSNET_I_MAX_LIMIT
    spread: int = 0        # TSNET_SPREAD_AUTO / _SORT / _RUNS (tsnet.h)

    def c(self):
        return tsnet_grad_params(self.lambda_kl, self.lambda_c, self.lambda_r, self.eps, self.interp_P, self.h_max,
                                 self.I_min, self.I_max, self.spread)


@dataclass
class StepParams:
    eta: float = 50.0
    momentum: float = 0.8
    gain_inc: float = 0.2
    gain_dec: float = 0.8
    gain_min: float = 0.01
    recenter: int = 0

    def c(self):
        return tsnet_step_params(self.eta, self.momentum, self.gain_inc, self.gain_dec, self.gain_min,
                                 int(self.recenter))


class CSR:
    """Device CSR matrix P (int64 indptr, int32 indices, fp32 values), plus an
    optional plan of the same P: column-blocked (tsnet_plan_build) or sliced ELL
    (tsnet_sell_build); `plan` is a uint8 device tensor (None = CSR kernel),
    `plan_kind` PLAN_CB / PLAN_SELL."""

    def __init__(self, indptr: torch.Tensor, indices: torch.Tensor, values: torch.Tensor, nnz: int | None = None):
        _require_cuda(indptr, indices, values)
        assert indptr.dtype == torch.int64 and indices.dtype == torch.int32 and values.dtype == torch.float32
        self.indptr, self.indices, self.values = indptr, indices, values
        self.n = indptr.numel() - 1
        self.nnz = int(indices.numel()) if nnz is None else int(nnz)
        self.plan = None
        self.plan_kind = 0
        self.plan_rows = (0, self.n)     # the rows the plan was built for (its shard)

    def c(self):
        return tsnet_csr(self.n, self.nnz, int(self.indices.numel()), self.indptr.data_ptr(),
                         self.indices.data_ptr() if self.indices.numel() else None,
                         self.values.data_ptr() if self.values.numel() else None,
                         self.plan.data_ptr() if self.plan is not None else None,
                         self.plan_kind if self.plan is not None else 0, self.plan_rows[0], self.plan_rows[1])

    def without_plan(self) -> "CSR":
        """Same P, CSR kernel (shares the tensors)."""
        q = CSR(self.indptr, self.indices, self.values, self.nnz)
        return q


# ------------------------------------------------------------------ C0
def tsnet_resolve_k(n: int, u: float, k: int = 0) -> int:
    return int(lib().tsnet_resolve_k(n, u, k))


def tsnet_build_P_workspace_bytes(n: int, k: int) -> int:
    return int(lib().tsnet_build_P_workspace_bytes(n, k))


def tsnet_build_P(indptr: torch.Tensor, indices: torch.Tensor, u: float = 40.0, k: int = 0, seed: int = 0,
                  capacity: int | None = None, stream=None):
    """C0 on the GPU.  Returns dict(P=CSR, knn_idx, knn_hop, knn_len, beta, k, status)."""
    _require_cuda(indptr, indices)
    dev = indptr.device
    n = indptr.numel() - 1
    k = tsnet_resolve_k(n, u, k)
    ws_bytes = tsnet_build_P_workspace_bytes(n, k)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    knn_idx = torch.empty((n, max(k, 1)), dtype=torch.int32, device=dev)
    knn_hop = torch.empty((n, max(k, 1)), dtype=torch.int32, device=dev)
    knn_len = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    beta = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    cap = 2 * n * k if capacity is None else capacity
    P_ip = torch.empty(n + 1, dtype=torch.int64, device=dev)
    P_ix = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    P_v = torch.empty(max(cap, 1), dtype=torch.float32, device=dev)
    g = tsnet_graph(n, indptr.data_ptr(), indices.data_ptr() if indices.numel() else None)
    P = tsnet_csr(n, 0, cap, P_ip.data_ptr(), P_ix.data_ptr(), P_v.data_ptr())
    st = lib().tsnet_build_P(ctypes.byref(g), float(u), k, seed & 0xFFFFFFFFFFFFFFFF, ctypes.byref(P),
                             _ptr(knn_idx), _ptr(knn_hop), _ptr(knn_len), _ptr(beta), _ptr(ws), ws_bytes,
                             _stream(stream))
    if st == TSNET_E_CAPACITY:
        return dict(status=st, required_nnz=int(P.nnz))
    _check("tsnet_build_P", st, ok=(TSNET_OK, TSNET_W_PERPLEXITY))
    nnz = int(P.nnz)
    del ws
    return dict(P=CSR(P_ip, P_ix[:nnz].clone(), P_v[:nnz].clone()), knn_idx=knn_idx[:, :k], knn_hop=knn_hop[:, :k],
                knn_len=knn_len[:n], beta=beta[:n], k=k, status=st)


# ------------------------------------------------------ Pivot MDS layout
def tsnet_pmds(indptr: torch.Tensor, indices: torch.Tensor, pivots: int = 250, seed: int = 0, hops: bool = False,
               stream=None):
    """Pivot MDS initial layout of the graph (set-up, blocking).  Returns a dict:
    Y (n x 2 fp32, device), pivots (int32[p]), eig (fp64[2]) and, with
    hops=True, the hop matrix (int32 p x n, pivot-major)."""
    _require_cuda(indptr, indices)
    n = indptr.numel() - 1
    p = min(int(pivots), n)
    dev = indptr.device
    g = tsnet_graph(n, indptr.data_ptr(), indices.data_ptr() if indices.numel() else None)
    Y = torch.empty((n, 2), dtype=torch.float32, device=dev)
    piv = torch.empty(p, dtype=torch.int32, device=dev)
    eig = torch.empty(2, dtype=torch.float64, device=dev)
    H = torch.empty((p, n), dtype=torch.int32, device=dev) if hops else None
    wb = int(lib().tsnet_pmds_workspace_bytes(n, p))
    ws = torch.empty(max(wb, 1), dtype=torch.uint8, device=dev)
    _check("tsnet_pmds", lib().tsnet_pmds(ctypes.byref(g), p, ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), _ptr(Y),
                                          _ptr(piv), _ptr(H) if H is not None else None, _ptr(eig), _ptr(ws), wb,
                                          _stream(stream)))
    out = {"Y": Y, "pivots": piv, "eig": eig}
    if H is not None:
        out["hops"] = H
    return out


# ---------------------------------------------- quality metrics, stand-alone move
def tsnet_quality(indptr: torch.Tensor, indices: torch.Tensor, Y: torch.Tensor, r: int = 2, stream=None):
    """(NP, stress) of the drawing Y of the graph (device tensors)."""
    _require_cuda(indptr, indices, Y)
    n = indptr.numel() - 1
    g = tsnet_graph(n, indptr.data_ptr(), indices.data_ptr() if indices.numel() else None)
    out = torch.empty(2, dtype=torch.float64, device=Y.device)
    wb = int(lib().tsnet_quality_workspace_bytes(n))
    ws = torch.empty(max(wb, 1), dtype=torch.uint8, device=Y.device)
    _check("tsnet_quality", lib().tsnet_quality(ctypes.byref(g), _ptr(Y), int(r), _ptr(out), _ptr(ws), wb,
                                                _stream(stream)))
    o = out.cpu().tolist()
    return o[0], o[1]


def tsnet_move(Y, vel, gains, grad, sp: StepParams, stream=None):
    """Gains/momentum move of step a7 with a given gradient (in place)."""
    _require_cuda(Y, vel, gains, grad)
    s = sp.c()
    _check("tsnet_move", lib().tsnet_move(_ptr(Y), _ptr(vel), _ptr(gains), _ptr(grad), Y.shape[0], ctypes.byref(s),
                                          _stream(stream)))


# ------------------------------------------------ column-blocked plan of P
def tsnet_plan_query(P: CSR, shard=None, stream=None):
    pb, wb = c_sz(0), c_sz(0)
    Pc = P.c()
    _check("tsnet_plan_query", lib().tsnet_plan_query(ctypes.byref(Pc), _shard(shard), ctypes.byref(pb),
                                                      ctypes.byref(wb), _stream(stream)))
    return int(pb.value), int(wb.value)


def tsnet_plan_build(P: CSR, shard=None, stream=None) -> CSR:
    """Build the column-blocked plan of P (set-up, blocking) and attach it: P.plan."""
    pbytes, wbytes = tsnet_plan_query(P, shard, stream)
    plan = torch.empty(max(pbytes, 1), dtype=torch.uint8, device=P.indptr.device)
    ws = torch.empty(max(wbytes, 1), dtype=torch.uint8, device=P.indptr.device)
    P.plan = None
    Pc = P.c()
    _check("tsnet_plan_build", lib().tsnet_plan_build(ctypes.byref(Pc), _shard(shard), _ptr(plan), pbytes, _ptr(ws),
                                                      wbytes, _stream(stream)))
    del ws
    P.plan = plan
    P.plan_kind = PLAN_CB
    P.plan_rows = (0, P.n) if shard is None else _shard_rows(shard)
    return P


# ------------------------------------------------------ sliced-ELL plan of P
def tsnet_sell_query(P: CSR, shard=None, stream=None):
    """(plan bytes, slots per stored entry) of the sliced-ELL plan."""
    pb, ratio = c_sz(0), ctypes.c_double(0.0)
    Pc = P.c()
    _check("tsnet_sell_query", lib().tsnet_sell_query(ctypes.byref(Pc), _shard(shard), ctypes.byref(pb),
                                                      ctypes.byref(ratio), _stream(stream)))
    return int(pb.value), float(ratio.value)


SELL_AUTO_MAX_SLOTS_PER_NNZ = 1.3


def attach_plan(P: CSR, plan="auto", shard=None, stream=None) -> CSR:
    """Attach the SpMV layout `plan` to P: "csr" (none), "cb" (column-blocked),
    "sell" (sliced ELL), or "auto": sliced ELL when its padding is at most
    SELL_AUTO_MAX_SLOTS_PER_NNZ slots per stored entry (meshes: cfg 5 pads
    1.027, 1028 vs 710 it/s), else CSR (power-law graphs, where hub rows pad
    the slices and the gathers are random anyway, and block models: cfg 3 pads
    1.49, CSR 6188 vs 5337 it/s)."""
    if plan in (None, False, "csr"):
        return P
    if plan in (True, "cb"):
        return tsnet_plan_build(P, shard, stream)
    if plan == "sell":
        return tsnet_sell_build(P, shard, stream)
    if plan == "auto":
        _, ratio = tsnet_sell_query(P, shard, stream)
        return tsnet_sell_build(P, shard, stream) if ratio <= SELL_AUTO_MAX_SLOTS_PER_NNZ else P
    raise ValueError(f"unknown plan {plan!r}")


def tsnet_sell_build(P: CSR, shard=None, stream=None) -> CSR:
    """Build the sliced-ELL plan of P (set-up, blocking) and attach it: P.plan."""
    pbytes, _ = tsnet_sell_query(P, shard, stream)
    plan = torch.empty(max(pbytes, 1), dtype=torch.uint8, device=P.indptr.device)
    P.plan = None
    Pc = P.c()
    _check("tsnet_sell_build", lib().tsnet_sell_build(ctypes.byref(Pc), _shard(shard), _ptr(plan), pbytes,
                                                      _stream(stream)))
    P.plan = plan
    P.plan_kind = PLAN_SELL
    P.plan_rows = (0, P.n) if shard is None else _shard_rows(shard)
    return P


def tsnet_plan_partition(indptr_host, row_begin: int, row_end: int, groups: int = 148, rows_cap: int = 8192):
    """Host cut of the column-blocked plan (pure): rows into panels.  Returns
    (P, row_panel, row_local, panel_off, panel_rows) numpy arrays."""
    import numpy as np
    ip = np.ascontiguousarray(indptr_host, dtype=np.int64)
    nr = row_end - row_begin
    maxp = max(1, nr)
    row_panel = np.zeros(max(nr, 1), np.int32)
    row_local = np.zeros(max(nr, 1), np.int32)
    panel_off = np.zeros(maxp + 1, np.int32)
    panel_rows = np.zeros(max(nr, 1), np.int32)
    P = lib().tsnet_plan_partition(ip.ctypes.data, row_begin, row_end, groups, rows_cap, row_panel.ctypes.data,
                                   row_local.ctypes.data, panel_off.ctypes.data, panel_rows.ctypes.data, maxp)
    if P < 0:
        raise TsnetError("tsnet_plan_partition", P)
    return P, row_panel[:nr], row_local[:nr], panel_off[:P + 1], panel_rows[:nr]


# ------------------------------------------------------ per-iteration path
def tsnet_workspace_bytes(n: int, nnz: int, gp: GradParams, shard=None) -> int:
    g = gp.c()
    return int(lib().tsnet_workspace_bytes(n, nnz, ctypes.byref(g), _shard(shard)))


def alloc_workspace(n: int, nnz: int, gp: GradParams, device="cuda") -> torch.Tensor:
    """Zero-initialised workspace (the header must start zeroed)."""
    return torch.zeros(max(tsnet_workspace_bytes(n, nnz, gp), 1), dtype=torch.uint8, device=device)


def tsnet_grad(P: CSR, Y: torch.Tensor, gp: GradParams, ws: torch.Tensor, grad=None, Z=None, shard=None,
               stream=None):
    _require_cuda(Y, ws)
    grad = torch.empty_like(Y) if grad is None else grad
    Z = torch.empty(1, dtype=torch.float64, device=Y.device) if Z is None else Z
    Pc, g = P.c(), gp.c()
    _check("tsnet_grad", lib().tsnet_grad(ctypes.byref(Pc), _ptr(Y), ctypes.byref(g), _shard(shard), _ptr(grad),
                                          _ptr(Z), _ptr(ws), ws.numel(), _stream(stream)))
    return grad, Z


def tsnet_grad_tree(P: CSR, Y: torch.Tensor, gp: GradParams, ws: torch.Tensor, theta: float = 0.5, variant: int = 0,
                    tree_ws=None, grad=None, Z=None, stream=None):
    """Quadtree gradient: variant 0 = BH-tsNET, 1 = FIt-tsNET (tsnet_grad_tree)."""
    _require_cuda(Y, ws)
    grad = torch.empty_like(Y) if grad is None else grad
    Z = torch.empty(1, dtype=torch.float64, device=Y.device) if Z is None else Z
    if tree_ws is None:
        tree_ws = torch.empty(max(int(lib().tsnet_tree_workspace_bytes(Y.shape[0])), 1), dtype=torch.uint8,
                              device=Y.device)
    Pc, g = P.c(), gp.c()
    _check("tsnet_grad_tree", lib().tsnet_grad_tree(ctypes.byref(Pc), _ptr(Y), ctypes.byref(g), float(theta),
                                                    int(variant), _ptr(grad), _ptr(Z), _ptr(ws), ws.numel(),
                                                    _ptr(tree_ws), tree_ws.numel(), _stream(stream)))
    return grad, Z


def tsnet_attr(P: CSR, Y: torch.Tensor, f_attr=None, shard=None, stream=None):
    """Attractive SpMV alone (a6) for the shard's rows (all rows if None)."""
    _require_cuda(Y)
    if f_attr is None:
        rb, re = (0, P.n) if shard is None else _shard_rows(shard)
        f_attr = torch.empty((re - rb, 2), dtype=Y.dtype, device=Y.device)
    Pc = P.c()
    _check("tsnet_attr", lib().tsnet_attr(ctypes.byref(Pc), _ptr(Y), _shard(shard), _ptr(f_attr), _stream(stream)))
    return f_attr


def tsnet_grad_parts(P: CSR, Y: torch.Tensor, gp: GradParams, ws: torch.Tensor, shard=None, stream=None):
    _require_cuda(Y, ws)
    f_attr = torch.empty_like(Y)
    f_field = torch.empty_like(Y)
    Z = torch.empty(1, dtype=torch.float64, device=Y.device)
    Pc, g = P.c(), gp.c()
    _check("tsnet_grad_parts", lib().tsnet_grad_parts(ctypes.byref(Pc), _ptr(Y), ctypes.byref(g), _shard(shard),
                                                      _ptr(f_attr), _ptr(f_field), _ptr(Z), _ptr(ws), ws.numel(),
                                                      _stream(stream)))
    return f_attr, f_field, Z


def tsnet_step(P: CSR, Y, vel, gains, gp: GradParams, sp: StepParams, ws, shard=None, stream=None):
    _require_cuda(Y, vel, gains, ws)
    Pc, g, s = P.c(), gp.c(), sp.c()
    _check("tsnet_step", lib().tsnet_step(ctypes.byref(Pc), _ptr(Y), _ptr(vel), _ptr(gains), ctypes.byref(g),
                                          ctypes.byref(s), _shard(shard), _ptr(ws), ws.numel(), _stream(stream)))


def tsnet_step_host(P: CSR, Y_host, vel_host, gains_host, gp: GradParams, sp: StepParams, ws, shard=None,
                    stream=None):
    """One iteration with HOST state tensors (pinned CPU memory), H2D + D2H inside."""
    for t in (Y_host, vel_host, gains_host):
        assert not t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
    Pc, g, s = P.c(), gp.c(), sp.c()
    _check("tsnet_step_host", lib().tsnet_step_host(ctypes.byref(Pc), _ptr(Y_host), _ptr(vel_host),
                                                    _ptr(gains_host), ctypes.byref(g), ctypes.byref(s),
                                                    _shard(shard), _ptr(ws), ws.numel(), _stream(stream)))


def tsnet_cost(P: CSR, Y, gp: GradParams, ws, mode: int = 0, shard=None, stream=None):
    _require_cuda(Y, ws)
    out = torch.empty(3, dtype=torch.float64, device=Y.device)
    Pc, g = P.c(), gp.c()
    _check("tsnet_cost", lib().tsnet_cost(ctypes.byref(Pc), _ptr(Y), ctypes.byref(g), mode, _shard(shard),
                                          _ptr(out), _ptr(ws), ws.numel(), _stream(stream)))
    return out


def tsnet_read_stats(ws, stream=None) -> dict:
    st = tsnet_stats()
    rc = lib().tsnet_read_stats(_ptr(ws), ctypes.byref(st), _stream(stream))
    _check("tsnet_read_stats", rc, ok=(TSNET_OK, TSNET_E_NONFINITE))
    return {f: getattr(st, f) for f, _ in tsnet_stats._fields_}


# ------------------------------------------------------------ multi-GPU
class Shard:
    """Host-side shard description (rank, world, row bounds, NCCL communicator).
    `c()` gives the tsnet_shard struct; the bounds array is kept alive here."""

    def __init__(self, rank: int, world: int, bounds, comm=None):
        import numpy as np
        self.rank, self.world = int(rank), int(world)
        self.bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        assert len(self.bounds) == self.world + 1
        self.comm = comm
        self.row_begin, self.row_end = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self._c = tsnet_shard(self.rank, self.world, self.row_begin, self.row_end, comm,
                              self.bounds.ctypes.data_as(ctypes.POINTER(c_i64)))

    def c(self):
        return self._c


def _shard_rows(shard):
    s = shard.c() if isinstance(shard, Shard) else shard
    return int(s.row_begin), int(s.row_end)


def _shard(shard):
    if shard is None:
        return None
    if isinstance(shard, Shard):
        return ctypes.byref(shard.c())
    return ctypes.byref(shard)


def tsnet_shard_rows(indptr_host, world: int):
    """nnz + rows balanced contiguous row bounds (host, pure)."""
    import numpy as np
    ip = np.ascontiguousarray(indptr_host, dtype=np.int64)
    b = np.zeros(world + 1, np.int64)
    r = lib().tsnet_shard_rows(ip.ctypes.data, len(ip) - 1, world, b.ctypes.data)
    if r != world:
        raise TsnetError("tsnet_shard_rows", r)
    return b


def tsnet_comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check("tsnet_comm_unique_id", lib().tsnet_comm_unique_id(buf))
    return bytes(buf)


def tsnet_comm_init(uid: bytes, world: int, rank: int, I_max: int = TSNET_I_MAX_LIMIT):
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    comm = c_vp()
    _check("tsnet_comm_init", lib().tsnet_comm_init(buf, world, rank, int(I_max), ctypes.byref(comm)))
    return comm.value


def tsnet_comm_peer_reduce(comm) -> bool:
    return bool(lib().tsnet_comm_peer_reduce(comm))


class _DeviceArray:
    """A device buffer owned elsewhere (the communicator), exposed to torch
    through __cuda_array_interface__ (no copy, no ownership)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def tsnet_comm_layout(comm, n: int, device=None) -> torch.Tensor:
    """The communicator's own replicated layout buffer (n x 2 fp32, collective;
    valid until tsnet_comm_destroy).  tsnet_step on this tensor pushes the
    moved positions to the peers instead of all-gathering them."""
    ptr = c_vp()
    _check("tsnet_comm_layout", lib().tsnet_comm_layout(comm, int(n), ctypes.byref(ptr)))
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    return torch.as_tensor(_DeviceArray(ptr.value, (int(n), 2), "<f4"), device=dev)


def tsnet_comm_layout_push(comm) -> bool:
    return bool(lib().tsnet_comm_layout_push(comm))


def tsnet_comm_layout_sync(comm, stream=None):
    _check("tsnet_comm_layout_sync", lib().tsnet_comm_layout_sync(comm, _stream(stream)))


def tsnet_grids_sum(ws_list, n: int, nnz: int, gp: GradParams, stream=None):
    """Sum the live charge grids of several workspaces (one device) into each."""
    arr = (c_vp * len(ws_list))(*[w.data_ptr() for w in ws_list])
    g = gp.c()
    _check("tsnet_grids_sum", lib().tsnet_grids_sum(len(ws_list), arr, ws_list[0].numel(), n, nnz, ctypes.byref(g),
                                                    _stream(stream)))


def tsnet_comm_destroy(comm):
    _check("tsnet_comm_destroy", lib().tsnet_comm_destroy(comm))


def tsnet_ws_grid(n: int, nnz: int, gp: GradParams):
    off, cnt = c_sz(0), c_sz(0)
    g = gp.c()
    _check("tsnet_ws_grid", lib().tsnet_ws_grid(n, nnz, ctypes.byref(g), ctypes.byref(off), ctypes.byref(cnt)))
    return int(off.value), int(cnt.value)


def ws_grid_view(ws: torch.Tensor, n: int, nnz: int, gp: GradParams) -> torch.Tensor:
    """fp32 view of the charge grid inside a workspace (for external reduction)."""
    off, cnt = tsnet_ws_grid(n, nnz, gp)
    return ws[off:off + 4 * cnt].view(torch.float32)


def tsnet_field_local(P: CSR, Y, gp: GradParams, ws, shard=None, stream=None):
    _require_cuda(Y, ws)
    Pc, g = P.c(), gp.c()
    _check("tsnet_field_local", lib().tsnet_field_local(ctypes.byref(Pc), _ptr(Y), ctypes.byref(g), _shard(shard),
                                                        _ptr(ws), ws.numel(), _stream(stream)))


def tsnet_step_finish(P: CSR, Y, vel, gains, gp: GradParams, sp: StepParams, ws, shard=None, stream=None):
    _require_cuda(Y, vel, gains, ws)
    Pc, g, s = P.c(), gp.c(), sp.c()
    _check("tsnet_step_finish", lib().tsnet_step_finish(ctypes.byref(Pc), _ptr(Y), _ptr(vel), _ptr(gains),
                                                        ctypes.byref(g), ctypes.byref(s), _shard(shard), _ptr(ws),
                                                        ws.numel(), _stream(stream)))


def tsnet_last_error() -> str:
    return lib().tsnet_last_error().decode(errors="replace")
