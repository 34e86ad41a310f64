"""B200-native L-tsNET gradient hot path (arXiv 2509.19785).

The product is libtsnet.so (CUDA kernels for sm_100a behind the C-ABI in
include/tsnet.h); this package is its thin ctypes binding plus the iteration
driver.  Importing the package does not load the library; the first call does
and raises if it is missing (no CPU fallback).
"""
from .tsnet import (CSR, GradParams, attach_plan, StepParams, TsnetError, alloc_workspace, lib, tsnet_attr, tsnet_build_P,  # noqa: F401
                    tsnet_build_P_workspace_bytes, tsnet_cost, tsnet_grad, tsnet_grad_parts, tsnet_grad_tree, tsnet_last_error,
                    tsnet_plan_build, tsnet_plan_partition, tsnet_plan_query, tsnet_pmds, tsnet_read_stats, tsnet_resolve_k,
                    tsnet_move, tsnet_quality, tsnet_sell_build, tsnet_sell_query, tsnet_step, tsnet_step_host, tsnet_workspace_bytes)
from .runner import Layout, stage_of, stage_params  # noqa: F401
