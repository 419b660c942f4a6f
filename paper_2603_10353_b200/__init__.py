"""B200-native S-HPLB sparse-attention hot path (arXiv 2603.10353).

Host API over libshplb.so (C ABI: include/shplb.h). See DESIGN.md.
"""
from ._native import (CudaError, InvalidArgument, LogicError, NcclError, NotSupported, ShplbError,
                      ShplbRuntimeError, build, lib)
from .api import (BLOCK, BLOCK_Q, BLOCK_TOPK, COLUMN_AGGREGATE_TOPK, HEAD_DIM, BudgetAllocation, Context, LoadReport, RecoveryCurve,
                  NcclComm, OutSegment, SimulationResult, barrier, plan_segments, default_budget_grid, greedy_assign, imbalance,
                  layer_work, maxmin_allocate, naive_assign, optimal_assign, profile_curves, refine_assign, simulate,
                  selection_kind, split_assign, tile_costs, top_p_budgets, uniform_allocate)
from . import formats  # noqa: E402  (allocation / assignment / profiles JSON, reference layout)
from . import experiments  # noqa: E402  (sweep / skyline on measured latency)

__all__ = [
    "BLOCK", "BLOCK_Q", "HEAD_DIM", "BudgetAllocation", "Context", "CudaError", "InvalidArgument",
    "LoadReport", "LogicError", "NotSupported", "RecoveryCurve", "ShplbError", "ShplbRuntimeError",
    "SimulationResult",
    "barrier", "build", "default_budget_grid", "greedy_assign", "imbalance", "layer_work", "lib",
    "maxmin_allocate", "naive_assign", "optimal_assign", "profile_curves", "simulate", "split_assign",
    "uniform_allocate", "top_p_budgets", "selection_kind", "BLOCK_TOPK", "COLUMN_AGGREGATE_TOPK",
    "NcclComm", "NcclError", "OutSegment", "plan_segments", "tile_costs", "refine_assign",
]
