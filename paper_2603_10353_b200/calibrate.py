"""Offline per-head budget table for a layer (the S-HPLB budget-allocation step).

Calibration rows (the last `rows` query rows of every head, which see the
whole context) are profiled into PerQueryTopK recovery curves on the grid
{0, 128, ..., n} (build_profiles, profiler.cpp:157-196: on the GPU profiler
when q/k are CUDA tensors and a context is given, else host C++), and the
max-min allocator (allocator.cpp:97-186) shifts budget from sparse to dense
heads starting from the uniform split of B = fraction * Hq * n tokens, in
128-token quanta with a 128-token floor, so every budget is a whole number of
128-key blocks.
"""
from __future__ import annotations

import time

import numpy as np

from . import api
from .workload import bf16_bits


def maxmin_budgets(q, k, fraction: float = 0.25, rows: int = 16, quantum: int = 128,
                   floor: int = 128, ctx=None):
    """q [Hq, n, d], k [Hkv, n, d] bf16 (any device) -> (budgets int64 [Hq], info dict).
    With ctx (an api.Context) and CUDA tensors the curves come from the GPU
    profiler, otherwise from the host one."""
    hq, n, _ = q.shape
    total = int(round(fraction * hq * n))
    t0 = time.time()
    grid = api.default_budget_grid(n, 128)
    if ctx is not None and getattr(q, "is_cuda", False):
        curves = ctx.profile_curves(q[:, n - rows:, :], k, grid)
    else:
        curves = api.profile_curves(bf16_bits(q[:, n - rows:, :]), bf16_bits(k), grid)
    alloc = api.maxmin_allocate(curves, total, quantum=quantum, floor=floor)
    info = {"total_tokens": total, "calibration_rows": rows,
            "profiler": "gpu" if ctx is not None and getattr(q, "is_cuda", False) else "host",
            "profile_s": round(time.time() - t0, 2), "transfers": alloc.transfers,
            "min_recovery_uniform": alloc.min_recovery_start,
            "min_recovery_maxmin": alloc.min_recovery_end}
    return alloc.budgets.astype(np.int64), info, curves


def uniform_budgets(hq: int, n: int, fraction: float = 0.25, floor: int = 128):
    """The same total split evenly (uniform_allocate, allocator.cpp:72-91)."""
    return api.uniform_allocate(hq, int(round(fraction * hq * n)), floor, n).budgets.astype(np.int64)
