"""Offline per-head budget table for a layer (the S-HPLB budget-allocation step).

Calibration: `rows` query rows evenly spaced through the
sequence (positions round(linspace(0, n-1, rows)), 128 by default) are
profiled into recovery curves on the grid {0, q, 2q, ..., n} (q = the
allocation quantum, the reference's grid_stride_of default), then the
max-min allocator (allocator.cpp:97-186) shifts budget from sparse to dense
heads starting from the uniform split of B = fraction * Hq * n tokens, in
q-token steps with a 128-token floor, so every budget is a whole number of
128-key blocks.

Curve kinds:
* "token"  — the reference's build_profiles(PerQueryTopK) (profiler.cpp:157-196):
             per-token top-k mass of each row over all n keys (no causal mask,
             as the reference's profile command). GPU profiler
             (shplb_profile_curves) or host C++; equal to the reference's to
             1e-12, so the table is the one the reference CLI would write.
* "colagg" — the same for ColumnAggregateTopK.
* "block"  — the kernels' own selection (shplb_profile_curves_block): causal
             rows, mass inside the key blocks kernel 2 keeps for the row's query
             block. The curve the layer call realises.
"""
from __future__ import annotations

import hashlib
import time

import numpy as np

from . import api
from .workload import bf16_bits

CURVE_KINDS = ("token", "colagg", "block")


def calibration_rows(n: int, rows: int = 128) -> np.ndarray:
    """Evenly spaced calibration row positions (strictly increasing)."""
    return np.unique(np.linspace(0, n - 1, min(rows, n)).round().astype(np.int64))


def table_digest(budgets) -> str:
    """Short digest of a budget table (int64 tokens), for comparing tables across runs."""
    return hashlib.sha256(np.ascontiguousarray(budgets, np.int64).tobytes()).hexdigest()[:16]


def profile_layer(q, k, *, kind: str = "token", rows: int = 128, quantum: int = 128, ctx=None,
                  block_q: int = api.BLOCK_Q):
    """Recovery curves of one layer. q [Hq, n, d], k [Hkv, n, d] bf16 (CUDA with
    ctx -> GPU profiler; host tensors -> host C++ profiler, token/colagg only)."""
    if kind not in CURVE_KINDS:
        raise ValueError(f"curve kind must be one of {CURVE_KINDS}")
    hq, n, _ = q.shape
    grid = api.default_budget_grid(n, quantum)
    pos = calibration_rows(n, rows)
    on_gpu = ctx is not None and getattr(q, "is_cuda", False)
    if kind == "block":
        if not on_gpu:
            raise ValueError("block-selection curves come from the GPU profiler (CUDA tensors and a context)")
        return ctx.profile_curves_block(q, k, pos, grid, block_q=block_q, causal=True), pos
    sel = 0 if kind == "token" else 1
    if on_gpu:
        import torch
        idx = torch.as_tensor(pos, device=q.device)
        return ctx.profile_curves(q.index_select(1, idx).contiguous(), k, grid, kind=sel), pos
    return api.profile_curves(bf16_bits(q[:, pos, :]), bf16_bits(k), grid, kind=sel), pos


def layer_budgets(q, k, fraction: float = 0.25, *, kind: str = "token", rows: int = 128,
                  quantum: int = 128, floor: int = 128, ctx=None, block_q: int = api.BLOCK_Q):
    """(budgets int64 [Hq], info dict, curves): max-min table of one layer."""
    hq, n, _ = q.shape
    total = int(round(fraction * hq * n))
    t0 = time.time()
    curves, pos = profile_layer(q, k, kind=kind, rows=rows, quantum=quantum, ctx=ctx, block_q=block_q)
    alloc = api.maxmin_allocate(curves, total, quantum=quantum, floor=floor)
    budgets = alloc.budgets.astype(np.int64)
    info = {"total_tokens": total, "curve_kind": kind, "calibration_rows": int(pos.size),
            "calibration": f"{pos.size} rows evenly spaced over [0, {n - 1}]",
            "grid_stride": quantum, "quantum": quantum, "floor": floor,
            "profiler": "gpu" if ctx is not None and getattr(q, "is_cuda", False) else "host",
            "profile_s": round(time.time() - t0, 3), "transfers": alloc.transfers,
            "min_recovery_uniform": alloc.min_recovery_start,
            "min_recovery_maxmin": alloc.min_recovery_end, "digest": table_digest(budgets)}
    return budgets, info, curves


def maxmin_budgets(q, k, fraction: float = 0.25, rows: int = 128, quantum: int = 128,
                   floor: int = 128, ctx=None, kind: str = "token"):
    """Compatibility wrapper of layer_budgets (token-level curves by default)."""
    return layer_budgets(q, k, fraction, kind=kind, rows=rows, quantum=quantum, floor=floor, ctx=ctx)


def uniform_budgets(hq: int, n: int, fraction: float = 0.25, floor: int = 128):
    """The same total split evenly (uniform_allocate, allocator.cpp:72-91)."""
    return api.uniform_allocate(hq, int(round(fraction * hq * n)), floor, n).budgets.astype(np.int64)
