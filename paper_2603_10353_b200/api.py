"""Python face of the B200 hot path, mirroring the reference operator API.

Names and argument meanings follow the reference's ``headbal`` namespace
(/root/reference/proj/include/headbal/*.hpp): the per-head budget table
(``uniform_allocate``, ``maxmin_allocate``), the head->GPU plan
(``naive_assign``, ``greedy_assign``, ``imbalance``), the barrier metric
(``simulate``, ``barrier``) and the sparse-attention entry point
(``sparse_attention_layer`` — the per-head-budget loop of ``run_skyline``
around ``sparse_attention``). Errors raise ``InvalidArgument`` (a
``ValueError``) where the reference throws ``std::invalid_argument``, with the
reference's message text.

Everything computes in libshplb.so (C++ host code and sm_100a kernels). torch
is used only to hold device memory and name the CUDA stream.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from ._native import (LayerShape, MaxminDiag, check, lib)

BLOCK = 128      # key block (pooling and K/V tile): 128 keys
BLOCK_Q = 256    # default query block: two 128-row halves share every K/V tile
HEAD_DIM = 128


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------------------
# Budget table (allocator.hpp)
# ---------------------------------------------------------------------------

@dataclass
class RecoveryCurve:
    """profiler.hpp:29-41 — sampled budget -> recovery, ending at (n_k, 1)."""
    budgets: np.ndarray
    recovery: np.ndarray
    context_length: int

    def recovery_at(self, budget: int) -> float:
        out = C.c_double()
        b, r = _i64(self.budgets), _f64(self.recovery)
        check(lib().shplb_recovery_at(b.size, _ptr(b), _ptr(r), int(budget), C.byref(out)))
        return float(out.value)

    def budget_for_recovery(self, p: float) -> int:
        """budget_for_recovery (profiler.cpp:198-209): smallest sampled budget
        reaching recovery p — a per-head top-p budget fixed offline."""
        out = C.c_int64()
        b, r = _i64(self.budgets), _f64(self.recovery)
        check(lib().shplb_budget_for_recovery(b.size, _ptr(b), _ptr(r), int(self.context_length), float(p),
                                              C.byref(out)))
        return int(out.value)


def top_p_budgets(curves, p: float) -> np.ndarray:
    """Per-head budgets of an offline top-p policy (the paper's top-p comparison,
    PAPER.md:174-177): each head gets the budget its own curve needs to reach
    recovery p, so the total and the per-head loads are whatever p implies."""
    return np.asarray([c.budget_for_recovery(p) for c in curves], np.int64)


@dataclass
class BudgetAllocation:
    """allocator.hpp:23-38 (budgets in tokens) plus the diagnostics."""
    budgets: np.ndarray
    total: int
    floor: int
    transfers: int = 0
    hit_iteration_cap: bool = False
    off_grid_evaluations: int = 0
    min_recovery_start: float = 0.0
    min_recovery_end: float = 0.0


def uniform_allocate(num_heads: int, total: int, floor: int, context_length: int) -> BudgetAllocation:
    out = np.empty(num_heads, np.int64)
    check(lib().shplb_uniform_allocate(num_heads, total, floor, context_length, _ptr(out)))
    return BudgetAllocation(out, total, floor)


def maxmin_allocate(curves: Sequence[RecoveryCurve], total: int, quantum: int = 64,
                    floor: int = 128, max_iterations: int = 0) -> BudgetAllocation:
    """Max-min budget shifting (allocator.hpp:53-54); bit-exact with the reference."""
    if len(curves) == 0:
        from ._native import InvalidArgument
        raise InvalidArgument("need at least one recovery curve")
    n_k = int(curves[0].context_length)
    for c in curves:
        if int(c.context_length) != n_k:
            from ._native import InvalidArgument
            raise InvalidArgument("all curves must share the context length")
    offsets = np.zeros(len(curves) + 1, np.int64)
    for h, c in enumerate(curves):
        offsets[h + 1] = offsets[h] + len(c.budgets)
    pb = _i64(np.concatenate([np.asarray(c.budgets) for c in curves]))
    pr = _f64(np.concatenate([np.asarray(c.recovery) for c in curves]))
    out = np.empty(len(curves), np.int64)
    diag = MaxminDiag()
    check(lib().shplb_maxmin_allocate(len(curves), n_k, _ptr(offsets), _ptr(pb), _ptr(pr), total,
                                      quantum, floor, max_iterations, _ptr(out), C.byref(diag)))
    return BudgetAllocation(out, total, floor, int(diag.transfers), bool(diag.hit_iteration_cap),
                            int(diag.off_grid_evaluations), float(diag.min_recovery_start),
                            float(diag.min_recovery_end))


def default_budget_grid(context_length: int, stride: int) -> np.ndarray:
    """profiler.cpp:385-392: {0, stride, 2*stride, ..., n_k}."""
    g = list(range(0, context_length, stride)) + [context_length]
    return np.asarray(g, np.int64)


def profile_curves(q_rows_bf16: np.ndarray, k_bf16: np.ndarray, grid: np.ndarray,
                   kind=0) -> list[RecoveryCurve]:
    """Recovery curves (build_profiles, profiler.cpp:157-196) from calibration
    query rows for selection `kind` (PerQueryTopK = 0 / "per_query_topk",
    ColumnAggregateTopK = 1 / "column_aggregate_topk"). q_rows_bf16: uint16
    [Hq][rows][d]; k_bf16: uint16 [Hkv][n_k][d] (bf16 bit patterns, host).
    Host C++, OpenMP."""
    q = np.ascontiguousarray(q_rows_bf16, np.uint16)
    k = np.ascontiguousarray(k_bf16, np.uint16)
    grid = _i64(grid)
    hq, rows, d = q.shape
    hkv, n_k, _ = k.shape
    out = np.empty((hq, grid.size), np.float64)
    check(lib().shplb_profile_curves_host_kind(_ptr(q), _ptr(k), hq, hkv, rows, n_k, d, _ptr(grid),
                                               grid.size, selection_kind(kind), _ptr(out)))
    return [RecoveryCurve(grid.copy(), out[h].copy(), n_k) for h in range(hq)]


# ---------------------------------------------------------------------------
# Head -> GPU plan (partitioner.hpp) and metric (simulator.hpp)
# ---------------------------------------------------------------------------

@dataclass
class LoadReport:
    """partitioner.hpp:25-30."""
    loads: np.ndarray
    total: int
    imbalance: float
    argmax_device: int


def naive_assign(budgets, devices: int, round_robin: bool = False) -> np.ndarray:
    b = _i64(budgets)
    out = np.empty(b.size, np.int32)
    check(lib().shplb_plan_naive(_ptr(b), b.size, devices, int(round_robin), _ptr(out)))
    return out


def greedy_assign(budgets, devices: int) -> np.ndarray:
    b = _i64(budgets)
    out = np.empty(b.size, np.int32)
    check(lib().shplb_plan_greedy(_ptr(b), b.size, devices, _ptr(out)))
    return out


def refine_assign(costs, devices: int, device_of_head=None) -> np.ndarray:
    """Whole-head local search on per-head costs (shplb_plan_refine; an extension
    beyond greedy_assign, partitioner.cpp:164-183): starting from device_of_head
    (default: greedy_assign(costs)), move or swap heads off the most loaded device
    while that lowers the maximum load. Returns the refined device_of_head."""
    c = _i64(costs)
    start = greedy_assign(c, devices) if device_of_head is None else device_of_head
    out = np.ascontiguousarray(start, np.int32).copy()
    if out.size != c.size:
        from ._native import InvalidArgument
        raise InvalidArgument(f"assignment covers {out.size} heads but {c.size} costs were given")
    check(lib().shplb_plan_refine(_ptr(c), c.size, devices, _ptr(out), None))
    return out


def optimal_assign(budgets, devices: int) -> np.ndarray:
    """optimal_assign (partitioner.cpp:185-234): minimum makespan, then the
    lexicographically smallest plan reaching it (N <= 24, D <= 4)."""
    b = _i64(budgets)
    out = np.empty(b.size, np.int32)
    check(lib().shplb_plan_optimal(_ptr(b), b.size, devices, _ptr(out)))
    return out


def imbalance(budgets, device_of_head, devices: int) -> LoadReport:
    b, a = _i64(budgets), _i32(device_of_head)
    if a.size != b.size:
        from ._native import InvalidArgument
        raise InvalidArgument(f"assignment covers {a.size} heads but {b.size} budgets were given")
    loads = np.empty(devices, np.int64)
    tot, imb, am = C.c_int64(), C.c_double(), C.c_int32()
    check(lib().shplb_imbalance(_ptr(b), b.size, _ptr(a), devices, _ptr(loads), C.byref(tot),
                                C.byref(imb), C.byref(am)))
    return LoadReport(loads, int(tot.value), float(imb.value), int(am.value))


@dataclass
class SplitPlan:
    """Sub-head plan (shplb_plan_split): segment i puts query blocks
    [qb_begin[i], qb_end[i]) of head `head[i]` on `device[i]`."""
    device: np.ndarray
    head: np.ndarray
    qb_begin: np.ndarray
    qb_end: np.ndarray
    loads: np.ndarray  # per-device cost in 128x128 tiles


def split_assign(budgets, devices: int, seq_len: int, block_q: int = BLOCK_Q,
                 causal: bool = True, query_tile_weight: int = 0) -> SplitPlan:
    """Sub-head balancer: whole heads in index order, cut at query-block
    boundaries so every device's tile cost (+ query_tile_weight per visited
    query half: shplb_plan_split_weighted) is within half a query block of
    total/devices (at most devices-1 heads are split)."""
    b = _i64(budgets)
    cap = b.size + devices
    dev, hd, qb0, qb1 = (np.empty(cap, np.int32) for _ in range(4))
    loads = np.empty(devices, np.int64)
    ns = C.c_int32()
    check(lib().shplb_plan_split_weighted(_ptr(b), b.size, seq_len, block_q, int(causal), devices,
                                          int(query_tile_weight), cap, _ptr(dev), _ptr(hd), _ptr(qb0),
                                          _ptr(qb1), C.byref(ns), _ptr(loads)))
    k = ns.value
    return SplitPlan(dev[:k].copy(), hd[:k].copy(), qb0[:k].copy(), qb1[:k].copy(), loads)


# Kernel 3's fixed cost per (query block, query half) it visits, in tile
# equivalents: a least-squares fit of measured per-rank shard times gives 3.4
# (C3, 128K) and 5.1 (C4, 64K) next to ~6.4 ns per tile (tools/plan_fit.py,
# profiles/r02/plan_fit_C3.txt). For whole heads it is a per-head constant.
QUERY_TILE_WEIGHT = 4


def tile_costs(budgets, seq_len: int, block_q: int = BLOCK_Q, causal: bool = True,
               query_tile_weight: int = 0) -> np.ndarray:
    """Per-head cost in kernel 3's 128x128 tiles: sum over query blocks of
    min(ceil(b_h/128), visible key blocks) x query halves holding rows — the
    work the layer call does for the head (shplb_layer_work per head) — plus
    query_tile_weight per visited query half (QUERY_TILE_WEIGHT models the
    per-tile fixed cost). Passed to greedy_assign instead of the budgets it is
    the documented extension of SURVEY a11 (the same LPT, weighted by causal
    tile cost rather than tokens)."""
    b = np.asarray(budgets, np.int64)
    nkb = (seq_len + BLOCK - 1) // BLOCK
    nqb = (seq_len + block_q - 1) // block_q
    qb = np.arange(nqb)
    last = np.minimum((qb + 1) * block_q, seq_len) - 1
    vis = np.minimum(last // BLOCK + 1, nkb) if causal else np.full(nqb, nkb)
    halves = np.array([sum(1 for hf in range(block_q // BLOCK) if q * block_q + hf * BLOCK < seq_len) for q in qb])
    kb = np.minimum((b + BLOCK - 1) // BLOCK, nkb)
    t = np.minimum(kb[:, None], vis[None, :]) * halves[None, :]
    return (t.sum(1) + int(query_tile_weight) * ((t > 0) * halves[None, :]).sum(1)).astype(np.int64)


@dataclass
class SimulationResult:
    """simulator.hpp:20-25."""
    device_latency: np.ndarray
    barrier_latency: float
    bubble_fraction: float


def simulate(loads, alpha: float = 0.0, beta: float = 1.0) -> SimulationResult:
    ld = _i64(loads)
    lat = np.empty(ld.size, np.float64)
    b, bub = C.c_double(), C.c_double()
    check(lib().shplb_simulate(_ptr(ld), ld.size, alpha, beta, _ptr(lat), C.byref(b), C.byref(bub)))
    return SimulationResult(lat, float(b.value), float(bub.value))


def barrier(device_latency) -> SimulationResult:
    """Barrier latency and bubble over MEASURED per-device latencies."""
    lat = _f64(device_latency)
    b, bub = C.c_double(), C.c_double()
    check(lib().shplb_barrier(_ptr(lat), lat.size, C.byref(b), C.byref(bub)))
    return SimulationResult(lat, float(b.value), float(bub.value))


# ---------------------------------------------------------------------------
# Sparse attention on the GPU (attention.hpp)
# ---------------------------------------------------------------------------

BLOCK_TOPK = 0               # SHPLB_BLOCK_TOPK: PerQueryTopK at block granularity
COLUMN_AGGREGATE_TOPK = 1    # SHPLB_COLUMN_AGGREGATE_TOPK: one kept key-block set per head
_KINDS = {"per_query_topk": BLOCK_TOPK, "column_aggregate_topk": COLUMN_AGGREGATE_TOPK}


def selection_kind(kind) -> int:
    """SHPLB_* selection kind from an int or the reference's policy name
    (selection_kind_from_string, workload.cpp:12-17, same error text)."""
    if isinstance(kind, str):
        if kind not in _KINDS:
            from ._native import InvalidArgument
            raise InvalidArgument(f'unknown selection policy "{kind}" '
                                  "(expected per_query_topk or column_aggregate_topk)")
        return _KINDS[kind]
    return int(kind)


def _shape(num_q_heads, num_kv_heads, seq_len, causal, validate=False, kv_map=None,
           head_dim=HEAD_DIM, block_q=BLOCK_Q, q_block_range=None, gather=None,
           kind=BLOCK_TOPK) -> LayerShape:
    sh = LayerShape(num_q_heads, num_kv_heads, seq_len, head_dim, block_q, BLOCK, int(causal),
                    selection_kind(kind), int(validate), None, None, None, 0, None, 0)
    if gather is not None:  # (output buffer device pointers, global head of each local q head, total heads)
        ptrs, head_of_q, total = gather
        arr = (C.c_void_p * len(ptrs))(*[int(x) for x in ptrs])
        hq_ = _i32(head_of_q)
        sh._gather_keepalive = (arr, hq_)
        sh.out_peers = C.cast(arr, C.c_void_p)
        sh.n_out_peers = len(ptrs)
        sh.out_head_of_q = hq_.ctypes.data
        sh.out_heads_total = int(total)
    if kv_map is not None:
        m = _i32(kv_map)
        sh._kv_map_keepalive = m  # the C struct only borrows the pointer
        sh.kv_head_of_q = m.ctypes.data
    if q_block_range is not None:
        r = _i32(np.asarray(q_block_range).reshape(-1))
        sh._range_keepalive = r
        sh.q_block_range = r.ctypes.data
    return sh


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dev_ptr(t, name, dtype=None):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        from ._native import InvalidArgument
        raise InvalidArgument(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        from ._native import InvalidArgument
        raise InvalidArgument(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        from ._native import InvalidArgument
        raise InvalidArgument(f"{name} must be contiguous")
    return C.c_void_p(t.data_ptr())


class Context:
    """shplb_ctx: per-device workspace. One per rank/device."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        check(lib().shplb_ctx_create(device, C.byref(self._h)))
        self.device = device

    def close(self) -> None:
        if self._h:
            check(lib().shplb_ctx_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(lib().shplb_ctx_launch_count(self._h))

    def set_timing(self, enable: bool) -> None:
        """Record per-kernel CUDA events in every layer call (see read_timing)."""
        check(lib().shplb_ctx_set_timing(self._h, int(enable)))

    def read_timing(self, max_calls: int = 4096) -> np.ndarray:
        """[calls, 3] ms of (kernel 1 pooling, kernel 2 score+select, kernel 3
        attention) per layer call since timing was enabled / last read."""
        buf = np.zeros((max_calls, 3), np.float64)
        n = C.c_int()
        check(lib().shplb_ctx_read_timing(self._h, _ptr(buf), max_calls, C.byref(n)))
        return buf[:n.value].copy()

    # -- offline profiler (GPU) ---------------------------------------------
    def profile_curves(self, q_rows, k, grid, stream=None, kind=0) -> list[RecoveryCurve]:
        """Recovery curves for selection `kind` on the GPU (shplb_profile_curves_kind;
        build_profiles + recovery_ratio, profiler.cpp:157-196,
        attention.cpp:151-184). q_rows: bf16 CUDA [Hq, rows, d] (the
        calibration rows), k: bf16 CUDA [Hkv, n_k, d]. Same results as the
        host profile_curves() to rounding."""
        import torch
        q_rows = q_rows.contiguous()
        k = k.contiguous()
        _dev_ptr(q_rows, "q_rows", torch.bfloat16)
        _dev_ptr(k, "k", torch.bfloat16)
        grid = _i64(grid)
        hq, rows, d = q_rows.shape
        hkv, n_k, _ = k.shape
        out = np.empty((hq, grid.size), np.float64)
        check(lib().shplb_profile_curves_kind(self._h, q_rows.data_ptr(), k.data_ptr(), hq, hkv, rows, n_k, d,
                                              _ptr(grid), grid.size, selection_kind(kind), _ptr(out),
                                              _stream_ptr(stream)))
        return [RecoveryCurve(grid.copy(), out[h].copy(), n_k) for h in range(hq)]

    def profile_curves_block(self, q, k, rows, grid, block_q=BLOCK_Q, causal=True,
                             stream=None) -> list[RecoveryCurve]:
        """Recovery curves of the kernels' own block selection
        (shplb_profile_curves_block): per q head, the mean over calibration rows
        (positions `rows`, strictly increasing) of the exact softmax mass inside
        the ceil(b/128) key blocks kernel 2 keeps for the row's query block.
        q [Hq, n, d], k [Hkv, n, d] bf16 CUDA (the whole layer)."""
        import torch
        q = q.contiguous()
        k = k.contiguous()
        _dev_ptr(q, "q", torch.bfloat16)
        _dev_ptr(k, "k", torch.bfloat16)
        grid = _i64(grid)
        rows = _i64(rows)
        hq, n, d = q.shape
        out = np.empty((hq, grid.size), np.float64)
        check(lib().shplb_profile_curves_block(self._h, q.data_ptr(), k.data_ptr(), hq, k.shape[0], n, d,
                                               block_q, int(bool(causal)), _ptr(rows), rows.size, _ptr(grid),
                                               grid.size, _ptr(out), _stream_ptr(stream)))
        return [RecoveryCurve(grid.copy(), out[h].copy(), n) for h in range(hq)]

    # -- kernel 1 ---------------------------------------------------------
    def block_scores(self, q, k, causal=True, stream=None, validate=False, out=None, kv_map=None,
                     block_q=BLOCK_Q):
        import torch
        hq, n, d = q.shape
        hkv = k.shape[0]
        nqb, nkb = (n + block_q - 1) // block_q, (n + BLOCK - 1) // BLOCK
        if out is None:
            out = torch.empty((hq, nqb, nkb), dtype=torch.float32, device=q.device)
        sh = _shape(hq, hkv, n, causal, validate, kv_map, d, block_q)
        check(lib().shplb_block_scores(self._h, C.byref(sh), _dev_ptr(q, "q", torch.bfloat16),
                                       _dev_ptr(k, "k", torch.bfloat16),
                                       _dev_ptr(out, "scores", torch.float32), _stream_ptr(stream)))
        return out

    # -- kernel 2 ---------------------------------------------------------
    def select_blocks(self, scores, k_blocks, n, causal=True, kmax=None, stream=None,
                      block_q=BLOCK_Q, kind=BLOCK_TOPK):
        import torch
        hq, nqb, _ = scores.shape
        kb = _i64(k_blocks)
        kmax = int(kb.max()) if kmax is None else int(kmax)
        idx = torch.empty((hq, nqb, kmax), dtype=torch.int32, device=scores.device)
        cnt = torch.empty((hq, nqb), dtype=torch.int32, device=scores.device)
        sh = _shape(hq, 1, n, causal, block_q=block_q, kind=kind)
        sh.num_kv_heads = 1
        check(lib().shplb_select_blocks(self._h, C.byref(sh), _dev_ptr(scores, "scores", torch.float32),
                                        _ptr(kb), kmax, _dev_ptr(idx, "idx"), _dev_ptr(cnt, "cnt"),
                                        _stream_ptr(stream)))
        return idx, cnt

    # -- kernel 3 ---------------------------------------------------------
    def block_sparse_attention(self, q, k, v, idx, cnt, causal=True, stream=None, out=None,
                               kv_map=None, block_q=BLOCK_Q):
        import torch
        hq, n, d = q.shape
        if out is None:
            out = torch.empty_like(q)
        sh = _shape(hq, k.shape[0], n, causal, kv_map=kv_map, head_dim=d, block_q=block_q)
        check(lib().shplb_block_sparse_attention(
            self._h, C.byref(sh), _dev_ptr(q, "q", torch.bfloat16), _dev_ptr(k, "k", torch.bfloat16),
            _dev_ptr(v, "v", torch.bfloat16), _dev_ptr(idx, "idx", torch.int32),
            _dev_ptr(cnt, "cnt", torch.int32), int(idx.shape[-1]), _dev_ptr(out, "out", torch.bfloat16),
            _stream_ptr(stream)))
        return out

    # -- the layer: kernels 1+2 fused, then 3 -----------------------------
    def sparse_attention_layer(self, q, k, v, budgets_tokens, causal=True, stream=None, out=None,
                               validate=False, kv_map=None, block_q=BLOCK_Q, q_block_range=None,
                               gather=None, kind=BLOCK_TOPK):
        """sparse_attention for every head with its own token budget under selection
        `kind` (BLOCK_TOPK / COLUMN_AGGREGATE_TOPK or the policy name). gather =
        (device pointers of full output buffers, global head index of each local
        q head, total heads): kernel 3 writes every output row into each buffer
        (fused head-parallel gather over NVLink peer memory); `out` is unused."""
        import torch
        hq, n, d = q.shape
        b = _i64(budgets_tokens)
        if b.size != hq:
            from ._native import InvalidArgument
            raise InvalidArgument(f"need one budget per query head ({hq}), got {b.size}")
        sh = _shape(hq, k.shape[0], n, causal, validate, kv_map, d, block_q, q_block_range, gather, kind)
        self._last_block_q = block_q
        if gather is not None:
            out_ptr = None
        else:
            if out is None:
                out = torch.empty_like(q)
            out_ptr = _dev_ptr(out, "out", torch.bfloat16)
        check(lib().shplb_sparse_attention_layer(
            self._h, C.byref(sh), _dev_ptr(q, "q", torch.bfloat16), _dev_ptr(k, "k", torch.bfloat16),
            _dev_ptr(v, "v", torch.bfloat16), _ptr(b), out_ptr, _stream_ptr(stream)))
        return out

    def dense_attention_layer(self, q, k, v, causal=True, stream=None, out=None, validate=False,
                              kv_map=None, block_q=BLOCK_Q):
        """Dense comparator (shplb_dense_attention_layer): every head over every
        causally visible key, through the same sm_100a kernel 3."""
        import torch
        hq, n, d = q.shape
        if out is None:
            out = torch.empty_like(q)
        sh = _shape(hq, k.shape[0], n, causal, validate, kv_map, d, block_q, None)
        check(lib().shplb_dense_attention_layer(
            self._h, C.byref(sh), _dev_ptr(q, "q", torch.bfloat16), _dev_ptr(k, "k", torch.bfloat16),
            _dev_ptr(v, "v", torch.bfloat16), _dev_ptr(out, "out", torch.bfloat16), _stream_ptr(stream)))
        return out

    def sparse_attention_layer_host(self, q, k, v, budgets_tokens, causal=True, out=None,
                                    stream=None, kv_map=None, block_q=BLOCK_Q, q_block_range=None,
                                    asynchronous=False, kind=BLOCK_TOPK):
        """The layer call on HOST bf16 tensors (pinned for async DMA): copy in,
        kernels 1-3, copy out, synchronise (shplb_sparse_attention_layer_host). With
        asynchronous=True nothing is synchronised (shplb_sparse_attention_layer_host_async):
        consecutive calls overlap one layer's copies with the previous layer's work;
        `out` is valid once `stream` completes."""
        import torch
        for t, nm in ((q, "q"), (k, "k"), (v, "v")):
            if t.is_cuda or t.dtype != torch.bfloat16 or not t.is_contiguous():
                from ._native import InvalidArgument
                raise InvalidArgument(f"{nm} must be a contiguous host bf16 tensor")
        hq, n, d = q.shape
        if out is None:
            out = torch.empty_like(q)
        b = _i64(budgets_tokens)
        if b.size != hq:
            from ._native import InvalidArgument
            raise InvalidArgument(f"need one budget per query head ({hq}), got {b.size}")
        sh = _shape(hq, k.shape[0], n, causal, False, kv_map, d, block_q, q_block_range, kind=kind)
        self._last_block_q = block_q
        fn = (lib().shplb_sparse_attention_layer_host_async if asynchronous
              else lib().shplb_sparse_attention_layer_host)
        check(fn(
            self._h, C.byref(sh), C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()),
            C.c_void_p(v.data_ptr()), _ptr(b), C.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def last_selection_work(self):
        """(tiles, FLOPs) kernel 3 computed in the last layer call (exact; syncs)."""
        t, f = C.c_int64(), C.c_double()
        check(lib().shplb_last_selection_work(self._h, C.byref(t), C.byref(f)))
        return int(t.value), float(f.value)

    def last_selection(self, num_q_heads: int, seq_len: int):
        """(idx, cnt) of the last layer call as torch views over the context workspace."""
        import torch
        ip, cp, km = C.c_void_p(), C.c_void_p(), C.c_int64()
        check(lib().shplb_last_selection(self._h, C.byref(ip), C.byref(cp), C.byref(km)))
        bq = getattr(self, "_last_block_q", BLOCK_Q)
        nqb = (seq_len + bq - 1) // bq
        kmax = int(km.value)
        idx = torch.empty((num_q_heads, nqb, kmax), dtype=torch.int32, device=f"cuda:{self.device}")
        cnt = torch.empty((num_q_heads, nqb), dtype=torch.int32, device=f"cuda:{self.device}")
        check(lib().shplb_copy_last_selection(self._h, C.c_void_p(idx.data_ptr()), idx.numel(),
                                              C.c_void_p(cnt.data_ptr()), cnt.numel(),
                                              _stream_ptr(None)))
        return idx, cnt


def layer_work(num_q_heads, num_kv_heads, seq_len, budgets_tokens, causal=True, kv_map=None,
               block_q=BLOCK_Q):
    """(128x128 tiles, algorithmic FLOPs 4*d*128*128*tiles) of one layer call, before
    selection: selected key blocks x live 128-row query halves (include/shplb.h)."""
    sh = _shape(num_q_heads, num_kv_heads, seq_len, causal, kv_map=kv_map, block_q=block_q)
    b = _i64(budgets_tokens)
    t, f = C.c_int64(), C.c_double()
    check(lib().shplb_layer_work(C.byref(sh), _ptr(b), C.byref(t), C.byref(f)))
    return int(t.value), float(f.value)


# ---------------------------------------------------------------------------
# Head parallelism across ranks: NCCL communicator + output reassembly
# (shplb_nccl_*, shplb_gather_segments / shplb_gather_heads, shplb_comm_barrier)
# ---------------------------------------------------------------------------

class OutSegment(C.Structure):
    """shplb_out_segment: rows [row_begin, row_end) of global head `head`, computed
    by rank `owner` at its local head index `local_head`."""
    _fields_ = [("head", C.c_int32), ("owner", C.c_int32), ("local_head", C.c_int32),
                ("reserved", C.c_int32), ("row_begin", C.c_int64), ("row_end", C.c_int64)]


def plan_segments(plan, world: int, num_heads: int, seq_len: int, block_q: int = BLOCK_Q):
    """Output segments of a whole-head plan (device_of_head) or a sub-head plan
    (split_assign result): every rank's heads in ascending order (its local
    layout), each with the rows it computes."""
    segs = []
    if isinstance(plan, SplitPlan):  # sub-head plan
        for r in range(world):
            sel = [i for i in range(len(plan.device)) if int(plan.device[i]) == r]
            sel.sort(key=lambda i: int(plan.head[i]))
            for li, i in enumerate(sel):
                r0 = int(plan.qb_begin[i]) * block_q
                r1 = min(int(plan.qb_end[i]) * block_q, seq_len)
                if r1 > r0:
                    segs.append((int(plan.head[i]), r, li, r0, r1))
    else:
        dev = np.asarray(plan)
        for r in range(world):
            for li, h in enumerate(np.nonzero(dev == r)[0].tolist()):
                segs.append((h, r, li, 0, seq_len))
    arr = (OutSegment * len(segs))()
    for i, (h, o, li, r0, r1) in enumerate(segs):
        arr[i] = OutSegment(h, o, li, 0, r0, r1)
    return arr


class NcclComm:
    """An NCCL communicator of the library (shplb_nccl_comm_init) for the
    head-parallel reassembly and barrier. Rank 0 makes the unique id
    (NcclComm.unique_id()) and the host ships it to every rank."""

    def __init__(self, device: int, nranks: int, rank: int, unique_id: bytes):
        self.device, self.nranks, self.rank = device, nranks, rank
        self._h = C.c_void_p()
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(lib().shplb_nccl_comm_init(device, nranks, rank, buf, 128, C.byref(self._h)))

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().shplb_nccl_get_unique_id(buf, 128))
        return buf.raw

    def gather_segments(self, ctx, out, local, segments, stream=None):
        """out [Hq, n, d] bf16 on every rank <- every segment from its owner's local buffer."""
        hq, n, d = out.shape
        check(lib().shplb_gather_segments(ctx._h, self._h, segments, len(segments), hq, n, d,
                                          C.c_void_p(local.data_ptr() if local is not None else 0),
                                          C.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def gather_heads(self, ctx, out, local, device_of_head, stream=None):
        """Whole-head plan form (shplb_gather_heads)."""
        hq, n, d = out.shape
        dev = np.ascontiguousarray(device_of_head, np.int32)
        if dev.size != hq:
            from ._native import InvalidArgument
            raise InvalidArgument(f"assignment covers {dev.size} heads but {hq} budgets were given")
        check(lib().shplb_gather_heads(ctx._h, self._h, hq, n, d, _ptr(dev),
                                       C.c_void_p(local.data_ptr() if local is not None else 0),
                                       C.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def barrier(self, stream=None):
        check(lib().shplb_comm_barrier(self._h, _stream_ptr(stream)))

    def close(self):
        if self._h:
            check(lib().shplb_nccl_comm_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
