"""Skyline and sweep drivers on MEASURED B200 latencies.

The reference evaluates placements with an affine cost model t_d = alpha +
beta * L_d over integer budget loads (simulator.cpp:28-47):

* ``sweep`` (simulator.cpp:111-149) — per parallelism degree and context
  length, naive vs greedy barrier latency, bubble, imbalance and speedup;
* ``run_skyline`` (commands.cpp:411-489) — per total budget and allocator
  (uniform, max-min), mean output error against dense attention and the
  greedy barrier latency.

Here the same experiments run the sm_100a hot path: every rank's shard of a
plan is executed and CUDA-event timed on the GPU (one GPU runs the ranks in
turn, so the numbers are the per-rank compute a D-GPU run performs; bench.py
times the real multi-process run and the all-gather), the barrier is the max
over ranks, the bubble 1 - mean/max (simulator.cpp:40-44), and output error
is the reference's output_error (attention.cpp:186-202: ||sparse - dense||_F
/ ||dense||_F per head, averaged) against the dense comparator
(shplb_dense_attention_layer). CSV writers keep the reference's columns
(write_sweep_csv / write_skyline_csv) with latencies in milliseconds.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import api
from ._native import InvalidArgument
from .head_parallel import rank_segments, rank_shard


def format_double(v: float) -> str:
    """std::to_chars shortest round-trip (simulator.cpp:22-26)."""
    if v == int(v) and abs(v) < 1e16:
        return str(int(v))
    return repr(float(v))


def _time(fn, steps: int, repeats: int = 3) -> float:
    """Median over `repeats` of the mean device time of `steps` back-to-back
    calls (CUDA events), after 2 warm-up calls. The median keeps one
    transient clock dip from being charged to one rank of a plan."""
    import torch
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(repeats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / steps)
    return float(np.median(times))


def _shard_call(ctx, q, k, v, shard, block_q: int = api.BLOCK_Q, kind=0):
    """A closure running one rank's shard (its q heads, the kv heads they read,
    optional query-block ranges) on its own copies of the inputs; None if empty."""
    import torch
    if not shard.heads:
        return None
    ql = q[shard.heads].contiguous()
    kl, vl = k[shard.kv_heads].contiguous(), v[shard.kv_heads].contiguous()
    out = torch.empty_like(ql)
    ranges = getattr(shard, "q_block_range", None)
    return lambda: ctx.sparse_attention_layer(ql, kl, vl, shard.budgets, out=out, kv_map=shard.kv_map,
                                              q_block_range=ranges, block_q=block_q, kind=kind)


def shard_latency_ms(ctx, q, k, v, shard, steps: int = 3, block_q: int = api.BLOCK_Q, kind=0) -> float:
    """Device time of one rank's shard."""
    fn = _shard_call(ctx, q, k, v, shard, block_q, kind)
    return 0.0 if fn is None else _time(fn, steps)


def shards_latency_ms(ctx, q, k, v, shards, steps: int = 3, rounds: int = 3, block_q: int = api.BLOCK_Q,
                      kind=0) -> list:
    """Device time of every rank's shard, timed in turn on this GPU: `rounds`
    passes over the ranks (each pass times every rank once), median per rank.
    Interleaving the ranks spreads the power-capped clock's drift over all of
    them instead of charging a slow stretch to whichever rank ran then."""
    fns = [_shard_call(ctx, q, k, v, sh, block_q, kind) for sh in shards]
    times = [[] for _ in fns]
    for _ in range(rounds):
        for r, fn in enumerate(fns):
            if fn is not None:
                times[r].append(_time(fn, steps, repeats=1))
    return [float(np.median(t)) if t else 0.0 for t in times]


def measured_barrier(ctx, q, k, v, budgets, device_of_head, devices: int, steps: int = 3, kind=0):
    """(per-rank ms, SimulationResult-like barrier/bubble) of a whole-head plan."""
    group = q.shape[0] // k.shape[0]
    per = shards_latency_ms(ctx, q, k, v, [rank_shard(device_of_head, r, group, budgets) for r in range(devices)],
                            steps, kind=kind)
    return per, api.barrier(per)


def measured_split_barrier(ctx, q, k, v, budgets, devices: int, steps: int = 3, kind=0):
    group = q.shape[0] // k.shape[0]
    sp = api.split_assign(budgets, devices, q.shape[1], query_tile_weight=api.QUERY_TILE_WEIGHT)
    per = shards_latency_ms(ctx, q, k, v, [rank_segments(sp, r, group, budgets) for r in range(devices)],
                            steps, kind=kind)
    return per, api.barrier(per), sp


@dataclass
class SweepRow:
    """simulator.hpp:43-52 (barrier_latency in measured ms)."""
    degree: int
    context_length: int
    allocator: str
    assigner: str
    barrier_latency: float
    bubble_fraction: float
    imbalance: float
    speedup_vs_naive: float
    per_rank_ms: list


def measured_sweep(ctx, layers: dict, degrees, allocator: str = "maxmin", steps: int = 3,
                   include_split: bool = True) -> list:
    """sweep() (simulator.cpp:111-149) on measured latency. layers maps
    context_length -> (q, k, v, budgets) (CUDA tensors, int64 budgets)."""
    for d in degrees:
        if d < 1:
            raise InvalidArgument("parallelism degree must be >= 1")
    rows = []
    for degree in degrees:
        for length, (q, k, v, budgets) in layers.items():
            naive = api.naive_assign(budgets, degree)
            greedy = api.greedy_assign(budgets, degree)
            per_n, res_n = measured_barrier(ctx, q, k, v, budgets, naive, degree, steps)
            per_g, res_g = measured_barrier(ctx, q, k, v, budgets, greedy, degree, steps)
            imb_n = api.imbalance(budgets, naive, degree).imbalance
            imb_g = api.imbalance(budgets, greedy, degree).imbalance
            rows.append(SweepRow(degree, length, allocator, "naive", res_n.barrier_latency,
                                 res_n.bubble_fraction, imb_n, 1.0, per_n))
            rows.append(SweepRow(degree, length, allocator, "greedy", res_g.barrier_latency,
                                 res_g.bubble_fraction, imb_g,
                                 1.0 if res_g.barrier_latency == 0 else res_n.barrier_latency / res_g.barrier_latency,
                                 per_g))
            # greedy_assign weighted by kernel 3's causal tile cost (api.tile_costs)
            gt = api.greedy_assign(api.tile_costs(budgets, q.shape[1]), degree)
            per_t, res_t = measured_barrier(ctx, q, k, v, budgets, gt, degree, steps)
            rows.append(SweepRow(degree, length, allocator, "greedy_tiles", res_t.barrier_latency,
                                 res_t.bubble_fraction, api.imbalance(budgets, gt, degree).imbalance,
                                 1.0 if res_t.barrier_latency == 0 else res_n.barrier_latency / res_t.barrier_latency,
                                 per_t))
            # whole-head local search (api.refine_assign) on tile cost + the per-query-tile
            # fixed cost, from greedy on that cost
            wc = api.tile_costs(budgets, q.shape[1], query_tile_weight=api.QUERY_TILE_WEIGHT)
            gr = api.refine_assign(wc, degree, api.greedy_assign(wc, degree))
            per_r, res_r = measured_barrier(ctx, q, k, v, budgets, gr, degree, steps)
            rows.append(SweepRow(degree, length, allocator, "greedy_refined", res_r.barrier_latency,
                                 res_r.bubble_fraction, api.imbalance(budgets, gr, degree).imbalance,
                                 1.0 if res_r.barrier_latency == 0 else res_n.barrier_latency / res_r.barrier_latency,
                                 per_r))
            if include_split:
                per_s, res_s, sp = measured_split_barrier(ctx, q, k, v, budgets, degree, steps)
                rows.append(SweepRow(degree, length, allocator, "split", res_s.barrier_latency,
                                     res_s.bubble_fraction, float(sp.loads.max() * degree / sp.loads.sum()),
                                     res_n.barrier_latency / res_s.barrier_latency, per_s))
    return rows


def write_sweep_csv(path_or_file, rows) -> None:
    """write_sweep_csv (simulator.cpp:151-160); barrier_latency in ms."""
    lines = ["degree,context_length,allocator,assigner,barrier_latency,bubble_fraction,imbalance,speedup_vs_naive"]
    for r in rows:
        lines.append(",".join([str(r.degree), str(r.context_length), r.allocator, r.assigner,
                               format_double(r.barrier_latency), format_double(r.bubble_fraction),
                               format_double(r.imbalance), format_double(r.speedup_vs_naive)]))
    _write(path_or_file, lines)


@dataclass
class SkylinePoint:
    """commands.hpp:70-76 (latencies in measured ms)."""
    total_budget: int
    allocator: str
    mean_output_error: float
    barrier_latency: float        # greedy placement
    naive_barrier_latency: float  # not serialized (as in the reference)
    max_output_error: float = 0.0  # worst head (not serialized): what max-min optimises


def output_error(sparse, dense) -> float:
    """attention.cpp:186-202 on one head: ||s - d||_F / ||d||_F, 0 if equal, inf if d = 0."""
    s = sparse.double()
    d = dense.double()
    diff = float(((s - d) ** 2).sum())
    if diff == 0.0:
        return 0.0
    den = float((d ** 2).sum()) ** 0.5
    return float("inf") if den == 0.0 else diff ** 0.5 / den


def measured_skyline(ctx, q, k, v, curves, devices: int, totals=None, quantum: int = 128, floor: int = 128,
                     steps: int = 3, causal: bool = True, policy=0) -> list:
    """run_skyline (commands.cpp:411-489) on measured latency: for each total
    budget (default 0.25/0.5/0.75/1.0 of Hq*n) and allocator (uniform,
    max-min), the mean per-head output error against dense attention and the
    greedy / naive barrier latency of the budgets at `devices` ranks, under
    selection `policy` (the SelectionKind of commands.cpp:464-470)."""
    import torch
    hq, n, _ = q.shape
    if totals is None:
        totals = [int(round(f * hq * n)) for f in (0.25, 0.5, 0.75, 1.0)]
    for t in totals:
        if t < hq * floor or t > hq * n:
            raise InvalidArgument(f"skyline budget {t} infeasible; feasible range is "
                                      f"[{hq * floor}, {hq * n}]")
    dense = ctx.dense_attention_layer(q, k, v, causal=causal)
    out = torch.empty_like(q)
    points = []
    for total in totals:
        for kind in ("uniform", "maxmin"):
            if kind == "uniform":
                budgets = api.uniform_allocate(hq, total, floor, n).budgets.astype(np.int64)
            else:
                budgets = api.maxmin_allocate(curves, total, quantum=quantum, floor=floor).budgets.astype(np.int64)
            ctx.sparse_attention_layer(q, k, v, budgets, out=out, causal=causal, kind=policy)
            torch.cuda.synchronize()
            errs = [output_error(out[h], dense[h]) for h in range(hq)]
            err = float(np.mean(errs))
            _, rg = measured_barrier(ctx, q, k, v, budgets, api.greedy_assign(budgets, devices), devices, steps,
                                     kind=policy)
            _, rn = measured_barrier(ctx, q, k, v, budgets, api.naive_assign(budgets, devices), devices, steps,
                                     kind=policy)
            points.append(SkylinePoint(int(total), kind, err, rg.barrier_latency, rn.barrier_latency,
                                       float(np.max(errs))))
    return points


@dataclass
class TopPPoint:
    """One offline top-p operating point: every head gets the
    budget its own curve needs to reach recovery p."""
    p: float
    total_budget: int
    mean_output_error: float
    naive_barrier_latency: float
    naive_bubble: float
    greedy_barrier_latency: float
    greedy_bubble: float


def measured_top_p(ctx, q, k, v, curves, devices: int, ps=(0.8, 0.9, 0.95), steps: int = 3,
                   causal: bool = True, policy=0) -> list:
    """The paper's top-p comparison on measured latency: per-head budgets from
    budget_for_recovery(curve, p) (profiler.cpp:198-209), their output error
    against dense attention, and the barrier latency / bubble of those budgets
    placed by even head parallelism (naive) and by the greedy balancer — the
    cross-GPU imbalance a per-head top-p budget creates."""
    import torch
    hq = q.shape[0]
    dense = ctx.dense_attention_layer(q, k, v, causal=causal)
    out = torch.empty_like(q)
    points = []
    for p in ps:
        budgets = api.top_p_budgets(curves, p)
        budgets = np.maximum(budgets, 1)
        ctx.sparse_attention_layer(q, k, v, budgets, out=out, causal=causal, kind=policy)
        torch.cuda.synchronize()
        err = float(np.mean([output_error(out[h], dense[h]) for h in range(hq)]))
        _, rn = measured_barrier(ctx, q, k, v, budgets, api.naive_assign(budgets, devices), devices, steps,
                                 kind=policy)
        _, rg = measured_barrier(ctx, q, k, v, budgets, api.greedy_assign(budgets, devices), devices, steps,
                                 kind=policy)
        points.append(TopPPoint(float(p), int(budgets.sum()), err, rn.barrier_latency, rn.bubble_fraction,
                                rg.barrier_latency, rg.bubble_fraction))
    return points


def write_skyline_csv(path_or_file, rows) -> None:
    """write_skyline_csv (commands.cpp:491-499); barrier_latency in ms."""
    lines = ["total_budget,allocator,mean_output_error,barrier_latency"]
    for r in rows:
        lines.append(",".join([str(r.total_budget), r.allocator, format_double(r.mean_output_error),
                               format_double(r.barrier_latency)]))
    _write(path_or_file, lines)


def _write(path_or_file, lines) -> None:
    text = "\n".join(lines) + "\n"
    if hasattr(path_or_file, "write"):
        path_or_file.write(text)
    else:
        with open(path_or_file, "w") as f:
            f.write(text)
