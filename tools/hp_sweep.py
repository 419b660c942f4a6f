"""Head-parallel sweep on one GPU: per-rank device latency of every rank's
shard under the even-HP (naive contiguous), S-HPLB (greedy LPT) and sub-head
(split) plans, for D in {1, 2, 4, 8}; plus the dense-attention and uniform-
budget comparators.

Each rank's shard (its q heads, the kv heads they read, its query-block
ranges) is run and CUDA-event timed in turn on the one GPU, so the numbers are
the per-rank compute a D-GPU run performs (the all-gather is not included;
bench.py measures it when run with N > 1). Barrier latency = max over ranks,
bubble = 1 - mean/max (simulator.cpp:28-47), speedup = T_naive / T_plan.

usage: python tools/hp_sweep.py C3 [--steps 5] [--dense] [--uniform]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200.calibrate import maxmin_budgets, uniform_budgets  # noqa: E402
from paper_2603_10353_b200.head_parallel import rank_segments, rank_shard  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402

CONFIGS = {  # BASELINE.json configs
    "C1": dict(q_heads=32, kv_heads=8, n=8192, devices=[1, 2]),
    "C2": dict(q_heads=32, kv_heads=8, n=32768, devices=[1]),
    "C3": dict(q_heads=32, kv_heads=8, n=131072, devices=[1, 2, 4, 8]),
    "C4": dict(q_heads=28, kv_heads=4, n=65536, devices=[1, 2, 4, 8]),
    "C5": dict(q_heads=64, kv_heads=8, n=131072, devices=[1, 8]),
}


def time_call(ctx, fn, steps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def shard_time(ctx, q, k, v, shard, steps, ranges=None):
    if not shard.heads:
        return 0.0
    ql = q[shard.heads].contiguous()
    kl, vl = k[shard.kv_heads].contiguous(), v[shard.kv_heads].contiguous()
    out = torch.empty_like(ql)
    ms = time_call(ctx, lambda: ctx.sparse_attention_layer(
        ql, kl, vl, shard.budgets, out=out, kv_map=shard.kv_map, q_block_range=ranges), steps)
    del ql, kl, vl, out
    return ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CONFIGS))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--dense", action="store_true", help="also time full (dense causal) attention")
    ap.add_argument("--uniform", action="store_true", help="also time uniform budgets")
    ap.add_argument("--fraction", type=float, default=0.25)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    hq, hkv, n = cfg["q_heads"], cfg["kv_heads"], cfg["n"]
    group = hq // hkv
    q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=2603), "cuda")
    budgets, info, _ = maxmin_budgets(q, k, a.fraction)
    ctx = P.Context(0)
    base = {"config": a.config, "q_heads": hq, "kv_heads": hkv, "seq_len": n,
            "budget_fraction": a.fraction, "budgets": budgets.tolist(), **info}
    print(json.dumps({"kind": "budget_table", **base}), flush=True)
    for D in cfg["devices"]:
        rows = {}
        wc = P.tile_costs(budgets, n, query_tile_weight=P.api.QUERY_TILE_WEIGHT)
        plans = {"naive": P.naive_assign(budgets, D), "greedy": P.greedy_assign(budgets, D),
                 "greedy_refined": P.refine_assign(wc, D, P.greedy_assign(wc, D))}
        for name, plan in plans.items():
            per = [shard_time(ctx, q, k, v, rank_shard(plan, r, group, budgets), a.steps)
                   for r in range(D)]
            rows[name] = (per, float(P.imbalance(budgets, plan, D).imbalance))
        sp = P.split_assign(budgets, D, n, query_tile_weight=P.api.QUERY_TILE_WEIGHT)
        per = []
        for r in range(D):
            seg = rank_segments(sp, r, group, budgets)
            per.append(shard_time(ctx, q, k, v, seg, a.steps, ranges=seg.q_block_range))
        rows["split"] = (per, float(sp.loads.max() * D / sp.loads.sum()))
        t_naive = max(rows["naive"][0])
        for name, (per, imb) in rows.items():
            res = P.barrier(per)
            print(json.dumps({"kind": "hp", "config": a.config, "devices": D, "plan": name,
                              "per_rank_ms": [round(x, 3) for x in per],
                              "barrier_ms": round(res.barrier_latency, 3),
                              "bubble": round(res.bubble_fraction, 4),
                              "speedup_vs_naive": round(t_naive / res.barrier_latency, 4),
                              "plan_cost_imbalance": round(imb, 4)}), flush=True)
    if a.uniform:
        ub = uniform_budgets(hq, n, a.fraction)
        full = rank_shard(np.zeros(hq, np.int32), 0, group, ub)
        ms_u = shard_time(ctx, q, k, v, full, a.steps)
        print(json.dumps({"kind": "uniform_budgets", "config": a.config, "ms": round(ms_u, 3)}),
              flush=True)
    if a.dense:
        dense = rank_shard(np.zeros(hq, np.int32), 0, group, np.full(hq, n, np.int64))
        ms_d = shard_time(ctx, q, k, v, dense, max(2, a.steps // 2))
        tiles, flops = ctx.last_selection_work()
        print(json.dumps({"kind": "dense", "config": a.config, "ms": round(ms_d, 3),
                          "tflops": round(flops / ms_d / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
