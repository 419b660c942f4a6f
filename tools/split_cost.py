"""Per-rank latency of head-parallel plans vs their cost model (dev tool, GPU).

usage: python tools/split_cost.py [out.json]
C3 layer 0 (the bench's inputs and max-min table). For D = 4 and 8, each rank's shard of the
sub-head plan (shplb_plan_split) and of greedy_assign is timed in turn on this GPU, several
rounds interleaved so clock drift under the power cap spreads over all ranks, next to the
rank's tile count (computed (query half, key block) tiles), query-tile count and head count.
A least-squares fit  ms = a * tiles + b * query_tiles + c * heads  over all ranks says how
much of a rank's time the plan's cost model (tiles only) leaves out.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200 import experiments as X  # noqa: E402
from paper_2603_10353_b200.calibrate import layer_budgets  # noqa: E402
from paper_2603_10353_b200.head_parallel import rank_segments, rank_shard  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402

n = int(os.environ.get("TUNE_N", "131072"))
rounds = int(os.environ.get("ROUNDS", "3"))
overheads = [int(x) for x in os.environ.get("OVERHEADS", "").split(",") if x]
q, k, v = make_layer(LayerSpec(seq_len=n, seed=2603), "cuda")
ctx = P.Context(0)
budgets, _, _ = layer_budgets(q, k, 0.25, ctx=ctx)
hq = q.shape[0]
group = hq // k.shape[0]
nqb = (n + 255) // 256
costs = P.tile_costs(budgets, n)  # per head, whole head


def head_qtile_cost(h, b, e):
    nkb = (n + 127) // 128
    kb = min((int(budgets[h]) + 127) // 128, nkb)
    qb = np.arange(b, e)
    vis = np.minimum(((np.minimum((qb + 1) * 256, n) - 1) // 128) + 1, nkb)
    t = np.minimum(kb, vis) * 2
    return int(t.sum()), int((t > 0).sum())


def plan_rows(kind, D, plan):
    shards, feats = [], []
    for r in range(D):
        if kind.startswith("split"):
            sh = rank_segments(plan, r, group, budgets)
            segs = [(h, int(a), int(b)) for h, (a, b) in zip(sh.heads, sh.q_block_range)]
        else:
            sh = rank_shard(plan, r, group, budgets)
            segs = [(h, 0, nqb) for h in sh.heads]
        tiles = qt = 0
        for h, a, b in segs:
            t, c = head_qtile_cost(h, a, b)
            tiles += t
            qt += c
        shards.append(sh)
        feats.append((tiles, qt, len(sh.heads)))
    return shards, feats


def split_with_overhead(D, c_tile):
    """Python restatement of shplb_plan_split with `c_tile` extra cost units per query tile."""
    nkb = (n + 127) // 128
    unit = []
    for h in range(hq):
        kb = min((int(budgets[h]) + 127) // 128, nkb)
        qb = np.arange(nqb)
        vis = np.minimum(((np.minimum((qb + 1) * 256, n) - 1) // 128) + 1, nkb)
        t = np.minimum(kb, vis) * 2
        unit.append(t + c_tile * (t > 0))
    total = int(sum(u.sum() for u in unit))
    dev, head, b0, b1 = [], [], [], []
    d, prefix = 0, 0
    for h in range(hq):
        begin = 0
        for qb in range(nqb):
            c = int(unit[h][qb])
            while d < D - 1 and (2 * prefix + c) * D >= 2 * total * (d + 1):
                if qb > begin:
                    dev.append(d), head.append(h), b0.append(begin), b1.append(qb)
                begin = qb
                d += 1
            prefix += c
        dev.append(d), head.append(h), b0.append(begin), b1.append(nqb)
    return P.api.SplitPlan(np.array(dev), np.array(head), np.array(b0), np.array(b1), np.zeros(D, np.int64))


plans = []
for D in (4, 8):
    plans.append(("split", D, P.split_assign(budgets, D, n)))
    plans.append(("greedy", D, P.greedy_assign(budgets, D)))
    for c in overheads:
        plans.append((f"split_c{c}", D, split_with_overhead(D, c)))
rows = {}
for kind, D, plan in plans:
    shards, feats = plan_rows(kind, D, plan)
    rows[(kind, D)] = {"feats": feats, "ms": [[] for _ in range(D)], "shards": shards}
for _ in range(rounds):
    for (kind, D), row in rows.items():
        for r, sh in enumerate(row["shards"]):
            row["ms"][r].append(X.shard_latency_ms(ctx, q, k, v, sh, steps=3))
out = {}
A, y = [], []
for (kind, D), row in rows.items():
    ms = [float(np.median(m)) for m in row["ms"]]
    res = P.barrier(ms)
    out[f"{kind}_D{D}"] = {"per_rank_ms": [round(x, 4) for x in ms], "bubble": round(res.bubble_fraction, 4),
                           "barrier_ms": round(res.barrier_latency, 4),
                           "tiles": [f[0] for f in row["feats"]], "query_tiles": [f[1] for f in row["feats"]],
                           "heads": [f[2] for f in row["feats"]]}
    for f, m in zip(row["feats"], ms):
        A.append(f)
        y.append(m)
coef, *_ = np.linalg.lstsq(np.array(A, np.float64), np.array(y), rcond=None)
out["fit_ms"] = {"per_tile_us": coef[0] * 1e3, "per_query_tile_us": coef[1] * 1e3, "per_head_us": coef[2] * 1e3,
                 "query_tile_in_tiles": coef[1] / coef[0]}
print(json.dumps(out, indent=1))
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)
