"""Per-rank shard latency of C3 layer 0 under each head plan at D = 4, 8 for
the current SHPLB_TILE_ORDER (dev tool, GPU box):
    for m in 0 1 2; do SHPLB_TILE_ORDER=$m python tools/shard_order.py; done"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200 import experiments as X  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402


def main():
    n, hq, hkv = 131072, 32, 8
    ctx = P.Context(0)
    q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=2603), "cuda")
    curves = ctx.profile_curves(q[:, n - 16:, :].contiguous(), k, P.default_budget_grid(n, 128))
    b = P.maxmin_allocate(curves, int(0.25 * hq * n), quantum=128, floor=128).budgets.astype(np.int64)
    full = X._time(lambda: ctx.sparse_attention_layer(q, k, v, b), 3)
    rows = X.measured_sweep(ctx, {n: (q, k, v, b)}, [4, 8], steps=3)
    out = {"order": os.environ.get("SHPLB_TILE_ORDER", "1"), "full_layer_ms": round(full, 3)}
    rows = X.measured_sweep(ctx, {n: (q, k, v, b)}, [4, 8], steps=3)
    out = {"order": os.environ.get("SHPLB_TILE_ORDER", "1"), "full_layer_ms": round(full, 3)}
    for D in (4, 8):
        for ov in (0, 3, 6, 9):
            per, res, sp = X.measured_split_barrier(ctx, q, k, v, b, D, 3, qblock_overhead=ov)
            out[f"D{D}_split_ov{ov}"] = {"barrier": round(res.barrier_latency, 3),
                                         "bubble": round(res.bubble_fraction, 4),
                                         "sum_ranks": round(float(np.sum(per)), 3)}
    for r in rows:
        out[f"D{r.degree}_{r.assigner}"] = {"barrier": round(r.barrier_latency, 3),
                                            "bubble": round(r.bubble_fraction, 4),
                                            "sum_ranks": round(float(np.sum(r.per_rank_ms)), 3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
