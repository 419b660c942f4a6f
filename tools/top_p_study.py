"""The paper's top-p argument measured on C3 layer 0 (dev
tool, GPU box): per-head top-p budgets from the calibration curves vs the
max-min table of the same total, their output error and the naive / greedy /
split barrier at D = 2, 4, 8. Writes JSON lines to stdout.
    python tools/top_p_study.py > profiles/r01/top_p_C3.jsonl"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200 import experiments as X  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402


def main():
    n, hq, hkv = int(os.environ.get("TOPP_N", "131072")), 32, 8
    ctx = P.Context(0)
    q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=2603), "cuda")
    curves = ctx.profile_curves(q[:, n - 16:, :].contiguous(), k, P.default_budget_grid(n, 128))
    dense = ctx.dense_attention_layer(q, k, v)
    import torch
    out = torch.empty_like(q)
    for p in (0.6, 0.7, 0.8):
        tp = np.maximum(P.top_p_budgets(curves, p), 128)
        total = int(tp.sum())
        mm = P.maxmin_allocate(curves, total, quantum=128, floor=128).budgets.astype(np.int64)
        for name, b in (("top_p", tp), ("maxmin_same_total", mm)):
            ctx.sparse_attention_layer(q, k, v, b, out=out)
            torch.cuda.synchronize()
            err = float(np.mean([X.output_error(out[h], dense[h]) for h in range(hq)]))
            row = {"p": p, "budgets": name, "total": total, "min_budget": int(b.min()), "max_budget": int(b.max()),
                   "mean_output_error": err}
            for D in (2, 4, 8):
                _, rn = X.measured_barrier(ctx, q, k, v, b, P.naive_assign(b, D), D, 2)
                _, rg = X.measured_barrier(ctx, q, k, v, b, P.greedy_assign(b, D), D, 2)
                _, rs, _ = X.measured_split_barrier(ctx, q, k, v, b, D, 2)
                row[f"D{D}"] = {"naive_ms": round(rn.barrier_latency, 3), "naive_bubble": round(rn.bubble_fraction, 4),
                                "greedy_ms": round(rg.barrier_latency, 3), "greedy_bubble": round(rg.bubble_fraction, 4),
                                "split_ms": round(rs.barrier_latency, 3), "split_bubble": round(rs.bubble_fraction, 4)}
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
