"""Output error and latency of block_q = 256 vs 128 on C3 layer 0 (dev tool,
GPU box): same max-min budgets, error = mean over heads of
||sparse - dense||_F / ||dense||_F (output_error, attention.cpp:186-202)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200 import experiments as X  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402

n, hq = 131072, 32
ctx = P.Context(0)
q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=8, seq_len=n, seed=2603), "cuda")
curves = ctx.profile_curves(q[:, n - 16:, :].contiguous(), k, P.default_budget_grid(n, 128))
dense = ctx.dense_attention_layer(q, k, v)
for frac in (0.125, 0.25):
    b = P.maxmin_allocate(curves, int(frac * hq * n), quantum=128, floor=128).budgets
    for bq in (256, 128):
        out = ctx.sparse_attention_layer(q, k, v, b, block_q=bq)
        torch.cuda.synchronize()
        err = float(np.mean([X.output_error(out[h], dense[h]) for h in range(hq)]))
        ms = X._time(lambda: ctx.sparse_attention_layer(q, k, v, b, block_q=bq, out=out), 3)
        print(json.dumps({"budget_fraction": frac, "block_q": bq, "mean_output_error": round(err, 5),
                          "layer_ms": round(ms, 3)}), flush=True)
