"""Time the GPU recovery-curve profiler against the host one on the C3 layer
(dev tool): python tools/profile_timing.py [rows ...]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, bf16_bits, make_layer  # noqa: E402

n = int(os.environ.get("TUNE_N", "131072"))
q, k, _ = make_layer(LayerSpec(seq_len=n, seed=2603), "cuda")
grid = P.default_budget_grid(n, 128)
ctx = P.Context(0)
for rows in [int(r) for r in sys.argv[1:]] or [16, 128]:
    qr = q[:, n - rows:, :].contiguous()
    ctx.profile_curves(qr, k, grid)  # warm-up (workspace, CUB temp)
    torch.cuda.synchronize()
    t0 = time.time()
    gpu = ctx.profile_curves(qr, k, grid)
    tg = time.time() - t0
    rec = {"rows": rows, "gpu_s": round(tg, 4)}
    if rows <= 16:
        t0 = time.time()
        host = P.profile_curves(bf16_bits(qr), bf16_bits(k), grid)
        rec["host_s"] = round(time.time() - t0, 3)
        rec["max_abs_diff"] = float(max(np.abs(g.recovery - h.recovery).max() for g, h in zip(gpu, host)))
    print(json.dumps(rec), flush=True)
