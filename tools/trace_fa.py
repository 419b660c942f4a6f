"""Run the C3 128K layer with a SHPLB_TRACE build of kernel 3 and keep the
clock64 timeline it prints for one CTA (dev tool).

usage: SHPLB_LIB=<trace build .so> python tools/trace_fa.py > trace.txt
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, bf16_bits, make_layer  # noqa: E402

n = int(os.environ.get("TUNE_N", "131072"))
q, k, v = make_layer(LayerSpec(seq_len=n, seed=2603), "cuda")
bfile = "/tmp/shplb_tune_budgets_%d.npy" % n
if os.path.exists(bfile):
    budgets = np.load(bfile)
else:
    curves = P.profile_curves(bf16_bits(q[:, n - 16:, :]), bf16_bits(k), P.default_budget_grid(n, 128))
    budgets = P.maxmin_allocate(curves, int(0.25 * 32 * n), 128, 128).budgets
    np.save(bfile, budgets)
ctx = P.Context(0)
out = torch.empty_like(q)
for _ in range(3):
    ctx.sparse_attention_layer(q, k, v, budgets, out=out)
torch.cuda.synchronize()
