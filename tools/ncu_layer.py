"""One C3 layer (bench layer 0: seed 2603, its max-min budget table from 128
evenly spaced calibration rows) run through the layer call a few times — the
workload the ncu captures under profiles/ profile (dev tool, GPU box):

  ncu --set full --clock-control none --import-source on -k regex:fa_sparse_kernel -s 2 -c 1 \
      -o gpurun_out/ncu_k3 python tools/ncu_layer.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200 import calibrate  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402

n = int(os.environ.get("TUNE_N", "131072"))
calls = int(os.environ.get("CALLS", "3"))
hq, hkv = int(os.environ.get("HQ", "32")), int(os.environ.get("HKV", "8"))  # C4: HQ=28 HKV=4 TUNE_N=65536
q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=2603), "cuda")
ctx = P.Context(0)
budgets, info, _ = calibrate.layer_budgets(q, k, 0.25, kind="token", rows=128, ctx=ctx)
out = torch.empty_like(q)
for _ in range(calls):
    ctx.sparse_attention_layer(q, k, v, budgets, out=out)
torch.cuda.synchronize()
tiles, flops = ctx.last_selection_work()
print({"digest": info["digest"], "tiles": tiles, "flops": flops})
