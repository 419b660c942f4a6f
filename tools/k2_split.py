"""Kernel 2's score and select parts timed separately on the C3 128K layer (dev
tool, GPU box): block_scores (pool + score, writing the score matrix),
select_blocks on it, and the fused layer's stage times."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402
from paper_2603_10353_b200 import experiments as X  # noqa: E402
n=131072
q,k,v = make_layer(LayerSpec(seq_len=n, seed=2603), "cuda")
ctx=P.Context(0)
b = np.full(32, n//4, np.int64)
sc = ctx.block_scores(q, k, block_q=256)
t_scores = X._time(lambda: ctx.block_scores(q, k, block_q=256, out=sc), 5)
t_sel = X._time(lambda: ctx.select_blocks(sc, (b+127)//128, n, block_q=256), 5)
ctx.set_timing(True)
for _ in range(5): ctx.sparse_attention_layer(q,k,v,b)
torch.cuda.synchronize()
t = ctx.read_timing().mean(0)
print({"block_scores_ms(k1+k2 score, writes 64MB)": t_scores, "select_from_scores_ms": t_sel, "layer_stages": t.tolist()})
