"""One layer through the C ABI for compute-sanitizer runs (dev tool): n = 16384
so kernel 2 walks several 64-block chunks of shared memory."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402

n = int(os.environ.get("SAN_N", "16384"))
q, k, v = make_layer(LayerSpec(num_q_heads=4, num_kv_heads=2, seq_len=n, seed=5), "cuda")
ctx = P.Context(0)
out = ctx.sparse_attention_layer(q, k, v, np.array([128, 2048, 8192, n], np.int64))
dense = ctx.dense_attention_layer(q, k, v)
torch.cuda.synchronize()
print("ok", float(out.float().abs().mean()), float(dense.float().abs().mean()))
