"""Device timeline of one host-buffer layer call (dev tool): kernels and memcpys
with start/end per stream, from a CUPTI trace (torch.profiler)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402

n = int(os.environ.get("TRACE_N", "131072"))
q, k, v = make_layer(LayerSpec(seq_len=n), "cuda")
budgets = np.full(32, n // 4, np.int64)
qh, kh, vh = (t.cpu().pin_memory() for t in (q, k, v))
out = torch.empty_like(qh).pin_memory()
ctx = P.Context(0)
s = torch.cuda.Stream()
for _ in range(2):
    ctx.sparse_attention_layer_host(qh, kh, vh, budgets, out=out, stream=s)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ctx.sparse_attention_layer_host(qh, kh, vh, budgets, out=out, stream=s)
    torch.cuda.synchronize()
path = "/tmp/trace_e2e.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy")]
t0 = min(e["ts"] for e in ev)
for e in sorted(ev, key=lambda e: e["ts"]):
    print(f"{(e['ts'] - t0) / 1e3:9.3f} ms  +{e['dur'] / 1e3:8.3f}  stream {e['args'].get('stream')}  {e['name'][:60]}")
