"""Kernel 1 / kernel 2 stage times of layer calls of different widths on the C3
128K layer (dev tool, GPU box): the whole layer (8 kv groups), one KV-head
chunk as the host-buffer entry issues it (1 group, 4 q heads) and a D = 8
rank's shard (greedy plan, layer 0). Run once per SHPLB_K2_SPLIT setting (0 =
fused score + select, 1 = key chunks split over grid.z + a select kernel; unset
= the library's rule) — the variable is read once per process:
    SHPLB_K2_SPLIT=0 python tools/k2_probe.py; SHPLB_K2_SPLIT=1 python tools/k2_probe.py
Prints one JSON line: per case k1 / k2 ms (median of 5 timed calls) and a hash
of the selection, which must not depend on the setting."""
import hashlib
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200.head_parallel import rank_shard  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402


def main():
    n, hq, hkv = 131072, 32, 8
    g = hq // hkv
    q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=2603), "cuda")
    rng = np.random.default_rng(0)
    b = (rng.integers(1, 512, hq) * 128).astype(np.int64)  # heterogeneous budgets, 128..65408 tokens
    ctx = P.Context(0)
    sh = rank_shard(P.greedy_assign(b, 8), 0, g, b)
    cases = {
        "layer": (q, k, v, b, None),
        "kv_chunk": (q[:g].contiguous(), k[:1].contiguous(), v[:1].contiguous(), b[:g], None),
        "rank_D8": (q[sh.heads].contiguous(), k[sh.kv_heads].contiguous(), v[sh.kv_heads].contiguous(),
                    sh.budgets, sh.kv_map),
    }
    res = {"SHPLB_K2_SPLIT": os.environ.get("SHPLB_K2_SPLIT", "auto")}
    for name, (qq, kk, vv, bb, kvm) in cases.items():
        out = torch.empty_like(qq)
        call = lambda: ctx.sparse_attention_layer(qq, kk, vv, bb, out=out, kv_map=kvm)  # noqa: E731
        call()
        torch.cuda.synchronize()
        ctx.set_timing(True)
        for _ in range(5):
            call()
        torch.cuda.synchronize()
        t = ctx.read_timing()
        ctx.set_timing(False)
        idx, cnt = ctx.last_selection(qq.shape[0], n)
        h = hashlib.sha256(idx.cpu().numpy().tobytes() + cnt.cpu().numpy().tobytes()).hexdigest()[:16]
        med = np.median(t, axis=0)
        res[name] = {"heads": int(qq.shape[0]), "k1_ms": round(float(med[0]), 4), "k2_ms": round(float(med[1]), 4),
                     "k3_ms": round(float(med[2]), 3), "selection_sha": h}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
