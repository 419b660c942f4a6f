"""Kernel 3 over a whole C3 layer in one launch vs one launch per kv group
(dev tool, GPU box). The selection is computed once (kernels 1-2, untimed);
then, interleaved over rounds so clock drift under the power cap spreads
evenly, the persistent kernel 3 runs (a) on the whole layer, (b) once per kv
group (4 q heads and their kv head each) on the same selection. Prints the
median ms per layer of each and the board energy per layer (NVML).
    python tools/k3_group_probe.py [rounds]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200.calibrate import layer_budgets  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402


def main():
    rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    n, hq, hkv = 131072, 32, 8
    g = hq // hkv
    q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=2603), "cuda")
    ctx = P.Context(0)
    budgets, _, _ = layer_budgets(q, k, 0.25, ctx=ctx)
    kb = (budgets + 127) // 128
    sc = ctx.block_scores(q, k)
    idx, cnt = ctx.select_blocks(sc, kb, n, kmax=int(kb.max()))
    del sc
    out = torch.empty_like(q)
    parts = [(q[i * g:(i + 1) * g], k[i:i + 1], v[i:i + 1], idx[i * g:(i + 1) * g].contiguous(),
              cnt[i * g:(i + 1) * g].contiguous(), out[i * g:(i + 1) * g]) for i in range(hkv)]

    def full():
        ctx.block_sparse_attention(q, k, v, idx, cnt, out=out)

    def grouped():
        for qq, kk, vv, ii, cc, oo in parts:
            ctx.block_sparse_attention(qq, kk, vv, ii, cc, out=oo)

    try:
        import pynvml
        pynvml.nvmlInit()
        nvh = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    except Exception:  # noqa: BLE001
        nvh = None
    res = {"full": [], "grouped": []}
    joules = {"full": [], "grouped": []}
    for fn in (full, grouped):
        fn()
    torch.cuda.synchronize()
    ref = out.clone()
    grouped()
    torch.cuda.synchronize()
    same = bool(torch.equal(out, ref))
    reps = 4
    for _ in range(rounds):
        for name, fn in (("full", full), ("grouped", grouped)):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            mj0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(nvh) if nvh else 0
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            mj1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(nvh) if nvh else 0
            res[name].append(e0.elapsed_time(e1) / reps)
            joules[name].append((mj1 - mj0) / 1e3 / reps)
    print(json.dumps({"bit_identical": same,
                      **{f"{k_}_ms": round(float(np.median(v_)), 3) for k_, v_ in res.items()},
                      **{f"{k_}_J": round(float(np.median(v_)), 2) for k_, v_ in joules.items()},
                      "rounds": {k_: [round(x, 3) for x in v_] for k_, v_ in res.items()}}))


if __name__ == "__main__":
    main()
