"""Where the e2e (host-buffer) time goes at C3: device-only layers (one launch
per layer vs one per KV-head chunk, as the host entry issues them) against the
async host-buffer entry, for L consecutive layers. Run on the B200:
    python tools/e2e_probe.py --layers 4
(set SHPLB_HOST_CHUNKS to change the host entry's pipeline depth)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--seq-len", type=int, default=131072)
    a = ap.parse_args()
    n, hq, hkv = a.seq_len, 32, 8
    ctx = P.Context(0)
    layers = []
    for l in range(a.layers):
        q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, layer=l), "cuda")
        grid = P.default_budget_grid(n, 128)
        curves = ctx.profile_curves(q[:, n - 16:, :].contiguous(), k, grid)
        b = P.maxmin_allocate(curves, int(0.25 * hq * n), quantum=128, floor=128).budgets.astype(np.int64)
        layers.append((q, k, v, b))
    out = torch.empty_like(layers[0][0])
    L = len(layers)

    def dev():
        for q, k, v, b in layers:
            ctx.sparse_attention_layer(q, k, v, b, out=out)

    def dev_chunked():
        g = hq // hkv
        for q, k, v, b in layers:
            for c in range(hkv):
                ctx.sparse_attention_layer(q[c * g:(c + 1) * g], k[c:c + 1], v[c:c + 1], b[c * g:(c + 1) * g],
                                           out=out[c * g:(c + 1) * g])

    ctx2 = P.Context(0)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]

    def dev_chunked_2ctx():  # chunk c on context/stream c & 1: chunk tails and K1/K2 overlap
        g = hq // hkv
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cur)
        for s_ in streams:
            s_.wait_event(ev)
        for q, k, v, b in layers:
            for c in range(hkv):
                s_ = streams[c & 1]
                (ctx, ctx2)[c & 1].sparse_attention_layer(q[c * g:(c + 1) * g], k[c:c + 1], v[c:c + 1],
                                                          b[c * g:(c + 1) * g], out=out[c * g:(c + 1) * g],
                                                          stream=s_)
        for s_ in streams:
            e = torch.cuda.Event()
            e.record(s_)
            cur.wait_event(e)

    host = [tuple(t.cpu().pin_memory() for t in (q, k, v)) for q, k, v, _ in layers]
    outs = [torch.empty(layers[0][0].shape, dtype=torch.bfloat16, pin_memory=True) for _ in layers]
    st = torch.cuda.current_stream()

    def e2e():
        for (hq_, hk_, hv_), o, (_, _, _, b) in zip(host, outs, layers):
            ctx.sparse_attention_layer_host(hq_, hk_, hv_, b, out=o, stream=st, asynchronous=True)
        st.synchronize()

    def h2d_only():
        for (hq_, hk_, hv_), (q, k, v, _) in zip(host, layers):
            q.copy_(hq_, non_blocking=True); k.copy_(hk_, non_blocking=True); v.copy_(hv_, non_blocking=True)

    def d2h_only():
        for o in outs:
            o.copy_(out, non_blocking=True)

    stage = {}
    for name, fn in (("full", dev), ("chunked", dev_chunked)):
        fn()
        torch.cuda.synchronize()
        ctx.set_timing(True)
        fn()
        torch.cuda.synchronize()
        t = ctx.read_timing()
        ctx.set_timing(False)
        stage[name] = [round(float(x) / L, 3) for x in t.sum(0)]  # k1, k2, k3 ms per layer
    res = {"layers": L, "stages_ms_per_layer": stage, "host_chunks": os.environ.get("SHPLB_HOST_CHUNKS", "8"),
           "dev_ms_per_layer": timed(dev) / L, "dev_chunked_ms_per_layer": timed(dev_chunked) / L,
           "dev_chunked_2streams_ms_per_layer": timed(dev_chunked_2ctx) / L,
           "e2e_ms_per_layer": timed(e2e) / L,
           "h2d_GBps": 3 * 0 + sum(t.numel() * 2 for hs in host for t in hs) / timed(h2d_only) / 1e6,
           "d2h_GBps": sum(o.numel() * 2 for o in outs) / timed(d2h_only) / 1e6}
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in res.items()}))


if __name__ == "__main__":
    main()
