"""Device timeline of L chained async host-buffer layer calls (dev tool, GPU box):
kernels and memcpys from a CUPTI trace (torch.profiler). Prints where the
compute stream idles between the first and the last kernel (gaps > 20 us, with
what the copy engines were doing), the H2D / D2H busy time, and the span.
    python tools/trace_e2e_chain.py [layers] [--device]
(--device: the same layers from device-resident inputs through the device
entry, as bench.py's `value` runs them.)"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    device = "--device" in sys.argv
    L = int(args[0]) if args else 4
    n = int(os.environ.get("TRACE_N", "131072"))
    rng = np.random.default_rng(0)
    layers = []
    for li in range(L):
        q, k, v = make_layer(LayerSpec(seq_len=n, seed=2603 + li), "cuda")
        b = (rng.integers(1, 512, 32) * 128).astype(np.int64)
        layers.append(((q, k, v) if device else tuple(t.cpu().pin_memory() for t in (q, k, v)), b))
        del q, k, v
    ctx = P.Context(0)
    s = torch.cuda.Stream()
    if device:
        outs = [torch.empty_like(layers[0][0][0]) for _ in range(L)]
    else:
        outs = [torch.empty(layers[0][0][0].shape, dtype=torch.bfloat16).pin_memory() for _ in range(L)]

    def step():
        for ((qh, kh, vh), b), o in zip(layers, outs):
            if device:
                ctx.sparse_attention_layer(qh, kh, vh, b, out=o, stream=s)
            else:
                ctx.sparse_attention_layer_host(qh, kh, vh, b, out=o, stream=s, asynchronous=True)
        s.synchronize()

    step()
    step()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
    ev = []
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        name = e.name
        kind = "h2d" if "HtoD" in name else "d2h" if "DtoH" in name else "memset" if "emset" in name else "kernel"
        ev.append((e.time_range.start, e.time_range.end, kind, name[:40]))
    ev.sort()
    kern = [(a, b, nm) for a, b, k_, nm in ev if k_ == "kernel"]
    t0, t1 = kern[0][0], max(b for _, b, _ in kern)
    gaps, cur, prev = [], kern[0][1], kern[0][2]
    for a, b, nm in kern[1:]:
        if a > cur + 20:
            h2d = sum(max(0, min(bb, a) - max(aa, cur)) for aa, bb, k_, _ in ev if k_ == "h2d")
            d2h = sum(max(0, min(bb, a) - max(aa, cur)) for aa, bb, k_, _ in ev if k_ == "d2h")
            inside = sorted({n_ for aa, bb, k_, n_ in ev if k_ in ("memset", "h2d", "d2h") and cur <= aa < a and
                             bb - aa < 100})  # short copies / memsets that started in the gap
            gaps.append({"at_ms": round((cur - t0) / 1e3, 3), "gap_ms": round((a - cur) / 1e3, 3),
                         "h2d_busy_ms": round(h2d / 1e3, 3), "d2h_busy_ms": round(d2h / 1e3, 3),
                         "after": prev, "before": nm, "short_ops_in_gap": inside})
        if b >= cur:
            cur, prev = b, nm
    first_h2d = min((a for a, _, k_, _ in ev if k_ == "h2d"), default=t0)
    last_d2h = max((b for _, b, k_, _ in ev if k_ == "d2h"), default=t1)
    busy = lambda kind: sum(b - a for a, b, k_, _ in ev if k_ == kind) / 1e3  # noqa: E731
    print(json.dumps({"layers": L, "span_ms": round((last_d2h - first_h2d) / 1e3, 3),
                      "kernel_span_ms": round((t1 - t0) / 1e3, 3),
                      "kernel_busy_ms": round(sum(b - a for a, b, _ in kern) / 1e3, 3),
                      "lead_in_ms (first H2D -> first kernel)": round((t0 - first_h2d) / 1e3, 3),
                      "tail_ms (last kernel -> last D2H)": round((last_d2h - t1) / 1e3, 3),
                      "h2d_busy_ms": round(busy("h2d"), 3), "d2h_busy_ms": round(busy("d2h"), 3),
                      "gaps_over_20us": gaps[:40], "n_gaps": len(gaps),
                      "gap_total_ms": round(sum(g["gap_ms"] for g in gaps), 3)}))


if __name__ == "__main__":
    main()
