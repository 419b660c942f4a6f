"""Measured sweep and skyline for a BASELINE config; CSVs in
the reference's columns (write_sweep_csv / write_skyline_csv), latencies in ms.

usage: python tools/skyline.py C3 --out profiles/r02/skyline [--degrees 1 2 4 8] [--steps 3]
       [--profile-kind token|block] [--targets per_query|per_head] [--fractions 0.0625 0.25 0.5]

Budget tables: max-min on recovery curves of 128 evenly spaced calibration rows
(calibrate.profile_layer): 'token' = the reference's PerQueryTopK curves,
'block' = the kernels' own block selection (shplb_profile_curves_block).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200 import calibrate  # noqa: E402
from paper_2603_10353_b200 import experiments as X  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402

CONFIGS = {"C1": (32, 8, 8192), "C2": (32, 8, 32768), "C3": (32, 8, 131072), "C4": (28, 4, 65536),
           "C5": (64, 8, 131072)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CONFIGS))
    ap.add_argument("--out", default="gpurun_out")
    ap.add_argument("--degrees", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--calib-rows", type=int, default=128)
    ap.add_argument("--profile-kind", choices=["token", "block"], default="token")
    ap.add_argument("--targets", choices=["per_query", "per_head"], default="per_query",
                    help="synthetic generator: per-query random targets, or per-head hot key blocks")
    ap.add_argument("--floor", type=int, default=128, help="AllocatorConfig.floor (tokens) of both tables")
    ap.add_argument("--fractions", type=float, nargs="+", default=[0.25, 0.5, 0.75, 1.0],
                    help="skyline total budgets as fractions of Hq*n")
    ap.add_argument("--skyline-devices", type=int, default=8)
    ap.add_argument("--requests", type=int, default=1,
                    help="batched multi-request prefill: R independent requests stacked along the "
                         "head axis (R*Hq balancer units; each request profiled and allocated on its own)")
    ap.add_argument("--no-skyline", action="store_true")
    a = ap.parse_args()
    hq, hkv, n = CONFIGS[a.config]
    ctx = P.Context(0)
    qs, ks, vs, bs, cs = [], [], [], [], []
    for r in range(a.requests):  # heads of request r are [r*hq, (r+1)*hq); GQA grouping is preserved
        q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=2603 + 104729 * r,
                                       targets=a.targets), "cuda")
        curves, _ = calibrate.profile_layer(q, k, kind=a.profile_kind, rows=a.calib_rows, ctx=ctx)
        bs.append(P.maxmin_allocate(curves, int(round(0.25 * hq * n)), quantum=128, floor=a.floor).budgets)
        qs.append(q), ks.append(k), vs.append(v), cs.extend(curves)
    if a.requests > 1:
        q, k, v = torch.cat(qs), torch.cat(ks), torch.cat(vs)
        del qs, ks, vs
    budgets = np.concatenate(bs)
    tag = a.config if a.requests == 1 else f"{a.config}x{a.requests}"
    tag += ("" if a.profile_kind == "token" else "_block") + ("" if a.targets == "per_query" else "_perhead")
    tag += "" if a.floor == 128 else f"_floor{a.floor}"
    os.makedirs(a.out, exist_ok=True)
    rows = X.measured_sweep(ctx, {n: (q, k, v, budgets)}, a.degrees, steps=a.steps)
    X.write_sweep_csv(os.path.join(a.out, f"sweep_{tag}.csv"), rows)
    for r in rows:
        print(json.dumps({"kind": "sweep", "config": tag, "requests": a.requests,
                          **{k_: v_ for k_, v_ in r.__dict__.items()}}), flush=True)
    if a.no_skyline:
        return
    curves = cs
    totals = [int(round(f * q.shape[0] * n)) for f in a.fractions]
    pts = X.measured_skyline(ctx, q, k, v, curves, devices=a.skyline_devices, steps=a.steps, totals=totals,
                             floor=a.floor)
    X.write_skyline_csv(os.path.join(a.out, f"skyline_{tag}.csv"), pts)
    for p in pts:
        print(json.dumps({"kind": "skyline", "config": tag, "profile_kind": a.profile_kind, "floor": a.floor,
                          "targets": a.targets, "fraction": p.total_budget / (q.shape[0] * n),
                          **p.__dict__}), flush=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
