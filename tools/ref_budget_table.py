"""Budget tables written by the REFERENCE itself (oracle/_ref = headbal, unmodified),
for the bench's reference arm and for checking our table against it.

For a bench layer (same seed and generator as bench.py, generated on the GPU as
bench.py does), the calibration rows (calibrate.calibration_rows: 128 evenly
spaced positions) go through headbal::build_profiles (PerQueryTopK, no causal
mask, grid stride = quantum; profiler.cpp:157-196) on the GQA-expanded fp64
heads, then headbal::maxmin_allocate (allocator.cpp:97-186) at each requested
budget fraction. Written in the reference's own formats (save_profiles /
save_allocation) under oracle/tables/. The same layer's table from this repo's
GPU profiler + max-min is compared and the result recorded in
oracle/tables/<tag>.check.json.

The reference profile costs ~230 s per 128K head on one core (1025 grid points x
128 rows x an nth_element over 131072 weights), so this runs once, offline, on
the GPU box (its 16 host cores) — not inside the bench.

usage: python tools/ref_budget_table.py [--layer 0] [--fractions 0.25 0.0625]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_10353_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2603_10353_b200 import calibrate  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, bf16_bits, make_layer  # noqa: E402

TABLES = os.path.join(ROOT, "oracle", "tables")


def tag_of(hq, hkv, n, seed, rows, quantum):
    return f"hq{hq}_kv{hkv}_n{n}_seed{seed}_rows{rows}_q{quantum}"


def f64(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--q-heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--seq-len", type=int, default=131072)
    ap.add_argument("--seed", type=int, default=2603)
    ap.add_argument("--layer", type=int, default=0, help="bench layer index (seed + 7919 * layer)")
    ap.add_argument("--rows", type=int, default=128)
    ap.add_argument("--quantum", type=int, default=128)
    ap.add_argument("--floor", type=int, default=128)
    ap.add_argument("--fractions", type=float, nargs="+", default=[0.25, 0.0625])
    a = ap.parse_args()
    if not O.ref_available():
        raise SystemExit("oracle/_ref/libheadbal_ref.so missing (make -C oracle on a host with /root/reference)")
    hq, hkv, n = a.q_heads, a.kv_heads, a.seq_len
    seed = a.seed + 7919 * a.layer
    q, k, _v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=seed), "cuda")
    pos = calibrate.calibration_rows(n, a.rows)
    grid = P.default_budget_grid(n, a.quantum)
    group = hq // hkv
    # GQA-expanded fp64 heads as the reference's AttentionWorkload holds them.
    Q = np.stack([f64(bf16_bits(q[h][torch.as_tensor(pos, device=q.device)])) for h in range(hq)])
    Kg = [f64(bf16_bits(k[g])) for g in range(hkv)]
    Vg = [f64(bf16_bits(_v[g])) for g in range(hkv)]
    K = np.stack([Kg[h // group] for h in range(hq)])
    V = np.stack([Vg[h // group] for h in range(hq)])
    del Kg, Vg
    t0 = time.time()
    rec = O.ref.build_profiles(Q, K, V, grid, causal=False, kind=0)
    prof_s = time.time() - t0
    del K, V
    os.makedirs(TABLES, exist_ok=True)
    tag = tag_of(hq, hkv, n, seed, pos.size, a.quantum)
    O.ref.save_profiles(os.path.join(TABLES, f"{tag}.profiles.json"), [grid] * hq, list(rec), n)
    # ours: GPU profiler + max-min on the same rows
    ctx = P.Context(0)
    check = {"tag": tag, "layer": a.layer, "seed": seed, "rows": pos.size, "grid_stride": a.quantum,
             "reference_build_profiles_s": round(prof_s, 1), "threads": O.ref.max_threads(), "fractions": {}}
    ours_curves, _ = calibrate.profile_layer(q, k, kind="token", rows=a.rows, quantum=a.quantum, ctx=ctx)
    check["max_curve_diff"] = float(max(np.abs(c.recovery - r).max() for c, r in zip(ours_curves, rec)))
    for f in a.fractions:
        total = int(round(f * hq * n))
        ref_b, transfers, cap = O.ref.maxmin_allocate([(grid, r) for r in rec], n, total, quantum=a.quantum,
                                                      floor=a.floor)
        O.ref.save_allocation(os.path.join(TABLES, f"{tag}.f{f}.allocation.json"), ref_b, total, a.floor)
        ours, info, _ = calibrate.layer_budgets(q, k, f, kind="token", rows=a.rows, quantum=a.quantum,
                                                floor=a.floor, ctx=ctx)
        check["fractions"][str(f)] = {"total": total, "reference_digest": calibrate.table_digest(ref_b),
                                      "ours_digest": info["digest"], "match": bool(np.array_equal(ref_b, ours)),
                                      "reference_transfers": transfers, "ours_transfers": info["transfers"],
                                      "min": int(ref_b.min()), "max": int(ref_b.max())}
    with open(os.path.join(TABLES, f"{tag}.check.json"), "w") as fh:
        json.dump(check, fh, indent=1)
    print(json.dumps(check))


if __name__ == "__main__":
    main()
