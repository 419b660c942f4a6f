"""Per-rank latency of the bench's head plans against their cost features (dev
tool, CPU): reads a bench.py JSON line (its `per_rank_projection`, layer 0 of
the C3 stack, every plan's per-rank ms) and the layer-0 budget table the bench
used (the reference-built table in oracle/tables, equal to the bench's own bit
for bit), rebuilds each plan, and fits
    ms = a * tiles + b * query_tiles + c * kv_heads + d
over all (plan, degree, rank) shards by least squares. Prints the fit, its
residuals, and each plan's modelled vs measured bubble.

usage: python tools/plan_fit.py gpurun_out/v4/bench.json
(the greedy_refined plan is rebuilt as the current bench builds it: a line taken
before it moved to the weighted cost refits against the wrong plan)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_10353_b200 as P  # noqa: E402

N, HQ, HKV, BQ = 131072, 32, 8, 256
TABLE = os.path.join(ROOT, "oracle", "tables", "hq32_kv8_n131072_seed2603_rows128_q128.f0.25.allocation.json")


def head_units(b):
    """(tiles, query tiles) per query block of a head with budget b."""
    nkb, nqb = (N + 127) // 128, (N + BQ - 1) // BQ
    qb = np.arange(nqb)
    vis = np.minimum((np.minimum((qb + 1) * BQ, N) - 1) // 128 + 1, nkb)
    t = np.minimum(min((int(b) + 127) // 128, nkb), vis) * 2
    return t, (t > 0) * 2


def shard_features(budgets, plan_name, plan, D):
    g = HQ // HKV
    feats = []
    for r in range(D):
        if plan_name == "split":
            segs = [(int(h), int(a), int(e)) for d, h, a, e in zip(plan.device, plan.head, plan.qb_begin,
                                                                  plan.qb_end) if d == r]
        else:
            segs = [(h, 0, (N + BQ - 1) // BQ) for h in range(HQ) if plan[h] == r]
        tiles = qt = 0
        for h, a, e in segs:
            t, q = head_units(budgets[h])
            tiles += int(t[a:e].sum())
            qt += int(q[a:e].sum())
        kv = len({h // g for h, _, _ in segs})
        feats.append((tiles, qt, kv))
    return feats


def main():
    line = json.load(open(sys.argv[1]))
    d = json.load(open(TABLE))
    budgets = np.array([e["budget"] for e in sorted(d["budgets"], key=lambda e: e["head"])], np.int64)
    proj = line["per_rank_projection"]["degrees"]
    X, y, tags = [], [], []
    for D_s, plans in proj.items():
        D = int(D_s)
        tc = P.tile_costs(budgets, N)
        built = {"naive": P.naive_assign(budgets, D), "greedy": P.greedy_assign(budgets, D),
                 "greedy_tiles": P.greedy_assign(tc, D)}
        wc = P.tile_costs(budgets, N, query_tile_weight=P.api.QUERY_TILE_WEIGHT)
        built["greedy_refined"] = P.refine_assign(wc, D, P.greedy_assign(wc, D))
        built["split"] = P.split_assign(budgets, D, N)
        for name, rec in plans.items():
            if "per_rank_ms" not in rec or name not in built:
                continue
            for r, (f, ms) in enumerate(zip(shard_features(budgets, name, built[name], D), rec["per_rank_ms"])):
                if f[0] == 0:
                    continue
                X.append([f[0], f[1], f[2], 1.0])
                y.append(ms)
                tags.append((D, name, r, f))
    X, y = np.array(X, float), np.array(y, float)
    coef, *_ = np.linalg.lstsq(X, y, rcond=None)
    pred = X @ coef
    a, b, c, d0 = coef
    print(json.dumps({"ms_per_tile_us": a * 1e3, "ms_per_query_tile_us": b * 1e3, "ms_per_kv_head": c,
                      "ms_const": d0, "query_tile_in_tiles": b / a, "kv_head_in_tiles": c / a,
                      "rms_resid_ms": float(np.sqrt(np.mean((y - pred) ** 2))), "shards": len(y)}))
    rows = {}
    for (D, name, r, f), ms, p in zip(tags, y, pred):
        rows.setdefault((D, name), []).append((ms, p, a * f[0]))
    for (D, name), v in sorted(rows.items()):
        ms = np.array([x[0] for x in v])
        pm = np.array([x[1] for x in v])
        tm = np.array([x[2] for x in v])
        bub = lambda t: 1 - t.mean() / t.max()  # noqa: E731
        print(f"D={D} {name:15s} measured bubble {bub(ms):.4f}  fit-model {bub(pm):.4f}  tiles-only {bub(tm):.4f}  "
              f"max resid {np.abs(ms - pm).max():.3f} ms")


if __name__ == "__main__":
    main()
