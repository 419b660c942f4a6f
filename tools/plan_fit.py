"""Per-rank latency of head plans against their cost features (dev tool, CPU).

Input: a bench.py JSON line (its `per_rank_projection`: layer 0 of the C3 stack)
or the JSON lines tools/skyline.py prints (`kind: sweep`, one per plan and
degree, any BASELINE config). The budget table is rebuilt on the CPU exactly as
the GPU run built it (C3: the reference-written table in oracle/tables, equal to
the bench's bit for bit; other configs: calibrate.layer_budgets with the host
profiler, equal to the GPU profiler's table), each plan is rebuilt as the
current code builds it, and
    ms = a * tiles + b * query_tiles + c * kv_heads + d
is fitted over all (plan, degree, rank) shards by least squares. Prints the fit,
its residual, and each plan's measured vs modelled bubble.

usage: python tools/plan_fit.py gpurun_out/v4/bench.json
       python tools/plan_fit.py profiles/r02/sweep/sweep.jsonl C4
(a line taken before greedy_refined moved to the weighted cost refits it
against the wrong plan)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_10353_b200 as P  # noqa: E402

BQ = 256
SHAPES = {"C1": (32, 8, 8192, 1), "C2": (32, 8, 32768, 1), "C3": (32, 8, 131072, 1), "C4": (28, 4, 65536, 1),
          "C5": (64, 8, 131072, 1), "C5x2": (64, 8, 131072, 2)}
C3_TABLE = os.path.join(ROOT, "oracle", "tables", "hq32_kv8_n131072_seed2603_rows128_q128.f0.25.allocation.json")


def budgets_for(cfg):
    hq, hkv, n, req = SHAPES[cfg]
    if cfg == "C3":
        d = json.load(open(C3_TABLE))
        return np.array([e["budget"] for e in sorted(d["budgets"], key=lambda e: e["head"])], np.int64)
    from paper_2603_10353_b200.calibrate import layer_budgets
    from paper_2603_10353_b200.workload import LayerSpec, make_layer
    out = []
    for r in range(req):  # as tools/skyline.py: request r has its own seed and table
        q, k, _ = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=2603 + 104729 * r), "cpu")
        out.append(layer_budgets(q, k, 0.25)[0])
    return np.concatenate(out).astype(np.int64)


def head_units(b, n):
    """(tiles, query tiles) per query block of a head with budget b."""
    nkb, nqb = (n + 127) // 128, (n + BQ - 1) // BQ
    qb = np.arange(nqb)
    vis = np.minimum((np.minimum((qb + 1) * BQ, n) - 1) // 128 + 1, nkb)
    t = np.minimum(min((int(b) + 127) // 128, nkb), vis) * 2
    return t, (t > 0) * 2


def plans_for(budgets, n, D):
    tc = P.tile_costs(budgets, n)
    wc = P.tile_costs(budgets, n, query_tile_weight=P.api.QUERY_TILE_WEIGHT)
    return {"naive": P.naive_assign(budgets, D), "greedy": P.greedy_assign(budgets, D),
            "greedy_tiles": P.greedy_assign(tc, D), "greedy_refined": P.refine_assign(wc, D, P.greedy_assign(wc, D)),
            "split": P.split_assign(budgets, D, n, query_tile_weight=P.api.QUERY_TILE_WEIGHT)}


def shard_features(budgets, n, group, plan_name, plan, D):
    hq, nqb = budgets.size, (n + BQ - 1) // BQ
    feats = []
    for r in range(D):
        if plan_name == "split":
            segs = [(int(h), int(a), int(e)) for d, h, a, e in zip(plan.device, plan.head, plan.qb_begin,
                                                                  plan.qb_end) if d == r]
        else:
            segs = [(h, 0, nqb) for h in range(hq) if plan[h] == r]
        tiles = qt = 0
        for h, a, e in segs:
            t, q = head_units(budgets[h], n)
            tiles += int(t[a:e].sum())
            qt += int(q[a:e].sum())
        feats.append((tiles, qt, len({h // group for h, _, _ in segs})))
    return feats


def load(path, cfg):
    """[(degree, plan, per_rank_ms)] and the config tag."""
    txt = open(path).read().strip()
    if cfg is None:  # a bench line
        line = json.loads(txt.splitlines()[-1])
        return [(int(D), name, rec["per_rank_ms"]) for D, plans in line["per_rank_projection"]["degrees"].items()
                for name, rec in plans.items() if "per_rank_ms" in rec], "C3"
    rows = [json.loads(x) for x in txt.splitlines() if x.startswith("{")]
    return [(r["degree"], r["assigner"], r["per_rank_ms"]) for r in rows
            if r.get("kind") == "sweep" and r["config"] == cfg], cfg


def main():
    runs, cfg = load(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
    hq, hkv, n, req = SHAPES[cfg]
    budgets = budgets_for(cfg)
    group = hq // hkv
    X, y, tags = [], [], []
    for D, name, per_rank in runs:
        plan = plans_for(budgets, n, D).get(name)
        if plan is None:
            continue
        for r, (f, ms) in enumerate(zip(shard_features(budgets, n, group, name, plan, D), per_rank)):
            if f[0] == 0:
                continue
            X.append([f[0], f[1], f[2], 1.0])
            y.append(ms)
            tags.append((D, name, r, f))
    X, y = np.array(X, float), np.array(y, float)
    coef, *_ = np.linalg.lstsq(X, y, rcond=None)
    pred = X @ coef
    a, b, c, d0 = coef
    print(json.dumps({"config": cfg, "ms_per_tile_us": a * 1e3, "ms_per_query_tile_us": b * 1e3,
                      "ms_per_kv_head": c, "ms_const": d0, "query_tile_in_tiles": b / a, "kv_head_in_tiles": c / a,
                      "rms_resid_ms": float(np.sqrt(np.mean((y - pred) ** 2))), "shards": len(y)}))
    rows = {}
    for (D, name, r, f), ms, p in zip(tags, y, pred):
        rows.setdefault((D, name), []).append((ms, p, a * f[0]))
    for (D, name), v in sorted(rows.items()):
        ms = np.array([x[0] for x in v])
        pm = np.array([x[1] for x in v])
        tm = np.array([x[2] for x in v])
        bub = lambda t: 1 - t.mean() / t.max()  # noqa: E731
        print(f"{cfg} D={D} {name:15s} measured bubble {bub(ms):.4f}  fit-model {bub(pm):.4f}  "
              f"tiles-only {bub(tm):.4f}  max resid {np.abs(ms - pm).max():.3f} ms")


if __name__ == "__main__":
    main()
