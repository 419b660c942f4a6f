"""Near-tie report: where kernel 2's fp32 block selection differs from an fp64
ranking of the same pooled blocks (north_star: "any near-tie divergence must be
documented").

For each BASELINE config (C1-C5, C5 with two requests stacked on the head
axis), layer 0 of the bench's generator with its max-min budget table (token
PerQueryTopK curves of 128 evenly spaced calibration rows; fractions 0.25 and
0.0625), the layer call's selection (kernels 1-2, fp32, bit-exact with the C
oracle) is compared row by row — one row = one (head, query block) — with the
selection the reference's rules make on fp64 scores: pooled Q / K block means in
fp64 (exact sums of bf16 values), dot product in fp64, scale 1/sqrt(d) after
the dot (attention.cpp:20,26), causal visibility (attention.cpp:28-30), the
min(k_h, visible) largest under (score desc, index asc) (attention.cpp:53-64).

For every divergent row it records how many blocks differ and the fp64 score
gap between the last block kept and the first block dropped by the fp64
ranking, relative to the score magnitude: a near-tie at fp32 resolution
(2^-24 ~ 6e-8 relative rounding per operation, ~1e-6 after a 128-term dot) is
what makes fp32 and fp64 disagree.

usage: python tools/near_tie_report.py [C1 C2 ...]  -> JSON lines (profiles/r02/near_tie.jsonl)
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200 import calibrate  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402

CONFIGS = {  # q heads, kv heads, n, requests
    "C1": (32, 8, 8192, 1), "C2": (32, 8, 32768, 1), "C3": (32, 8, 131072, 1),
    "C4": (28, 4, 65536, 1), "C5": (64, 8, 131072, 2),
}


def fp64_selection(q, k, bq, counts):
    """idx [H, nqb, kmax] (ascending, -1 padded) of the fp64 ranking, and the
    relative boundary gap per row."""
    hq, n, d = q.shape
    hkv = k.shape[0]
    group = hq // hkv
    nqb, nkb = n // bq, n // 128
    kmax = int(counts.max())
    qp = q.view(hq, nqb, bq, d).double().mean(2)
    kp = k.view(hkv, nkb, 128, d).double().mean(2)
    idx = torch.full((hq, nqb, kmax), -1, dtype=torch.int64, device=q.device)
    gap = torch.full((hq, nqb), float("inf"), dtype=torch.float64, device=q.device)
    vis = torch.clamp(((torch.arange(nqb, device=q.device) + 1) * bq - 1) // 128 + 1, max=nkb)
    cols = torch.arange(nkb, device=q.device)
    for h in range(hq):
        s = (qp[h] @ kp[h // group].T) * (1.0 / np.sqrt(d))  # [nqb, nkb] fp64
        s = torch.where(cols[None, :] < vis[:, None], s, torch.full_like(s, -float("inf")))
        order = torch.sort(s, dim=1, descending=True, stable=True)  # stable: ties -> lower index first
        c = counts[h].to(q.device)
        keep = torch.arange(nkb, device=q.device)[None, :] < c[:, None]
        chosen = torch.where(keep, order.indices, torch.full_like(order.indices, nkb))
        chosen = torch.sort(chosen, dim=1).values[:, :kmax]
        idx[h] = torch.where(chosen < nkb, chosen, torch.full_like(chosen, -1))
        # gap between the last kept and the first dropped fp64 score (rows that drop something)
        ci = torch.clamp(c - 1, min=0).long()
        last = order.values.gather(1, ci[:, None])[:, 0]
        nxt = order.values.gather(1, torch.clamp(c, max=nkb - 1).long()[:, None])[:, 0]
        scale = torch.maximum(last.abs(), torch.tensor(1e-300, dtype=torch.float64, device=q.device))
        has_drop = (c < vis) & torch.isfinite(nxt)
        gap[h] = torch.where(has_drop, (last - nxt) / scale, gap[h])
    return idx, gap


def report(cfg, fraction, ctx):
    hq, hkv, n, reqs = CONFIGS[cfg]
    parts, budgets = [], []
    for r in range(reqs):
        q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=2603 + 101 * r), "cuda")
        b, _, _ = calibrate.layer_budgets(q, k, fraction, kind="token", rows=128, ctx=ctx)
        parts.append((q, k, v))
        budgets.append(b)
    q, k, v = (torch.cat([p[i] for p in parts]) if reqs > 1 else parts[0][i] for i in range(3))
    b = np.concatenate(budgets)
    bq = P.BLOCK_Q
    ctx.sparse_attention_layer(q, k, v, b, block_q=bq)
    idx_g, cnt_g = ctx.last_selection(q.shape[0], n)
    torch.cuda.synchronize()
    idx64, gap = fp64_selection(q, k, bq, cnt_g)
    kmax = idx64.shape[2]
    g = idx_g[:, :, :kmax].long()
    diff_rows = (g != idx64).any(dim=2)
    rows = int(diff_rows.numel())
    nd = int(diff_rows.sum())
    out = {"config": cfg, "fraction": fraction, "q_heads": int(q.shape[0]), "seq_len": n, "block_q": bq,
           "rows": rows, "divergent_rows": nd, "divergent_fraction": nd / rows,
           "rows_with_a_drop": int(torch.isfinite(gap).sum())}
    if nd:
        # blocks differing per divergent row (symmetric difference / 2)
        dcount = []
        hs, qs = torch.nonzero(diff_rows, as_tuple=True)
        for h, qb in zip(hs.tolist()[:2000], qs.tolist()[:2000]):
            a = set(g[h, qb][g[h, qb] >= 0].tolist())
            c = set(idx64[h, qb][idx64[h, qb] >= 0].tolist())
            dcount.append(len(a ^ c) // 2)
        gd = gap[diff_rows]
        out.update({"max_blocks_differing": int(max(dcount)), "mean_blocks_differing": float(np.mean(dcount)),
                    "max_rel_gap_divergent": float(gd.max()), "median_rel_gap_divergent": float(gd.median()),
                    "median_rel_gap_all_rows": float(gap[torch.isfinite(gap)].median())})
    return out


def main():
    cfgs = sys.argv[1:] or list(CONFIGS)
    ctx = P.Context(0)
    for cfg in cfgs:
        for f in (0.25, 0.0625):
            print(json.dumps(report(cfg, f, ctx)), flush=True)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
