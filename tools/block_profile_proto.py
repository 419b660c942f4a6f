"""Prototype (dev tool): recovery curves of the kernels' OWN selection policy
(top-k 128-key blocks ranked by pooled block score, causal, rows spread over
the whole sequence) vs the reference's token-level PerQueryTopK curves on the
last rows; compare the skyline error of max-min budgets from each.

usage: python tools/block_profile_proto.py C3
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200 import experiments as X  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402

CONFIGS = {"C1": (32, 8, 8192), "C3": (32, 8, 131072), "C4": (28, 4, 65536)}
cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
hq, hkv, n = CONFIGS[cfg]
R = int(os.environ.get("ROWS", "64"))
TARGETS = os.environ.get("TARGETS", "per_query")
q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=2603, targets=TARGETS), "cuda")
ctx = P.Context(0)
grid = P.default_budget_grid(n, 128)
bq = P.BLOCK_Q
sc = ctx.block_scores(q, k, causal=True, block_q=bq)  # [hq, nqb, nkb] fp32, -inf invisible
torch.cuda.synchronize()
nkb = (n + 127) // 128
pos = torch.tensor([(r + 1) * n // R - 1 for r in range(R)], device="cuda")
group = hq // hkv
curves = []
tok_spread = []
for h in range(hq):
    qr = q[h, pos].float()
    s = (qr @ k[h // group].float().T) / (128 ** 0.5)
    keyidx = torch.arange(n, device="cuda")
    s = s.masked_fill(keyidx[None, :] > pos[:, None], float("-inf"))
    w = torch.softmax(s.double(), dim=-1)
    pad = nkb * 128 - n
    if pad:
        w = torch.nn.functional.pad(w, (0, pad))
    mass = w.view(R, nkb, 128).sum(-1)  # [R, nkb]
    bs = sc[h, pos // bq].double()  # [R, nkb] pooled scores of each row's query block
    # rank desc, ties by lower index: sort by (-score, index) via stable argsort of -score
    order = torch.argsort(-bs, dim=-1, stable=True)
    cm = torch.cumsum(torch.gather(mass, 1, order), dim=-1)  # [R, nkb]
    cm = torch.cat([torch.zeros(R, 1, dtype=cm.dtype, device="cuda"), cm], dim=1)
    kb = torch.clamp(torch.as_tensor((grid + 127) // 128, device="cuda"), max=nkb)
    rec = cm[:, kb].mean(0).cpu().numpy()
    rec[-1] = 1.0
    rec = np.maximum.accumulate(np.minimum(rec, 1.0))
    curves.append(P.RecoveryCurve(grid.copy(), rec, n))
    # token-level PerQueryTopK on the same spread, causal rows
    ws = torch.sort(w[:, :n], dim=-1, descending=True).values
    cw = torch.cat([torch.zeros(R, 1, dtype=ws.dtype, device="cuda"), torch.cumsum(ws, dim=-1)], dim=1)
    rt = cw[:, torch.as_tensor(grid, device="cuda")].mean(0).cpu().numpy()
    rt[-1] = 1.0
    tok_spread.append(P.RecoveryCurve(grid.copy(), np.maximum.accumulate(np.minimum(rt, 1.0)), n))
tok = ctx.profile_curves(q[:, n - 16:, :].contiguous(), k, grid)
dense = ctx.dense_attention_layer(q, k, v)
out = torch.empty_like(q)
res = {}
for frac in (0.125, 0.25, 0.5):
    total = int(round(frac * hq * n))
    for name, cv in (("uniform", None), ("maxmin_token", tok), ("maxmin_token_spread", tok_spread),
                     ("maxmin_block", curves)):
        b = (P.uniform_allocate(hq, total, 128, n).budgets if cv is None
             else P.maxmin_allocate(cv, total, quantum=128, floor=128).budgets)
        ctx.sparse_attention_layer(q, k, v, b, out=out)
        torch.cuda.synchronize()
        errs = [X.output_error(out[h], dense[h]) for h in range(hq)]
        res[f"{frac}:{name}"] = (round(float(np.mean(errs)), 4), round(float(np.max(errs)), 4))
        print(json.dumps({"config": cfg, "targets": TARGETS, "fraction": frac, "alloc": name,
                          "mean_err": res[f"{frac}:{name}"][0],
                          "max_err": res[f"{frac}:{name}"][1]}), flush=True)
