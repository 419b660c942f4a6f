"""Where kernel 3's cycles go, tile by tile (dev tool, GPU).

usage: SHPLB_LIB=<trace build of the persistent kernel> python tools/tile_trace.py --persist [out.json]
(build: K3=persist tools/build_variants.sh ttp "-DSHPLB_TILETRACE")

Runs the C3 128K layer (the bench's layer-0 inputs and max-min table), reads the per-CTA
timestamps the trace build records (entry, setup done, first S landed, last P.V landed,
output stored, exit; clock64 of the SM the CTA ran on) and splits the launch's SM-cycles into
  prologue   entry -> first S landed (barrier init, TMEM alloc, cluster sync, Q/K load, S(0))
  steady     first S -> last P.V landed (per block: steady / nsel)
  epilogue   last P.V -> exit (merge, TMA store, cluster sync, dealloc)
  gap        exit of a CTA -> entry of the next CTA on the same SM (launch of the next cluster)
  tail       last exit on the SM -> the launch's last exit
The fit steady = a + b * nsel over all tiles gives the per-block period b.
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from paper_2603_10353_b200 import _native  # noqa: E402
from paper_2603_10353_b200.calibrate import layer_budgets  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, make_layer  # noqa: E402

persist = "--persist" in sys.argv
if persist:
    sys.argv.remove("--persist")
n = int(os.environ.get("TUNE_N", "131072"))
q, k, v = make_layer(LayerSpec(seq_len=n, seed=2603), "cuda")
ctx = P.Context(0)
budgets, _, _ = layer_budgets(q, k, 0.25, ctx=ctx)
out = torch.empty_like(q)
for _ in range(3):
    ctx.sparse_attention_layer(q, k, v, budgets, out=out)
torch.cuda.synchronize()
if persist:
    assert C.CDLL(_native.LIB_PATH).shplb_debug_tiletrace_persist_clear() == 0
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
ctx.sparse_attention_layer(q, k, v, budgets, out=out)
e1.record()
torch.cuda.synchronize()
layer_ms = e0.elapsed_time(e1)

lib = C.CDLL(_native.LIB_PATH)
if persist:
    # per tile (schedule order): first S landed, last P.V landed, epilogue done, smid | nsel << 32
    buf = np.zeros((1 << 16, 12), dtype=np.uint64)  # [cluster * 512 + tile of the cluster]
    assert lib.shplb_debug_tiletrace_persist(buf.ctypes.data_as(C.c_void_p), C.c_size_t(buf.nbytes)) == 0
    t = buf[buf[:, 3] != 0].astype(np.int64)
    ntile = len(t)
    s0, pv, ep = t[:, 0], t[:, 1], t[:, 2]
    smid, nsel = t[:, 3] & 0xFFFFFFFF, t[:, 3] >> 32
    steady = pv - s0
    A = np.stack([np.ones(ntile), nsel], 1).astype(np.float64)
    coef, *_ = np.linalg.lstsq(A, steady.astype(np.float64), rcond=None)
    bound, spans, parts = [], [], []
    for sm in np.unique(smid):
        o = np.where(smid == sm)[0]
        o = o[np.argsort(s0[o])]
        bound.extend((s0[o[1:]] - pv[o[:-1]]).tolist())  # last P.V of a tile -> first S of the next seen
        spans.append(ep[o[-1]] - s0[o[0]])
        a, b = o[:-1], o[1:]  # previous tile, next tile; times relative to the previous tile's last P.V
        parts.append(np.stack([t[a, 2] - pv[a], t[a, 4] - pv[a], t[b, 7] - pv[a], t[b, 5] - pv[a],
                               t[b, 6] - pv[a], s0[b] - pv[a], t[b, 8] - pv[a], t[b, 9] - pv[a],
                               t[b, 10] - pv[a], t[a, 11] - pv[a]], 1))
    parts = np.concatenate(parts)
    boundary_detail = dict(zip(["staged", "stored", "next_q_issued", "next_q_seen_by_s_issuer",
                                "next_s0_issued", "next_s0_seen_by_softmax", "next_s0_past_s_free",
                                "next_s0_past_k_full", "next_k0_issued", "last_s_issued"],
                               [float(np.median(parts[:, i])) for i in range(parts.shape[1])]))
    res = {"layer_ms": layer_ms, "tiles": int(ntile), "leader_sms": int(len(spans)),
           "fit_steady_cycles": {"per_tile": float(coef[0]), "per_block": float(coef[1])},
           "mean_cycles_per_tile": {"steady": float(steady.mean()), "epilogue": float((ep - pv).mean()),
                                    "boundary_last_pv_to_next_first_s": float(np.mean(bound))},
           "boundary_median_cycles_after_last_pv": boundary_detail,
           "share_of_span": {"steady": float(steady.sum() / np.sum(spans)),
                             "boundaries": float(np.sum(bound) / np.sum(spans))},
           "span_cycles": {"mean": float(np.mean(spans)), "min": float(np.min(spans)), "max": float(np.max(spans))},
           "steady_cycles_per_block_total": float(steady.sum() / nsel.sum())}
    print(json.dumps(res, indent=1))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(res, f, indent=1)
        np.save(sys.argv[1].replace(".json", ".npy"), t)
    sys.exit(0)
ncta = 2 * int(np.ceil(n / 256)) * 32
buf = np.zeros((1 << 16, 8), dtype=np.uint64)
rc = lib.shplb_debug_tiletrace(buf.ctypes.data_as(C.c_void_p), C.c_size_t(buf.nbytes))
assert rc == 0, rc
t = buf[:ncta].astype(np.int64)
smid = t[:, 1] & 0xFFFFFFFF
nsel = t[:, 1] >> 32
c_entry, c_setup, c_s0, c_pv, c_st, c_exit = t[:, 2], t[:, 3], t[:, 4], t[:, 5], t[:, 6], t[:, 7]
live = nsel > 0
pro = (c_s0 - c_entry)[live]
steady = (c_pv - c_s0)[live]
epi = (c_exit - c_pv)[live]
A = np.stack([np.ones(live.sum()), nsel[live]], 1).astype(np.float64)
coef, *_ = np.linalg.lstsq(A, steady.astype(np.float64), rcond=None)
gaps, tails, busy = [], [], []
last_exit = 0
per_sm_span = []
for s in np.unique(smid):
    m = np.where(smid == s)[0]
    o = m[np.argsort(c_entry[m])]
    gaps.extend((c_entry[o[1:]] - c_exit[o[:-1]]).tolist())
    per_sm_span.append((c_entry[o[0]], c_exit[o[-1]], (c_exit[o] - c_entry[o]).sum(), len(o)))
span = np.array([b - a for a, b, _, _ in per_sm_span], dtype=np.float64)
busy = np.array([c for _, _, c, _ in per_sm_span], dtype=np.float64)
tot_pro, tot_steady, tot_epi = pro.sum(), steady.sum(), epi.sum()
nsm = len(per_sm_span)
res = {
    "layer_ms": layer_ms, "ctas": int(ncta), "sms": int(nsm), "blocks_per_cta_mean": float(nsel.mean()),
    "fit_steady_cycles": {"per_tile": float(coef[0]), "per_block": float(coef[1])},
    "mean_cycles_per_cta": {"prologue": float(pro.mean()), "setup": float((c_setup - c_entry)[live].mean()),
                            "first_s_after_setup": float((c_s0 - c_setup)[live].mean()),
                            "steady": float(steady.mean()), "epilogue": float(epi.mean()),
                            "epi_store": float((c_st - c_pv)[live].mean()),
                            "gap_between_ctas": float(np.mean(gaps))},
    "share_of_sm_span": {
        "prologue": float(tot_pro / span.sum()), "steady": float(tot_steady / span.sum()),
        "epilogue": float(tot_epi / span.sum()), "gaps": float(np.sum(gaps) / span.sum()),
    },
    "sm_span_cycles": {"mean": float(span.mean()), "min": float(span.min()), "max": float(span.max())},
    "tiles_per_sm": {"min": int(min(x[3] for x in per_sm_span)), "max": int(max(x[3] for x in per_sm_span))},
    "steady_cycles_per_block_total": float(tot_steady / nsel[live].sum()),
    "span_cycles_per_block": float(span.mean() * nsm / nsel.sum()),
}
print(json.dumps(res, indent=1))
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(res, f, indent=1)
    np.save(sys.argv[1].replace(".json", ".npy"), t)
