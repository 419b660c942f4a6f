"""Generate tests/golden/*.json by running the UNMODIFIED reference library
(oracle/_ref/libheadbal_ref.so, compiled from /root/reference/proj/src).

Run here (the container that has /root/reference):  python tools/make_golden.py
The fixtures are small and committed; the GPU box never needs the reference.

Contents
* attention_kat.json   — token-level sparse/dense attention outputs of the
  reference (headbal::sparse_attention / dense_attention) on small seeded heads
  with bf16-exact integer Q/K (so fp32 and fp64 rank scores identically) and
  the in-code known answers of proj/tests/test_attention.cpp (single key, zero
  Q, two-key softmax, ties -> lower index, full budget == dense).
* budget_kat.json      — uniform / max-min budget tables (allocator.cpp) incl.
  the 2-head worked instance of test_allocator.cpp:79-94 and max-min on
  curves profiled by the reference's own build_profiles.
* plan_kat.json        — naive / greedy plans, loads, imbalance, simulate
  (partitioner.cpp, simulator.cpp) for the SURVEY §4 known answers and seeded
  random budget vectors.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def ramp(n_k, sat, stride):
    b = list(range(0, n_k + 1, stride))
    if b[-1] != n_k:
        b.append(n_k)
    r = [min(1.0, x / sat) for x in b]
    return b, r


def attention_kat():
    rng = np.random.default_rng(2603)
    cases = []
    for seed in range(12):
        n_q, n_k = int(rng.integers(2, 6)), int(rng.integers(8, 24))
        d = [4, 16, 64][seed % 3]
        Q = rng.integers(-3, 4, (n_q, d)).astype(np.float64)
        K = rng.integers(-3, 4, (n_k, d)).astype(np.float64)
        V = np.round(rng.standard_normal((n_k, d)) * 64) / 64  # bf16-exact
        outs = []
        for causal in (False, True):
            for k in sorted({1, 3, min(7, n_k), n_k}):
                out = O.ref.sparse_attention(Q, K, V, k, causal=causal)
                outs.append({"k": k, "causal": causal, "out": np.round(out, 15).tolist()})
        cases.append({"name": f"rand{seed}", "Q": Q.tolist(), "K": K.tolist(), "V": V.tolist(),
                      "outputs": outs})
    # In-code known answers of proj/tests/test_attention.cpp.
    kat = []
    kat.append({"name": "single_key", "Q": [[0.3, -1.7]], "K": [[2.0, 0.5]], "V": [[4.0, -9.0]],
                "k": 1, "causal": False})
    kat.append({"name": "two_key_softmax", "Q": [[1.0, 0.0]], "K": [[1.0, 0.0], [0.0, 1.0]],
                "V": [[1.0, 2.0], [3.0, 4.0]], "k": 2, "causal": False})
    kat.append({"name": "ties_lower_index", "Q": [[1.0, 0.0]],
                "K": [[1.0, 0.0], [1.0, 0.0], [0.0, 1.0]],
                "V": [[10.0, 0.0], [-10.0, 0.0], [0.0, 0.0]], "k": 1, "causal": False})
    kat.append({"name": "zero_q_uniform", "Q": [[0.0] * 3] * 2,
                "K": [[1, 2, 0], [0, 1, 1], [2, 0, 1], [1, 1, 1]],
                "V": [[1, 0, 2], [0, 3, 1], [2, 2, 0], [1, 1, 1]], "k": 4, "causal": False})
    for c in kat:
        c["out"] = O.ref.sparse_attention(np.array(c["Q"], float), np.array(c["K"], float),
                                          np.array(c["V"], float), c["k"], causal=c["causal"]).tolist()
        c["dense"] = O.ref.dense_attention(np.array(c["Q"], float), np.array(c["K"], float),
                                           np.array(c["V"], float)).tolist()
    return {"source": "headbal::sparse_attention / dense_attention (oracle/_ref)",
            "random": cases, "kat": kat}


def budget_kat():
    out = {"source": "headbal::uniform_allocate / maxmin_allocate (oracle/_ref)"}
    out["uniform"] = [
        {"args": [4, 4096, 0, 4096], "budgets": O.ref.uniform_allocate(4, 4096, 0, 4096).tolist()},
        {"args": [3, 10, 1, 16], "budgets": O.ref.uniform_allocate(3, 10, 1, 16).tolist()},
    ]
    worked = [ramp(4096, 256, 64), ramp(4096, 4096, 64)]
    b, tr, cap = O.ref.maxmin_allocate(worked, 4096, 2048, quantum=64, floor=128)
    out["maxmin_worked"] = {"curves": worked, "n_k": 4096, "total": 2048, "quantum": 64,
                            "floor": 128, "budgets": b.tolist(), "transfers": tr}
    # curves from the reference's own profiler on seeded heads
    rng = np.random.default_rng(7)
    profiled = []
    for case in range(4):
        h, n_q, n_k, d = 6, 4, 512, 8
        Q = rng.standard_normal((h, n_q, d)) * rng.uniform(0.3, 3.0, (h, 1, 1))
        K = rng.standard_normal((h, n_k, d))
        V = rng.standard_normal((h, n_k, d))
        grid = list(range(0, n_k, 32)) + [n_k]
        rec = O.ref.build_profiles(Q, K, V, grid)
        curves = [(grid, rec[i].tolist()) for i in range(h)]
        total = h * 192
        b, tr, cap = O.ref.maxmin_allocate(curves, n_k, total, quantum=32, floor=64)
        profiled.append({"curves": curves, "n_k": n_k, "total": total, "quantum": 32, "floor": 64,
                         "budgets": b.tolist(), "transfers": tr, "hit_cap": cap})
    out["maxmin_profiled"] = profiled
    return out


def plan_kat():
    out = {"source": "headbal::naive_assign / greedy_assign / imbalance / simulate (oracle/_ref)"}
    cases = [([7, 6, 5, 4, 3, 2], 2), ([3, 3, 2, 2, 2], 2), ([8, 8, 1, 1], 2), ([128] * 28, 8)]
    rng = np.random.default_rng(11)
    for _ in range(12):
        n = int(rng.integers(4, 65))
        dev = int(rng.choice([2, 3, 4, 8]))
        if dev > n:
            dev = n
        b = (rng.integers(1, 64, n) * 128).tolist()
        cases.append((b, dev))
    rows = []
    for b, dev in cases:
        g = O.ref.greedy_assign(b, dev)
        nv = O.ref.naive_assign(b, dev)
        rr = O.ref.naive_assign(b, dev, round_robin=True)
        lg, ig, ag = O.ref.imbalance(b, g, dev)
        ln, inn, an = O.ref.imbalance(b, nv, dev)
        lat, T, bub = O.ref.simulate(lg, 0.0, 1.0)
        rows.append({"budgets": list(map(int, b)), "devices": dev, "greedy": g.tolist(),
                     "naive": nv.tolist(), "round_robin": rr.tolist(),
                     "greedy_loads": lg.tolist(), "greedy_imbalance": ig,
                     "naive_loads": ln.tolist(), "naive_imbalance": inn,
                     "greedy_barrier": T, "greedy_bubble": bub})
    out["cases"] = rows
    return out


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: make -C oracle (needs /root/reference)")
    os.makedirs(OUT, exist_ok=True)
    for name, fn in [("attention_kat", attention_kat), ("budget_kat", budget_kat),
                     ("plan_kat", plan_kat)]:
        with open(os.path.join(OUT, name + ".json"), "w") as f:
            json.dump(fn(), f)
        print("wrote", name)


if __name__ == "__main__":
    main()
