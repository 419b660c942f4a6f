"""CPU anchor: one whole C1 layer — 32 q / 8 kv heads x 8192
tokens, causal, every head through the reference's headbal::sparse_attention
with its reference-built max-min budget (the run_skyline loop,
commands.cpp:464-470) — timed end to end on this host's cores, best of 3
(bench_attention.cpp:71-90), beside the sampled estimator bench.py uses for
C3. Needs the GPU only to generate the seeded inputs.

usage: python tools/cpu_anchor.py [repeats=3]  -> one JSON line
"""
import json
import os
import sys
from types import SimpleNamespace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import oracle as O  # noqa: E402

repeats = int(sys.argv[1]) if len(sys.argv) > 1 else 3
args = SimpleNamespace(seed=2603, budget_fraction=0.25, calib_rows=128)
res = bench.c1_full_layer(args, repeats)
res.update({"threads": O.ref.max_threads(), "cpu_model": bench.cpu_model()})
print(json.dumps(res))
