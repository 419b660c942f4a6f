"""Time kernel 3 for several libshplb builds on one workload (dev tool).

usage: python tools/tune_fa.py lib1.so[:block_q] lib2.so ...   (each a full libshplb variant)
Each variant runs in a fresh subprocess (SHPLB_LIB=<path>) on the C3 128K layer with
the bench's max-min budget table; prints ms per layer, per-stage ms, SM clock, and the
board energy per layer from the NVML energy counter (at the power cap, time follows energy).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys, numpy as np, torch
sys.path.insert(0, %(root)r)
import paper_2603_10353_b200 as P
from paper_2603_10353_b200.workload import LayerSpec, make_layer, bf16_bits
n = %(n)d
q, k, v = make_layer(LayerSpec(seq_len=n, seed=2603), "cuda")
bfile = "/tmp/shplb_tune_budgets_%%d.npy" %% n
if os.path.exists(bfile):
    budgets = np.load(bfile)
else:
    curves = P.profile_curves(bf16_bits(q[:, n - 16:, :]), bf16_bits(k), P.default_budget_grid(n, 128))
    budgets = P.maxmin_allocate(curves, int(0.25 * 32 * n), 128, 128).budgets
    np.save(bfile, budgets)
ctx = P.Context(0)
out = torch.empty_like(q)
kw = {} if %(bq)d == 0 else {"block_q": %(bq)d}
for _ in range(3):
    ctx.sparse_attention_layer(q, k, v, budgets, out=out, **kw)
torch.cuda.synchronize()
ctx.set_timing(True)
import subprocess
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                        "-lms", "100"], stdout=subprocess.PIPE, text=True)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
try:
    import pynvml
    pynvml.nvmlInit()
    nvh = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    mj0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(nvh)
except Exception:
    nvh = None
e0.record()
for _ in range(%(steps)d):
    ctx.sparse_attention_layer(q, k, v, budgets, out=out, **kw)
e1.record()
torch.cuda.synchronize()
joules = (pynvml.nvmlDeviceGetTotalEnergyConsumption(nvh) - mj0) / 1e3 / %(steps)d if nvh is not None else None
smi.terminate()
vals = [l.split(",") for l in smi.communicate()[0].strip().splitlines() if "," in l]
clk = sorted(float(a) for a, b in vals) if vals else [0.0]
pw = sorted(float(b) for a, b in vals) if vals else [0.0]
st = ctx.read_timing().mean(0)
tiles, flops = P.layer_work(32, 8, n, budgets)
print(json.dumps({"ms": e0.elapsed_time(e1) / %(steps)d, "k3_ms": st[2], "k2_ms": st[1],
                  "k1_ms": st[0], "k3_tflops": flops / st[2] / 1e9,
                  "sm_mhz": clk[len(clk) // 2], "power_w": pw[len(pw) // 2],
                  "k3_mcycles": st[2] * clk[len(clk) // 2] / 1e3, "joules_per_layer": joules,
                  "avg_power_w": joules / (e0.elapsed_time(e1) / %(steps)d / 1e3) if joules else None}))
"""


def main():
    n = int(os.environ.get("TUNE_N", "131072"))
    steps = int(os.environ.get("TUNE_STEPS", "10"))
    for spec in sys.argv[1:]:  # path[:block_q]
        lib, _, bq = spec.partition(":")
        env = dict(os.environ, SHPLB_LIB=os.path.abspath(lib))
        args = {"root": ROOT, "n": n, "steps": steps, "bq": int(bq or 0)}
        r = subprocess.run([sys.executable, "-c", CHILD % args],
                           env=env, capture_output=True, text=True, timeout=240)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-2000:]
        print(spec.split("/")[-1], line, flush=True)


if __name__ == "__main__":
    main()
