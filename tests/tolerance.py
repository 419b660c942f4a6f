"""Output tolerance of kernel 3 against the fp64 oracle, derived from the bf16 floor.

Kernel 3 writes bf16, so even an exact kernel differs from the fp64 oracle by the
rounding of its output to bf16. That rounding alone sets a floor on the mean
relative error of every comparison:

    floor = sum |bf16(ref) - ref| / sum |ref|        (~1.4e-3 on Gaussian V)

— below the north_star's 1e-3 example, so no bf16 kernel can reach it. Each
check therefore computes the floor of ITS OWN reference rows and gates on a
multiple of it, plus the north_star's absolute bound:

    max |gpu - ref|              <= MAX_ABS            (2e-2)
    sum |gpu - ref| / sum |ref|  <= FLOOR_MULT * floor + 1e-12     (FLOOR_MULT = 2)

FLOOR_MULT = 2.0: what the kernel adds on top of the output rounding is the
rounding of P to bf16 before P.V (relative 2^-9 per weight, averaging out over
the kept keys) and fp32 accumulation. Measured over all 543 GPU parity
comparisons of the final round-2 build (profiles/r02/tolerance_ratios.jsonl,
written with SHPLB_TOL_LOG; kernel 3 with the row-max skip): mean-rel / floor
median 1.52, p99 1.76, max 1.87 (a sampled C5 x 2 check) — against the
exact-max build's 1.49 / 1.71 / 1.83 over the same tests the per-comparison
change averages +0.003 (P against a stale running max rounds differently, not
worse) — so the gate sits 7% above the worst case, and an error that doubled
the kernel's own share over the floor on a typical comparison (1.52 -> 2.04)
would fail it.
"""
import json
import os

import numpy as np
import torch

MAX_ABS = 2e-2
FLOOR_MULT = float(os.environ.get("SHPLB_FLOOR_MULT_MEASURE", "2.0"))  # env override: measurement runs only


def bf16_floor(ref: np.ndarray) -> float:
    r = torch.from_numpy(np.ascontiguousarray(ref, dtype=np.float64)).to(torch.bfloat16).double().numpy()
    den = np.abs(ref).sum()
    return float(np.abs(r - ref).sum() / den) if den > 0 else 0.0


def output_errors(gpu, ref: np.ndarray):
    """(max-abs, mean-rel, floor) of bf16 GPU output (tensor or array) against fp64 ref."""
    if isinstance(gpu, torch.Tensor):
        gpu = gpu.float().cpu().numpy()
    g = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    diff = np.abs(g - ref)
    den = np.abs(ref).sum()
    rel = float(diff.sum() / den) if den > 0 else float(diff.sum())
    return float(diff.max()) if diff.size else 0.0, rel, bf16_floor(ref)


def check_output(gpu, ref: np.ndarray, what="") -> tuple:
    mx, rel, floor = output_errors(gpu, ref)
    log = os.environ.get("SHPLB_TOL_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps({"test": os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0],
                                "what": str(what), "max_abs": mx, "mean_rel": rel, "floor": floor,
                                "ratio": rel / floor if floor > 0 else None}) + "\n")
    assert mx <= MAX_ABS, f"{what}: max-abs {mx:.3e} > {MAX_ABS}"
    assert rel <= FLOOR_MULT * floor + 1e-12, (
        f"{what}: mean-rel {rel:.3e} > {FLOOR_MULT} x bf16 floor {floor:.3e} (ratio {rel / max(floor, 1e-300):.2f})")
    return mx, rel, floor
