"""TEST INFRASTRUCTURE ONLY — ctypes access to the parity oracle.

Two libraries, both built by ``oracle/Makefile``:

* ``oracle/build/liboracle.so`` — our plain-C restatement of the reference's
  sparse-attention algorithm at block granularity (``shplb_oracle.c``; every
  function cites the reference file:line it follows).
* ``oracle/_ref/libheadbal_ref.so`` — the UNMODIFIED reference library
  (``/root/reference/proj/src``) behind an extern "C" shim
  (``oracle/ref_shim.cpp``). Used to pin the restatement and, in bench.py, as
  the reference CPU arm.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` legs may import this module. The product package
(``paper_2603_10353_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libheadbal_ref.so")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")

_orc = None
_ref = None


def build() -> None:
    """Build the oracle (and the reference when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load_oracle():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.orc_pool_blocks.argtypes = [_u16p, C.c_int64, C.c_int32, C.c_int32, _f32p]
        L.orc_score_scale.argtypes = [C.c_int32]
        L.orc_score_scale.restype = C.c_float
        i64, i32 = C.c_int64, C.c_int32
        L.orc_visible_blocks.argtypes = [i64, i64, i64, i32, i32, C.c_int]
        L.orc_visible_blocks.restype = i64
        L.orc_block_scores.argtypes = [_f32p, _f32p, i64, i64, i32, i32, i32, C.c_int, _f32p]
        L.orc_score_rows.argtypes = [_f32p, _f32p, i64, i64, i32, _f32p]
        L.orc_select_topk.argtypes = [_f32p, i64, i64, i32, i32, C.c_int, i64, i64, _i32p, _i32p]
        L.orc_topk_row.argtypes = [_f64p, i64, i64, _i64p]
        L.orc_block_sparse_attention.argtypes = [_u16p, _u16p, _u16p, i64, i64, i32, i32, i32,
                                                 C.c_int, _i32p, _i32p, i64, _f64p]
        L.orc_det_ex2.argtypes = [C.c_float]
        L.orc_det_ex2.restype = C.c_float
        L.orc_colagg_select.argtypes = [_f32p, i64, i64, i32, i32, C.c_int, i64, i64, _i32p, _i32p]
        L.orc_layer_kind.argtypes = [_u16p, _u16p, _u16p, i32, i32, i64, i64, i32, i32, i32, C.c_int,
                                     C.c_int, _i64p, i64, _f32p, _i32p, _i32p, C.c_void_p]
        L.orc_layer.argtypes = [_u16p, _u16p, _u16p, i32, i32, i64, i64, i32, i32, i32, C.c_int,
                                _i64p, i64, _f32p, _i32p, _i32p, C.c_void_p]
        L.orc_recovery_at.argtypes = [_i64p, _f64p, C.c_int64, C.c_int64]
        L.orc_recovery_at.restype = C.c_double
        L.orc_uniform_allocate.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, _i64p]
        L.orc_maxmin_allocate.argtypes = [C.c_int32, C.c_int64, _i64p, _i64p, _f64p, C.c_int64,
                                          C.c_int64, C.c_int64, C.c_int64, _i64p,
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
        L.orc_naive_assign.argtypes = [C.c_int32, C.c_int32, C.c_int, _i32p]
        L.orc_greedy_assign.argtypes = [_i64p, C.c_int32, C.c_int32, _i32p]
        L.orc_imbalance.argtypes = [_i64p, C.c_int32, _i32p, C.c_int32, _i64p,
                                    C.POINTER(C.c_int32)]
        L.orc_imbalance.restype = C.c_double
        L.orc_barrier.argtypes = [_f64p, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _load_ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(
                f"{REF_SO} missing: build it here with `make -C oracle` (needs /root/reference)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        attn = [_f64p, _f64p, _f64p, C.c_int64, C.c_int64, C.c_int64, C.c_int64]
        L.ref_dense_attention.argtypes = attn + [C.c_int, C.c_void_p, _f64p]
        L.ref_sparse_attention.argtypes = attn + [C.c_int, C.c_int64, C.c_int, _f64p]
        L.ref_serial_sparse_attention.argtypes = attn + [C.c_int, C.c_int64, C.c_int, _f64p]
        L.ref_sparse_attention_timed.argtypes = attn + [C.c_int, C.c_int64, C.c_int, _f64p,
                                                        C.POINTER(C.c_double)]
        L.ref_recovery_ratio.argtypes = [_f64p, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                         C.POINTER(C.c_double)]
        L.ref_build_profiles.argtypes = [_f64p, _f64p, _f64p, C.c_int32, C.c_int64, C.c_int64,
                                         C.c_int64, _i64p, C.c_int64, C.c_int, C.c_int, _f64p]
        L.ref_uniform_allocate.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int64, _i64p]
        L.ref_maxmin_allocate.argtypes = [C.c_int32, C.c_int64, _i64p, _i64p, _f64p, C.c_int64,
                                          C.c_int64, C.c_int64, C.c_int64, _i64p,
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                          C.POINTER(C.c_int64)]
        L.ref_budget_for_recovery.argtypes = [C.c_int64, C.c_int64, _i64p, _f64p, C.c_double,
                                              C.POINTER(C.c_int64)]
        L.ref_stability_score.argtypes = [C.c_int32, C.c_int32, _i32p, _i32p, C.c_int64, _i64p, _i64p, _f64p,
                                          C.c_char_p, C.c_double, C.c_int, C.POINTER(C.c_double)]
        L.ref_naive_assign.argtypes = [_i64p, C.c_int32, C.c_int32, C.c_int, _i32p]
        L.ref_greedy_assign.argtypes = [_i64p, C.c_int32, C.c_int32, _i32p]
        L.ref_optimal_assign.argtypes = [_i64p, C.c_int32, C.c_int32, _i32p]
        L.ref_imbalance.argtypes = [_i64p, C.c_int32, _i32p, C.c_int32, _i64p,
                                    C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                    C.POINTER(C.c_int32)]
        L.ref_simulate.argtypes = [_i64p, C.c_int32, C.c_double, C.c_double, _f64p,
                                   C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_max_threads.restype = C.c_int
        cp, vp = C.c_char_p, C.c_void_p
        L.ref_save_allocation.argtypes = [cp, C.c_int32, _i32p, _i32p, _i64p, C.c_int64, C.c_int64]
        L.ref_load_allocation.argtypes = [cp, C.c_int32, _i32p, _i32p, _i64p, C.POINTER(C.c_int32),
                                          C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.ref_save_assignment.argtypes = [cp, C.c_int32, _i32p, _i32p, _i32p, C.c_int32, _i64p,
                                          C.c_double]
        L.ref_load_assignment.argtypes = [cp, C.c_int32, C.c_int32, _i32p, _i32p, _i32p,
                                          C.POINTER(C.c_int32), C.POINTER(C.c_int32), _i64p,
                                          C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        L.ref_save_profiles.argtypes = [cp, C.c_int32, _i32p, _i32p, C.c_int64, _i64p, _i64p,
                                        _f64p, C.c_int, cp, cp]
        L.ref_load_profiles.argtypes = [cp, C.c_int32, C.c_int64, _i32p, _i32p, _i64p, _i64p,
                                        _f64p, C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int), vp, vp, C.c_int64]
        _ref = L
    return _ref


class ReferenceError(Exception):
    """A C++ exception raised inside the reference library."""


def _ref_check(rc: int) -> None:
    if rc != 0:
        raise ReferenceError(_load_ref().ref_last_error().decode())


# --------------------------------------------------------------------------
# bf16 helpers (numpy has no bf16: we carry raw uint16 bit patterns)
# --------------------------------------------------------------------------

def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (what torch's .bfloat16() does)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + rounding) >> 16).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# --------------------------------------------------------------------------
# Block-level restatement
# --------------------------------------------------------------------------

def nblocks(n: int, b: int) -> int:
    return (n + b - 1) // b


def pool_blocks(x_bits: np.ndarray, block: int) -> np.ndarray:
    x_bits = np.ascontiguousarray(x_bits, dtype=np.uint16)
    n, d = x_bits.shape
    out = np.empty((nblocks(n, block), d), np.float32)
    _load_oracle().orc_pool_blocks(x_bits, n, d, block, out)
    return out


def score_scale(d: int) -> float:
    return float(_load_oracle().orc_score_scale(d))


def visible_blocks(qb: int, n: int, bq: int, bk: int, causal: bool, n_k: int = None) -> int:
    """Key blocks visible to query block qb (n query rows, n_k keys, default n_k = n)."""
    return int(_load_oracle().orc_visible_blocks(qb, n, n if n_k is None else n_k, bq, bk,
                                                 int(causal)))


def block_scores(qp: np.ndarray, kp: np.ndarray, n: int, bq: int, bk: int,
                 causal: bool, n_k: int = None) -> np.ndarray:
    d = qp.shape[1]
    n_k = n if n_k is None else n_k
    out = np.empty((nblocks(n, bq), nblocks(n_k, bk)), np.float32)
    _load_oracle().orc_block_scores(np.ascontiguousarray(qp, np.float32),
                                    np.ascontiguousarray(kp, np.float32), n, n_k, d, bq, bk,
                                    int(causal), out)
    return out


def select_topk(scores: np.ndarray, n: int, bq: int, bk: int, causal: bool, k_blocks: int,
                kmax: int, n_k: int = None):
    nqb = nblocks(n, bq)
    idx = np.empty((nqb, kmax), np.int32)
    cnt = np.empty(nqb, np.int32)
    _load_oracle().orc_select_topk(np.ascontiguousarray(scores, np.float32), n,
                                   n if n_k is None else n_k, bq, bk, int(causal), k_blocks,
                                   kmax, idx, cnt)
    return idx, cnt


def colagg_select(scores: np.ndarray, n: int, bq: int, bk: int, causal: bool, k_blocks: int,
                  kmax: int, n_k: int = None):
    """Block-level ColumnAggregateTopK for one head (see orc_colagg_select)."""
    nqb = nblocks(n, bq)
    idx = np.empty((nqb, kmax), np.int32)
    cnt = np.empty(nqb, np.int32)
    _load_oracle().orc_colagg_select(np.ascontiguousarray(scores, np.float32), n,
                                     n if n_k is None else n_k, bq, bk, int(causal), k_blocks,
                                     kmax, idx, cnt)
    return idx, cnt


def det_ex2(x: float) -> float:
    return float(_load_oracle().orc_det_ex2(x))


def topk_row(values: np.ndarray, k: int) -> np.ndarray:
    values = np.ascontiguousarray(values, np.float64)
    out = np.empty(k, np.int64)
    _load_oracle().orc_topk_row(values, values.size, k, out)
    return out


def layer(q_bits, k_bits, v_bits, k_blocks, *, bq=128, bk=128, causal=True, kmax=None,
          with_output=True, kind=0):
    """Whole layer: pooled scores, selections and fp64 outputs for every q head.

    q_bits [Hq, n_q, d], k_bits/v_bits [Hkv, n_k, d] (bf16 bit patterns);
    k_blocks [Hq] per-head budgets in blocks.
    """
    q_bits = np.ascontiguousarray(q_bits, np.uint16)
    k_bits = np.ascontiguousarray(k_bits, np.uint16)
    v_bits = np.ascontiguousarray(v_bits, np.uint16)
    hq, n, d = q_bits.shape
    hkv, n_k = k_bits.shape[0], k_bits.shape[1]
    nqb, nkb = nblocks(n, bq), nblocks(n_k, bk)
    k_blocks = np.ascontiguousarray(k_blocks, np.int64)
    if kmax is None:
        kmax = int(min(nkb, k_blocks.max()))
    scores = np.empty((hq, nqb, nkb), np.float32)
    idx = np.empty((hq, nqb, kmax), np.int32)
    cnt = np.empty((hq, nqb), np.int32)
    out = np.empty((hq, n, d), np.float64) if with_output else None
    _load_oracle().orc_layer_kind(q_bits, k_bits, v_bits, hq, hkv, n, n_k, d, bq, bk, int(causal),
                                  int(kind), k_blocks, kmax, scores, idx, cnt,
                                  out.ctypes.data if with_output else None)
    return scores, idx, cnt, out


def sparse_rows(q_bits_h, k_bits_g, v_bits_g, rows, sel_blocks, *, bq=128, bk=128, causal=True):
    """fp64 outputs of selected query rows of one head (numpy restatement of
    orc_block_sparse_attention for row subsets at full sequence length).

    rows: query indices (all in one query block); sel_blocks: that block's
    selected key blocks. Follows attention.cpp:35-49 on the kept tokens.
    """
    n, d = k_bits_g.shape
    toks = np.concatenate([np.arange(b * bk, min(n, (b + 1) * bk)) for b in sorted(sel_blocks)])
    K = bf16_bits_to_f32(k_bits_g[toks]).astype(np.float64)
    V = bf16_bits_to_f32(v_bits_g[toks]).astype(np.float64)
    scale = 1.0 / np.sqrt(d)
    out = np.zeros((len(rows), d), np.float64)
    for r, i in enumerate(rows):
        q = bf16_bits_to_f32(q_bits_h[i]).astype(np.float64)
        keep = toks <= i if causal else np.ones_like(toks, bool)
        if not keep.any():
            continue
        s = (K[keep] @ q) * scale
        w = np.exp(s - s.max())
        out[r] = (w / w.sum()) @ V[keep]
    return out


def pooled_scores_rows(q_bits_h, kp, qbs, *, bq=128, bk=128, causal=True):
    """Block scores of the query blocks `qbs` of one head against the pooled
    keys `kp` [nkb][d] of its kv head (C restatement, bit-exact with kernel 1)."""
    n = q_bits_h.shape[0]
    rows = []
    for qb in qbs:
        rows.append(pool_blocks(q_bits_h[qb * bq:min(n, (qb + 1) * bq)], bq)[0])
    qp = np.ascontiguousarray(np.stack(rows), np.float32)
    nkb, d = kp.shape
    out = np.empty((len(qbs), nkb), np.float32)
    _load_oracle().orc_score_rows(qp, np.ascontiguousarray(kp, np.float32), len(qbs), nkb, d, out)
    for r, qb in enumerate(qbs):
        out[r, visible_blocks(qb, n, bq, bk, causal):] = -np.inf
    return out


# --------------------------------------------------------------------------
# Budget table / plan / metric restatement
# --------------------------------------------------------------------------

def block_selection_profile(q_bits, k_bits, rows, grid, *, bq=128, causal=True):
    """Recovery curves of the block selector (restates shplb_profile_curves_block):
    per q head h and calibration row at position p, the kept blocks at budget b
    are the ceil(b/128) best of the row's query block under kernel 2's rule
    (pooled fp32 scores from the C restatement, (score desc, index asc), visible
    blocks only); recovery = the row's exact fp64 softmax mass over keys j <= p
    (causal) inside them (recovery_ratio's kept-set mass, attention.cpp:151-184),
    averaged over rows (build_profiles, profiler.cpp:157-196).

    q_bits [Hq, n, d], k_bits [Hkv, n, d] bf16 bit patterns -> [Hq, len(grid)]."""
    q_bits = np.ascontiguousarray(q_bits, np.uint16)
    k_bits = np.ascontiguousarray(k_bits, np.uint16)
    hq, n, d = q_bits.shape
    hkv = k_bits.shape[0]
    group = hq // hkv
    nkb = nblocks(n, 128)
    grid = np.asarray(grid, np.int64)
    rows = np.asarray(rows, np.int64)
    out = np.zeros((hq, grid.size))
    for g in range(hkv):
        K = bf16_bits_to_f32(k_bits[g]).astype(np.float64)
        kp = pool_blocks(k_bits[g], 128)
        for h in range(g * group, (g + 1) * group):
            bs = block_scores(pool_blocks(q_bits[h], bq), kp, n, bq, 128, causal)
            Q = bf16_bits_to_f32(q_bits[h][rows]).astype(np.float64)
            S = (Q @ K.T) * (1.0 / np.sqrt(d))
            for r, p in enumerate(rows):
                end = p + 1 if causal else n
                s = S[r, :end]
                w = np.exp(s - s.max())
                mass = np.zeros(nkb)
                np.add.at(mass, np.arange(end) // 128, w)
                mass /= w.sum()
                qb = p // bq
                vis = visible_blocks(qb, n, bq, 128, causal)
                sc = bs[qb, :vis].astype(np.float32)
                sc = np.where(sc == 0, np.float32(0), sc)  # -0.0 ties with +0.0
                order = np.lexsort((np.arange(vis), -sc.astype(np.float64)))
                cum = np.concatenate([[0.0], np.cumsum(mass[order])])
                kb = np.minimum((grid + 127) // 128, vis)
                out[h] += np.minimum(cum[kb], 1.0)
    return out / rows.size


def _flatten_curves(curves):
    offsets = np.zeros(len(curves) + 1, np.int64)
    for h, (b, _) in enumerate(curves):
        offsets[h + 1] = offsets[h] + len(b)
    pb = np.concatenate([np.asarray(b, np.int64) for b, _ in curves])
    pr = np.concatenate([np.asarray(r, np.float64) for _, r in curves])
    return offsets, pb, pr


def uniform_allocate(n, total, floor, n_k):
    out = np.empty(n, np.int64)
    if _load_oracle().orc_uniform_allocate(n, total, floor, n_k, out):
        raise ValueError("infeasible total")
    return out


def maxmin_allocate(curves, n_k, total, quantum=64, floor=128, max_iterations=0):
    """curves: list of (budgets, recoveries) per head."""
    offsets, pb, pr = _flatten_curves(curves)
    out = np.empty(len(curves), np.int64)
    tr = C.c_int64()
    cap = C.c_int32()
    if _load_oracle().orc_maxmin_allocate(len(curves), n_k, offsets, pb, pr, total, quantum,
                                          floor, max_iterations, out, C.byref(tr), C.byref(cap)):
        raise ValueError("infeasible total")
    return out, int(tr.value), bool(cap.value)


def naive_assign(n, devices, round_robin=False):
    out = np.empty(n, np.int32)
    if _load_oracle().orc_naive_assign(n, devices, int(round_robin), out):
        raise ValueError("bad device count")
    return out


def greedy_assign(budgets, devices):
    budgets = np.ascontiguousarray(budgets, np.int64)
    out = np.empty(budgets.size, np.int32)
    _load_oracle().orc_greedy_assign(budgets, budgets.size, devices, out)
    return out


def imbalance(budgets, dev, devices):
    budgets = np.ascontiguousarray(budgets, np.int64)
    loads = np.empty(devices, np.int64)
    am = C.c_int32()
    imb = _load_oracle().orc_imbalance(budgets, budgets.size,
                                       np.ascontiguousarray(dev, np.int32), devices, loads,
                                       C.byref(am))
    return loads, float(imb), int(am.value)


def barrier(latencies):
    lat = np.ascontiguousarray(latencies, np.float64)
    b, bub = C.c_double(), C.c_double()
    _load_oracle().orc_barrier(lat, lat.size, C.byref(b), C.byref(bub))
    return float(b.value), float(bub.value)


# --------------------------------------------------------------------------
# The reference itself (oracle/_ref)
# --------------------------------------------------------------------------

class ref:
    """Thin wrappers over the compiled, unmodified reference library."""

    @staticmethod
    def dense_attention(Q, K, V, causal=False, with_weights=False):
        Q, K, V = (np.ascontiguousarray(a, np.float64) for a in (Q, K, V))
        out = np.empty((Q.shape[0], V.shape[1]), np.float64)
        w = np.empty((Q.shape[0], K.shape[0]), np.float64) if with_weights else None
        _ref_check(_load_ref().ref_dense_attention(
            Q, K, V, Q.shape[0], K.shape[0], Q.shape[1], V.shape[1], int(causal),
            w.ctypes.data if with_weights else None, out))
        return (w, out) if with_weights else out

    @staticmethod
    def sparse_attention(Q, K, V, budget, causal=False, kind=0, serial=False):
        Q, K, V = (np.ascontiguousarray(a, np.float64) for a in (Q, K, V))
        out = np.empty((Q.shape[0], V.shape[1]), np.float64)
        fn = _load_ref().ref_serial_sparse_attention if serial else _load_ref().ref_sparse_attention
        _ref_check(fn(Q, K, V, Q.shape[0], K.shape[0], Q.shape[1], V.shape[1], kind, budget,
                      int(causal), out))
        return out

    @staticmethod
    def sparse_attention_timed(Q, K, V, budget, causal=False, kind=0):
        """(output, seconds spent inside headbal::sparse_attention)."""
        Q, K, V = (np.ascontiguousarray(a, np.float64) for a in (Q, K, V))
        out = np.empty((Q.shape[0], V.shape[1]), np.float64)
        sec = C.c_double()
        _ref_check(_load_ref().ref_sparse_attention_timed(
            Q, K, V, Q.shape[0], K.shape[0], Q.shape[1], V.shape[1], kind, budget, int(causal),
            out, C.byref(sec)))
        return out, float(sec.value)

    @staticmethod
    def build_profiles(Q, K, V, grid, causal=False, kind=0):
        """Q/K/V [H, n, d] fp64 -> recovery [H, len(grid)]."""
        Q, K, V = (np.ascontiguousarray(a, np.float64) for a in (Q, K, V))
        grid = np.ascontiguousarray(grid, np.int64)
        h, n_q, d = Q.shape
        out = np.empty((h, grid.size), np.float64)
        _ref_check(_load_ref().ref_build_profiles(Q, K, V, h, n_q, K.shape[1], d, grid, grid.size,
                                                  kind, int(causal), out))
        return out

    @staticmethod
    def stability_score(groups, p, norm="max"):
        """groups: [(request name, [(layer, head)], [curve])] with curves having
        .budgets / .recovery and one shared context length."""
        n_groups, n_heads = len(groups), len(groups[0][1])
        layers = np.array([lh[0] for _, ids, _ in groups for lh in ids], np.int32)
        heads = np.array([lh[1] for _, ids, _ in groups for lh in ids], np.int32)
        curves = [c for _, _, cs in groups for c in cs]
        offsets = np.zeros(len(curves) + 1, np.int64)
        for i, c in enumerate(curves):
            offsets[i + 1] = offsets[i] + len(c.budgets)
        b = np.ascontiguousarray(np.concatenate([np.asarray(c.budgets, np.int64) for c in curves]))
        r = np.ascontiguousarray(np.concatenate([np.asarray(c.recovery, np.float64) for c in curves]))
        names = b"".join(name.encode().ljust(64, b"\0")[:64] for name, _, _ in groups)
        out = C.c_double()
        _ref_check(_load_ref().ref_stability_score(n_groups, n_heads, layers, heads, int(curves[0].context_length),
                                                   offsets, b, r, names, float(p), 0 if norm == "max" else 1,
                                                   C.byref(out)))
        return float(out.value)

    @staticmethod
    def uniform_allocate(n, total, floor, n_k):
        out = np.empty(n, np.int64)
        _ref_check(_load_ref().ref_uniform_allocate(n, total, floor, n_k, out))
        return out

    @staticmethod
    def maxmin_allocate(curves, n_k, total, quantum=64, floor=128, max_iterations=0):
        offsets, pb, pr = _flatten_curves(curves)
        out = np.empty(len(curves), np.int64)
        tr, cap, off = C.c_int64(), C.c_int32(), C.c_int64()
        _ref_check(_load_ref().ref_maxmin_allocate(len(curves), n_k, offsets, pb, pr, total,
                                                   quantum, floor, max_iterations, out,
                                                   C.byref(tr), C.byref(cap), C.byref(off)))
        return out, int(tr.value), bool(cap.value)

    @staticmethod
    def naive_assign(budgets, devices, round_robin=False):
        budgets = np.ascontiguousarray(budgets, np.int64)
        out = np.empty(budgets.size, np.int32)
        _ref_check(_load_ref().ref_naive_assign(budgets, budgets.size, devices, int(round_robin),
                                                out))
        return out

    @staticmethod
    def greedy_assign(budgets, devices):
        budgets = np.ascontiguousarray(budgets, np.int64)
        out = np.empty(budgets.size, np.int32)
        _ref_check(_load_ref().ref_greedy_assign(budgets, budgets.size, devices, out))
        return out

    @staticmethod
    def optimal_assign(budgets, devices):
        budgets = np.ascontiguousarray(budgets, np.int64)
        out = np.empty(budgets.size, np.int32)
        _ref_check(_load_ref().ref_optimal_assign(budgets, budgets.size, devices, out))
        return out

    @staticmethod
    def imbalance(budgets, dev, devices):
        budgets = np.ascontiguousarray(budgets, np.int64)
        loads = np.empty(devices, np.int64)
        tot, imb, am = C.c_int64(), C.c_double(), C.c_int32()
        _ref_check(_load_ref().ref_imbalance(budgets, budgets.size,
                                             np.ascontiguousarray(dev, np.int32), devices, loads,
                                             C.byref(tot), C.byref(imb), C.byref(am)))
        return loads, float(imb.value), int(am.value)

    @staticmethod
    def simulate(loads, alpha=0.0, beta=1.0):
        loads = np.ascontiguousarray(loads, np.int64)
        lat = np.empty(loads.size, np.float64)
        b, bub = C.c_double(), C.c_double()
        _ref_check(_load_ref().ref_simulate(loads, loads.size, alpha, beta, lat, C.byref(b),
                                            C.byref(bub)))
        return lat, float(b.value), float(bub.value)

    # -- file formats (allocator.cpp:223-275, partitioner.cpp:268-336,
    #    profiler.cpp:300-383) ------------------------------------------------
    @staticmethod
    def save_allocation(path, budgets, total, floor, heads=None):
        budgets = np.ascontiguousarray(budgets, np.int64)
        n = budgets.size
        hl = np.asarray(heads if heads is not None else [(0, h) for h in range(n)], np.int32).reshape(n, 2)
        _ref_check(_load_ref().ref_save_allocation(str(path).encode(), n, np.ascontiguousarray(hl[:, 0]),
                                                   np.ascontiguousarray(hl[:, 1]), budgets, total, floor))

    @staticmethod
    def load_allocation(path, max_n=4096):
        lay, hd = np.empty(max_n, np.int32), np.empty(max_n, np.int32)
        b = np.empty(max_n, np.int64)
        n, tot, fl = C.c_int32(), C.c_int64(), C.c_int64()
        _ref_check(_load_ref().ref_load_allocation(str(path).encode(), max_n, lay, hd, b, C.byref(n),
                                                   C.byref(tot), C.byref(fl)))
        k = n.value
        return b[:k].copy(), list(zip(lay[:k].tolist(), hd[:k].tolist())), int(tot.value), int(fl.value)

    @staticmethod
    def save_assignment(path, device_of_head, devices, loads, imbalance, heads=None):
        dev = np.ascontiguousarray(device_of_head, np.int32)
        n = dev.size
        hl = np.asarray(heads if heads is not None else [(0, h) for h in range(n)], np.int32).reshape(n, 2)
        _ref_check(_load_ref().ref_save_assignment(str(path).encode(), n, np.ascontiguousarray(hl[:, 0]),
                                                   np.ascontiguousarray(hl[:, 1]), dev, devices,
                                                   np.ascontiguousarray(loads, np.int64), float(imbalance)))

    @staticmethod
    def load_assignment(path, max_n=4096, max_devices=1024):
        lay, hd, dev = (np.empty(max_n, np.int32) for _ in range(3))
        loads = np.empty(max_devices, np.int64)
        n, nd, tot, imb = C.c_int32(), C.c_int32(), C.c_int64(), C.c_double()
        _ref_check(_load_ref().ref_load_assignment(str(path).encode(), max_n, max_devices, lay, hd, dev,
                                                   C.byref(n), C.byref(nd), loads, C.byref(tot), C.byref(imb)))
        k = n.value
        return (dev[:k].copy(), list(zip(lay[:k].tolist(), hd[:k].tolist())), int(nd.value),
                loads[:nd.value].copy(), int(tot.value), float(imb.value))

    @staticmethod
    def save_profiles(path, budgets_list, recovery_list, context_length, heads=None, kind=0,
                      request="calibration", task="synthetic"):
        n = len(budgets_list)
        offsets = np.zeros(n + 1, np.int64)
        offsets[1:] = np.cumsum([len(b) for b in budgets_list])
        pb = np.ascontiguousarray(np.concatenate([np.asarray(b, np.int64) for b in budgets_list]))
        pr = np.ascontiguousarray(np.concatenate([np.asarray(r, np.float64) for r in recovery_list]))
        hl = np.asarray(heads if heads is not None else [(0, h) for h in range(n)], np.int32).reshape(n, 2)
        _ref_check(_load_ref().ref_save_profiles(str(path).encode(), n, np.ascontiguousarray(hl[:, 0]),
                                                 np.ascontiguousarray(hl[:, 1]), context_length, offsets, pb,
                                                 pr, kind, request.encode(), task.encode()))

    @staticmethod
    def load_profiles(path, max_heads=1024, max_points=1 << 22):
        lay, hd = np.empty(max_heads, np.int32), np.empty(max_heads, np.int32)
        off = np.zeros(max_heads + 1, np.int64)
        pb, pr = np.empty(max_points, np.int64), np.empty(max_points, np.float64)
        n, ctxl, kind = C.c_int32(), C.c_int64(), C.c_int()
        req, task = C.create_string_buffer(1024), C.create_string_buffer(1024)
        _ref_check(_load_ref().ref_load_profiles(str(path).encode(), max_heads, max_points, lay, hd, off, pb,
                                                 pr, C.byref(n), C.byref(ctxl), C.byref(kind), req, task, 1024))
        k = n.value
        curves = [(pb[off[h]:off[h + 1]].copy(), pr[off[h]:off[h + 1]].copy()) for h in range(k)]
        return (curves, list(zip(lay[:k].tolist(), hd[:k].tolist())), int(ctxl.value), int(kind.value),
                req.value.decode(), task.value.decode())

    @staticmethod
    def max_threads() -> int:
        return int(_load_ref().ref_max_threads())
