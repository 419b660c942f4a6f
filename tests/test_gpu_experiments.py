"""Dense comparator (shplb_dense_attention_layer) and the measured sweep /
skyline drivers."""
import io

import numpy as np
import pytest
import torch
from tolerance import check_output

import paper_2603_10353_b200 as P
from oracle import oracle as O
from paper_2603_10353_b200 import experiments as X
from paper_2603_10353_b200.workload import LayerSpec, bf16_bits, make_layer

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,causal,bq", [(1024, True, 256), (777, True, 128), (640, False, 256)])
def test_dense_layer_equals_full_budget_sparse_and_oracle(cuda_ctx, n, causal, bq):
    spec = LayerSpec(num_q_heads=4, num_kv_heads=2, seq_len=n, seed=21)
    q, k, v = make_layer(spec, "cpu")
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    dense = cuda_ctx.dense_attention_layer(qd, kd, vd, causal=causal, block_q=bq)
    full = cuda_ctx.sparse_attention_layer(qd, kd, vd, np.full(4, n, np.int64), causal=causal, block_q=bq)
    torch.cuda.synchronize()
    assert torch.equal(dense, full), "dense comparator differs from the all-blocks sparse layer"
    nkb = (n + 127) // 128
    _, _, _, ref = O.layer(bf16_bits(q), bf16_bits(k), bf16_bits(v), np.full(4, nkb, np.int64), bq=bq,
                           causal=causal, kmax=nkb)
    check_output(dense, ref, "dense comparator")


def test_measured_sweep_and_skyline_small(cuda_ctx):
    spec = LayerSpec(num_q_heads=8, num_kv_heads=2, seq_len=2048, seed=5)
    q, k, v = make_layer(spec, "cuda")
    n = spec.seq_len
    curves = cuda_ctx.profile_curves(q[:, n - 16:, :].contiguous(), k, P.default_budget_grid(n, 128))
    budgets = P.maxmin_allocate(curves, int(0.25 * 8 * n), quantum=128, floor=128).budgets
    rows = X.measured_sweep(cuda_ctx, {n: (q, k, v, budgets)}, [1, 2], steps=1)
    plans = ["naive", "greedy", "greedy_tiles", "greedy_refined", "split"]
    assert [(r.degree, r.assigner) for r in rows] == [(d, a) for d in (1, 2) for a in plans]
    for r in rows:
        assert r.barrier_latency > 0 and 0.0 <= r.bubble_fraction < 1.0
        assert r.barrier_latency == pytest.approx(max(r.per_rank_ms))
    buf = io.StringIO()
    X.write_sweep_csv(buf, rows)
    assert buf.getvalue().splitlines()[0] == ("degree,context_length,allocator,assigner,barrier_latency,"
                                              "bubble_fraction,imbalance,speedup_vs_naive")
    pts = X.measured_skyline(cuda_ctx, q, k, v, curves, devices=2, steps=1)
    assert [(p.allocator) for p in pts] == ["uniform", "maxmin"] * 4
    full = [p for p in pts if p.total_budget == 8 * n]
    # all keys kept: the sparse layer is the dense one -> zero error (attention.cpp:186-202)
    assert all(p.mean_output_error == 0.0 for p in full)
    # more budget never hurts: error falls monotonically with the total, per allocator
    for kind in ("uniform", "maxmin"):
        e = [p.mean_output_error for p in pts if p.allocator == kind]
        assert all(a >= b for a, b in zip(e, e[1:])), (kind, e)
    with pytest.raises(P.InvalidArgument, match="infeasible"):
        X.measured_skyline(cuda_ctx, q, k, v, curves, devices=2, totals=[10])
    # ColumnAggregateTopK skyline (run_skyline's policy): its own curves, full budget exact,
    # and on this (seeded) workload one shared key set per head is no more accurate than
    # per-query block selection at the same uniform budgets
    ca_curves = cuda_ctx.profile_curves(q[:, n - 16:, :].contiguous(), k, P.default_budget_grid(n, 128),
                                        kind="column_aggregate_topk")
    ca = X.measured_skyline(cuda_ctx, q, k, v, ca_curves, devices=2, steps=1, policy="column_aggregate_topk")
    assert all(p.mean_output_error == 0.0 for p in ca if p.total_budget == 8 * n)
    pq_uniform = [p.mean_output_error for p in pts if p.allocator == "uniform"]
    ca_uniform = [p.mean_output_error for p in ca if p.allocator == "uniform"]
    assert all(c >= q_ - 1e-6 for c, q_ in zip(ca_uniform, pq_uniform))


def test_measured_top_p(cuda_ctx):
    """The offline top-p comparison: budgets from each head's
    curve; a larger p never lowers any head's budget or raises the error, and
    the greedy balancer is never worse than even head parallelism on them."""
    spec = LayerSpec(num_q_heads=8, num_kv_heads=2, seq_len=2048, seed=5)
    q, k, v = make_layer(spec, "cuda")
    n = spec.seq_len
    curves = cuda_ctx.profile_curves(q[:, n - 16:, :].contiguous(), k, P.default_budget_grid(n, 128))
    pts = X.measured_top_p(cuda_ctx, q, k, v, curves, devices=2, ps=(0.5, 0.9, 1.0), steps=1)
    assert [p.p for p in pts] == [0.5, 0.9, 1.0]
    assert pts[-1].total_budget == 8 * n and pts[-1].mean_output_error == 0.0  # p = 1 keeps everything
    for a, b in zip(pts, pts[1:]):
        assert a.total_budget <= b.total_budget and a.mean_output_error >= b.mean_output_error - 1e-9
    b5, b9 = P.top_p_budgets(curves, 0.5), P.top_p_budgets(curves, 0.9)
    assert np.all(b5 <= b9)
    for p in pts:  # shards of ~0.06 ms: 5% + 20 us of timing noise
        assert p.greedy_barrier_latency <= p.naive_barrier_latency * 1.05 + 0.02
