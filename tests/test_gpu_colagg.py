"""GPU parity for SHPLB_COLUMN_AGGREGATE_TOPK (ColumnAggregateTopK at block
granularity, attention.cpp:136-148): kept sets and per-block counts BIT-EXACT
with orc_colagg_select (same fp32 ops in the same order, det_ex2 instead of
MUFU), outputs within the kernel-3 tolerance of tests/test_gpu_parity.py.
"""
import numpy as np
import pytest
import torch

import paper_2603_10353_b200 as P
from oracle import oracle as O
from paper_2603_10353_b200.workload import LayerSpec, bf16_bits, make_layer
from test_gpu_parity import _scores_equal
from tolerance import check_output

pytestmark = pytest.mark.gpu

KIND = P.COLUMN_AGGREGATE_TOPK


def run_case(ctx, spec, k_blocks, causal=True, bq=256, with_output=True):
    q, k, v = make_layer(spec, "cpu")
    qb, kb, vb = bf16_bits(q), bf16_bits(k), bf16_bits(v)
    k_blocks = np.asarray(k_blocks, np.int64)
    nkb = (spec.seq_len + 127) // 128
    kmax = int(min(nkb, k_blocks.max()))
    sc_o, idx_o, cnt_o, out_o = O.layer(qb, kb, vb, k_blocks, bq=bq, causal=causal, kmax=kmax,
                                        kind=1, with_output=with_output)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()

    sc = ctx.block_scores(qd, kd, causal=causal, block_q=bq)
    idx, cnt = ctx.select_blocks(sc, k_blocks, spec.seq_len, causal=causal, kmax=kmax, block_q=bq,
                                 kind=KIND)
    torch.cuda.synchronize()
    assert _scores_equal(sc.cpu().numpy(), sc_o)
    assert np.array_equal(cnt.cpu().numpy(), cnt_o), "column-aggregate counts differ"
    assert np.array_equal(idx.cpu().numpy(), idx_o), "column-aggregate kept sets differ"

    budgets = np.minimum(k_blocks * 128, spec.seq_len)
    out = ctx.sparse_attention_layer(qd, kd, vd, budgets, causal=causal, block_q=bq, kind=KIND)
    torch.cuda.synchronize()
    idx2, cnt2 = ctx.last_selection(spec.num_q_heads, spec.seq_len)
    assert np.array_equal(cnt2.cpu().numpy(), cnt_o)
    assert np.array_equal(idx2.cpu().numpy(), idx_o), "layer-call selection differs"
    out_k = ctx.block_sparse_attention(qd, kd, vd, idx, cnt, causal=causal, block_q=bq)
    torch.cuda.synchronize()
    assert torch.equal(out, out_k), "layer call differs from kernel-by-kernel path"
    if with_output:
        check_output(out, out_o, "column aggregate")
    return out, cnt_o


@pytest.mark.parametrize("bq", [256, 128])
@pytest.mark.parametrize("causal", [True, False])
def test_small_gqa_layer(cuda_ctx, causal, bq):
    run_case(cuda_ctx, LayerSpec(num_q_heads=4, num_kv_heads=2, seq_len=1024, seed=1),
             [1, 3, 8, 5], causal=causal, bq=bq)


@pytest.mark.parametrize("bq", [256, 128])
@pytest.mark.parametrize("n", [1, 100, 129, 300, 1000, 1536])
def test_ragged_lengths(cuda_ctx, n, bq):
    spec = LayerSpec(num_q_heads=2, num_kv_heads=1, seq_len=n, seed=70 + n)
    nkb = (n + 127) // 128
    run_case(cuda_ctx, spec, [1, max(1, nkb // 2 + 1)], causal=True, bq=bq)
    run_case(cuda_ctx, spec, [nkb, 1], causal=False, bq=bq)


def test_empty_query_blocks_give_zero_rows(cuda_ctx):
    """A query block that sees none of its head's kept blocks outputs zeros
    (attention.cpp:40-41 all-masked rows)."""
    spec = LayerSpec(num_q_heads=2, num_kv_heads=1, seq_len=2048, seed=12, targets="per_head",
                     hot_max=2)
    out, cnt = run_case(cuda_ctx, spec, [1, 2], causal=True, bq=128)
    o = out.float().cpu()
    for h in range(2):
        for qb in np.nonzero(cnt[h] == 0)[0]:
            assert torch.count_nonzero(o[h, qb * 128:(qb + 1) * 128]) == 0


def test_full_budget_equals_per_query(cuda_ctx):
    """k = every block: both policies keep every visible block."""
    spec = LayerSpec(num_q_heads=2, num_kv_heads=1, seq_len=640, seed=13)
    q, k, v = (t.cuda() for t in make_layer(spec, "cpu"))
    a = cuda_ctx.sparse_attention_layer(q, k, v, [640, 640], kind=P.BLOCK_TOPK)
    b = cuda_ctx.sparse_attention_layer(q, k, v, [640, 640], kind="column_aggregate_topk")
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_unknown_policy_name():
    with pytest.raises(P.InvalidArgument, match="unknown selection policy"):
        P.selection_kind("sliding_window")


def test_bad_kind_rejected(cuda_ctx):
    spec = LayerSpec(num_q_heads=2, num_kv_heads=1, seq_len=256, seed=1)
    q, k, v = (t.cuda() for t in make_layer(spec, "cpu"))
    with pytest.raises(P.NotSupported, match="selection kind"):
        cuda_ctx.sparse_attention_layer(q, k, v, [128, 128], kind=7)


def test_host_entry_kind(cuda_ctx):
    spec = LayerSpec(num_q_heads=4, num_kv_heads=2, seq_len=1024, seed=21)
    q, k, v = make_layer(spec, "cpu")
    b = [256, 512, 128, 1024]
    dev = cuda_ctx.sparse_attention_layer(q.cuda(), k.cuda(), v.cuda(), b, kind=KIND)
    host = cuda_ctx.sparse_attention_layer_host(q.pin_memory(), k.pin_memory(), v.pin_memory(), b,
                                                kind=KIND)
    torch.cuda.synchronize()
    assert torch.equal(dev.cpu(), host)


def test_selection_at_32k(cuda_ctx):
    """At 32K x 8 heads the kept sets stay bit-exact (scores + selection only)."""
    spec = LayerSpec(num_q_heads=8, num_kv_heads=2, seq_len=32768, seed=31)
    run_case(cuda_ctx, spec, [8, 16, 32, 64, 128, 5, 1, 256], causal=True, bq=256, with_output=False)
