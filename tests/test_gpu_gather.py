"""Fused head-parallel output gather (shplb_layer_shape.out_peers): kernel 3's
epilogue stores every output row into several full-layer buffers at the head's
global index. On one GPU the "peers" are distinct local buffers — the same
stores a rank issues to its peers' buffers over NVLink."""
import numpy as np
import pytest
import torch

import paper_2603_10353_b200 as P
from paper_2603_10353_b200.head_parallel import PeerOutputs, rank_segments, rank_shard
from paper_2603_10353_b200.workload import LayerSpec, make_layer

pytestmark = pytest.mark.gpu


def _layer(hq=8, hkv=2, n=1024, seed=3):
    q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=seed), "cuda")
    budgets = np.array([128, 384, 1024, 256, 640, 128, 896, 512][:hq], np.int64)
    return q, k, v, budgets


@pytest.mark.parametrize("bq", [256, 128])
def test_fused_gather_writes_every_buffer_at_global_heads(cuda_ctx, bq):
    q, k, v, budgets = _layer()
    hq, n, d = q.shape
    ref = cuda_ctx.sparse_attention_layer(q, k, v, budgets, block_q=bq)
    # this "rank" holds heads 5, 1, 6 of the layer (a greedy-style scattered shard)
    heads = [1, 5, 6]
    sh = rank_shard(np.array([1, 0, 1, 1, 1, 0, 0, 1]), 0, hq // k.shape[0], budgets)
    assert sh.heads == heads
    bufs = [torch.full((hq, n, d), 7.0, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    ql = q[heads].contiguous()
    kl, vl = k[sh.kv_heads].contiguous(), v[sh.kv_heads].contiguous()
    out = cuda_ctx.sparse_attention_layer(ql, kl, vl, sh.budgets, kv_map=sh.kv_map, block_q=bq,
                                          gather=([b.data_ptr() for b in bufs], heads, hq))
    torch.cuda.synchronize()
    assert out is None
    for b in bufs:
        assert torch.equal(b[heads], ref[heads])
        others = [h for h in range(hq) if h not in heads]
        assert bool((b[others] == 7.0).all()), "rows of other heads must be untouched"


def test_fused_gather_reassembles_a_split_plan(cuda_ctx):
    q, k, v, budgets = _layer(n=2000)
    hq, n, d = q.shape
    ref = cuda_ctx.sparse_attention_layer(q, k, v, budgets)
    plan = P.split_assign(budgets, 3, n)
    full = torch.zeros((hq, n, d), dtype=torch.bfloat16, device="cuda")
    group = hq // k.shape[0]
    for r in range(3):  # every rank writes its segments straight into the shared layout
        seg = rank_segments(plan, r, group, budgets)
        if not seg.heads:
            continue
        cuda_ctx.sparse_attention_layer(q[seg.heads].contiguous(), k[seg.kv_heads].contiguous(),
                                        v[seg.kv_heads].contiguous(), seg.budgets, kv_map=seg.kv_map,
                                        q_block_range=seg.q_block_range,
                                        gather=([full.data_ptr()], seg.heads, hq))
    torch.cuda.synchronize()
    assert torch.equal(full, ref)


def test_fused_gather_argument_errors(cuda_ctx):
    q, k, v, budgets = _layer(hq=2, hkv=1, n=256)
    buf = torch.zeros_like(q)
    with pytest.raises(P.InvalidArgument, match=r"output head 2 out of range \[0, 2\)"):
        cuda_ctx.sparse_attention_layer(q, k, v, budgets[:2], gather=([buf.data_ptr()], [0, 2], 2))
    with pytest.raises(P.NotSupported, match="at most 8 output buffers"):
        cuda_ctx.sparse_attention_layer(q, k, v, budgets[:2], gather=([buf.data_ptr()] * 9, [0, 1], 2))


def test_peer_outputs_single_rank(cuda_ctx):
    po = PeerOutputs(4, 512, 128, world=1, rank=0, device="cuda:0", sets=2)
    assert po.ptrs(0) == [po.local[0].data_ptr()] and po.ptrs(3) == [po.local[1].data_ptr()]
    po.close()
