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


def test_ipc_handle_carries_offset_inside_allocation(cuda_ctx):
    import ctypes as C

    from paper_2603_10353_b200._native import check, lib
    big = torch.empty(1 << 20, dtype=torch.bfloat16, device="cuda")
    sub = big[4096:]
    offs = []
    for t in (big, sub):
        h = (C.c_char * 72)()
        check(lib().shplb_ipc_handle(C.c_void_p(t.data_ptr()), h, 72))
        offs.append(int.from_bytes(bytes(h)[64:72], "little"))
    assert offs[1] - offs[0] == 4096 * 2


def _two_rank_worker(rank, port, result):
    import os

    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        torch.cuda.set_device(0)
        ctx = P.Context(0)
        q, k, v, budgets = _layer(n=1500)
        hq = q.shape[0]
        ref = ctx.sparse_attention_layer(q, k, v, budgets)
        po = PeerOutputs(hq, q.shape[1], q.shape[2], world=2, rank=rank, device="cuda:0", sets=2)
        for b, plan in enumerate((P.greedy_assign(budgets, 2), P.split_assign(budgets, 2, q.shape[1]))):
            group = hq // k.shape[0]
            if b == 0:
                sh = rank_shard(plan, rank, group, budgets)
                rng = None
            else:
                sh = rank_segments(plan, rank, group, budgets)
                rng = sh.q_block_range
            if sh.heads:
                ctx.sparse_attention_layer(q[sh.heads].contiguous(), k[sh.kv_heads].contiguous(),
                                           v[sh.kv_heads].contiguous(), sh.budgets, kv_map=sh.kv_map,
                                           q_block_range=rng, gather=(po.ptrs(b), sh.heads, hq))
            torch.cuda.synchronize()
            dist.barrier()
            result[2 * rank + b] = int(torch.equal(po.local[b], ref))
        dist.barrier()
        po.close()
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_peer_outputs_two_processes_one_gpu():
    """Two ranks (processes) on one GPU: each maps the other's output buffers by
    CUDA IPC and its kernel 3 writes its heads (greedy plan) / head segments
    (split plan) into both; afterwards both ranks hold the full layer."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx_mp = mp.get_context("spawn")
    result = ctx_mp.Array("i", [0, 0, 0, 0])
    procs = [ctx_mp.Process(target=_two_rank_worker, args=(r, port, result)) for r in range(2)]
    for p_ in procs:
        p_.start()
    for p_ in procs:
        p_.join(timeout=300)
    assert all(p_.exitcode == 0 for p_ in procs)
    assert list(result) == [1, 1, 1, 1]
