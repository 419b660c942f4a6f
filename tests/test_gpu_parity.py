"""GPU parity: kernels 1-3 and the layer call against the oracle.

* Kernel 1 (block scores) and kernel 2 (selected block sets) must be
  BIT-EXACT with the C restatement (oracle/shplb_oracle.c) — integer decisions
  on fp32 scores computed in the same fixed order on both sides.
* Kernel 3 outputs must match the fp64 oracle on the same kept sets within
  the bf16 tolerance of tests/tolerance.py: max-abs <= 2e-2 and mean-rel <=
  2 x the bf16 rounding floor of the compared reference rows (the floor is
  ~1.4e-3, so the north_star's 1e-3 example is below what any bf16 output can
  reach; the gate is derived per comparison instead).
"""
import numpy as np
import pytest
import torch

import paper_2603_10353_b200 as P
from oracle import oracle as O
from paper_2603_10353_b200.workload import LayerSpec, bf16_bits, make_layer

pytestmark = pytest.mark.gpu

from tolerance import check_output  # noqa: E402


def _scores_equal(a: np.ndarray, b: np.ndarray) -> bool:
    # bitwise on the fp32 patterns (-inf included), -0.0 folded onto +0.0
    a = np.where(a == 0, np.float32(0), a).astype(np.float32)
    b = np.where(b == 0, np.float32(0), b).astype(np.float32)
    return np.array_equal(a.view(np.uint32), b.view(np.uint32))


def run_case(ctx, spec: LayerSpec, k_blocks, causal=True, bq=256):
    q, k, v = make_layer(spec, "cpu")
    qb, kb, vb = bf16_bits(q), bf16_bits(k), bf16_bits(v)
    k_blocks = np.asarray(k_blocks, np.int64)
    nkb = (spec.seq_len + 127) // 128
    kmax = int(min(nkb, k_blocks.max()))
    sc_o, idx_o, cnt_o, out_o = O.layer(qb, kb, vb, k_blocks, bq=bq, causal=causal, kmax=kmax)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()

    sc = ctx.block_scores(qd, kd, causal=causal, block_q=bq)
    torch.cuda.synchronize()
    assert _scores_equal(sc.cpu().numpy(), sc_o), "kernel 1 scores differ from the oracle"

    idx, cnt = ctx.select_blocks(sc, k_blocks, spec.seq_len, causal=causal, kmax=kmax, block_q=bq)
    torch.cuda.synchronize()
    assert np.array_equal(cnt.cpu().numpy(), cnt_o), "kernel 2 counts differ"
    assert np.array_equal(idx.cpu().numpy(), idx_o), "kernel 2 block sets differ"

    out = ctx.block_sparse_attention(qd, kd, vd, idx, cnt, causal=causal, block_q=bq)
    torch.cuda.synchronize()
    mx, rel, _ = check_output(out, out_o, "kernel 3")

    budgets = np.minimum(k_blocks * 128, spec.seq_len)
    out2 = ctx.sparse_attention_layer(qd, kd, vd, budgets, causal=causal, block_q=bq)
    torch.cuda.synchronize()
    idx2, cnt2 = ctx.last_selection(spec.num_q_heads, spec.seq_len)
    assert np.array_equal(cnt2.cpu().numpy(), cnt_o)
    assert np.array_equal(idx2.cpu().numpy(), idx_o), "fused score+select differs from the oracle"
    assert torch.equal(out2, out), "layer call differs from kernel-by-kernel path"
    return mx, rel


@pytest.mark.parametrize("bq", [256, 128])
@pytest.mark.parametrize("causal", [True, False])
def test_small_gqa_layer(cuda_ctx, causal, bq):
    spec = LayerSpec(num_q_heads=4, num_kv_heads=2, seq_len=1024, seed=1)
    run_case(cuda_ctx, spec, [1, 3, 8, 5], causal=causal, bq=bq)


@pytest.mark.parametrize("bq", [256, 128])
@pytest.mark.parametrize("n", [1, 100, 128, 129, 256, 300, 1000, 1536])
def test_ragged_lengths(cuda_ctx, n, bq):
    spec = LayerSpec(num_q_heads=2, num_kv_heads=1, seq_len=n, seed=7 + n)
    nkb = (n + 127) // 128
    run_case(cuda_ctx, spec, [1, max(1, nkb // 2 + 1)], causal=True, bq=bq)
    run_case(cuda_ctx, spec, [nkb, 1], causal=False, bq=bq)


@pytest.mark.parametrize("bq", [256, 128])
def test_mha_and_wide_gqa(cuda_ctx, bq):
    run_case(cuda_ctx, LayerSpec(num_q_heads=3, num_kv_heads=3, seq_len=768, seed=3), [2, 6, 1],
             bq=bq)
    run_case(cuda_ctx, LayerSpec(num_q_heads=8, num_kv_heads=1, seq_len=640, seed=4),
             [1, 2, 3, 4, 5, 5, 2, 1], bq=bq)


def test_full_budget_equals_dense(cuda_ctx):
    """k = all blocks keeps every visible token: dense causal attention
    (test_attention.cpp:119-126 'sparse at full budget equals dense')."""
    spec = LayerSpec(num_q_heads=2, num_kv_heads=1, seq_len=512, seed=11)
    q, k, v = make_layer(spec, "cpu")
    out = cuda_ctx.sparse_attention_layer(q.cuda(), k.cuda(), v.cuda(), [512, 512], causal=True)
    torch.cuda.synchronize()
    for h in range(2):
        Q = q[h].double().numpy()
        K = k[0].double().numpy()
        V = v[0].double().numpy()
        ref = O.ref.dense_attention(Q, K, V, causal=True) if O.ref_available() else None
        if ref is None:
            s = Q @ K.T / np.sqrt(128)
            s[np.triu_indices(512, 1)] = -np.inf
            w = np.exp(s - s.max(1, keepdims=True))
            ref = (w / w.sum(1, keepdims=True)) @ V
        check_output(out[h], ref, f"head {h}")


@pytest.mark.parametrize("bq", [256, 128])
def test_single_kept_block_is_block_softmax(cuda_ctx, bq):
    """k = 1: each query block keeps exactly one key block (cf. 'budget one keeps
    the argmax key', test_attention.cpp:128-141, at block granularity). With
    bq = 256 and a future-half block kept, the first half's rows are zero."""
    spec = LayerSpec(num_q_heads=2, num_kv_heads=2, seq_len=512, seed=5)
    run_case(cuda_ctx, spec, [1, 1], causal=True, bq=bq)


def test_ties_break_toward_lower_block(cuda_ctx):
    """Identical key blocks give identical pooled scores; the lower block index
    must win (test_attention.cpp:187-195 at block granularity)."""
    spec = LayerSpec(num_q_heads=2, num_kv_heads=1, seq_len=1024, seed=9)
    q, k, v = make_layer(spec, "cpu")
    k = k.clone()
    for b in range(1, 8):  # every key block a copy of block 0
        k[:, b * 128:(b + 1) * 128] = k[:, 0:128]
    qb, kb, vb = bf16_bits(q), bf16_bits(k), bf16_bits(v)
    k_blocks = np.array([3, 2], np.int64)
    sc_o, idx_o, cnt_o, out_o = O.layer(qb, kb, vb, k_blocks, bq=128, causal=False, kmax=3)
    sc = cuda_ctx.block_scores(q.cuda(), k.cuda(), causal=False, block_q=128)
    idx, cnt = cuda_ctx.select_blocks(sc, k_blocks, 1024, causal=False, kmax=3, block_q=128)
    torch.cuda.synchronize()
    assert np.array_equal(idx.cpu().numpy(), idx_o)
    assert (idx_o[0, :, :3] == np.array([0, 1, 2])).all()
    assert (idx_o[1, :, :2] == np.array([0, 1])).all()


def test_kv_map_subset_of_heads(cuda_ctx):
    """A head-parallel rank holds an arbitrary subset of q heads plus the kv
    heads they read; the explicit kv map must reproduce the full layer's rows."""
    spec = LayerSpec(num_q_heads=8, num_kv_heads=4, seq_len=768, seed=21)
    q, k, v = make_layer(spec, "cpu")
    budgets = np.array([128, 256, 384, 512, 640, 128, 256, 768])
    full = cuda_ctx.sparse_attention_layer(q.cuda(), k.cuda(), v.cuda(), budgets, causal=True)
    heads = [1, 6, 7]  # kv heads 0, 3, 3
    kv_needed = sorted({h // 2 for h in heads})
    kv_map = [kv_needed.index(h // 2) for h in heads]
    part = cuda_ctx.sparse_attention_layer(q[heads].contiguous().cuda(),
                                           k[kv_needed].contiguous().cuda(),
                                           v[kv_needed].contiguous().cuda(), budgets[heads],
                                           causal=True, kv_map=kv_map)
    torch.cuda.synchronize()
    assert torch.equal(part, full[heads])


def test_errors_match_reference_messages(cuda_ctx):
    spec = LayerSpec(num_q_heads=2, num_kv_heads=1, seq_len=256, seed=2)
    q, k, v = (t.cuda() for t in make_layer(spec, "cpu"))
    with pytest.raises(P.InvalidArgument, match=r"budget k = 0 out of range \[1, 256\]"):
        cuda_ctx.sparse_attention_layer(q, k, v, [0, 128])
    with pytest.raises(P.InvalidArgument, match=r"budget k = 257 out of range \[1, 256\]"):
        cuda_ctx.sparse_attention_layer(q, k, v, [257, 128])
    bad = q.clone()
    bad[1, 3, 5] = float("nan")
    with pytest.raises(P.InvalidArgument, match="Q contains NaN or Inf"):
        cuda_ctx.sparse_attention_layer(bad, k, v, [128, 128], validate=True)
    with pytest.raises(P.NotSupported):
        cuda_ctx.sparse_attention_layer(q[:, :, :64].contiguous(), k[:, :, :64].contiguous(),
                                        v[:, :, :64].contiguous(), [128, 128])


@pytest.mark.parametrize("hkv", [1, 3, 8])
def test_host_buffer_entry_matches_device_call(cuda_ctx, hkv):
    """shplb_sparse_attention_layer_host (pinned host buffers, KV-head-chunked
    copy/compute pipeline) returns exactly the device-buffer layer result."""
    spec = LayerSpec(num_q_heads=2 * hkv, num_kv_heads=hkv, seq_len=1100, seed=30 + hkv)
    q, k, v = make_layer(spec, "cpu")
    budgets = np.array([128 * (1 + (h % 5)) for h in range(2 * hkv)])
    dev = cuda_ctx.sparse_attention_layer(q.cuda(), k.cuda(), v.cuda(), budgets)
    torch.cuda.synchronize()
    qh, kh, vh = (t.pin_memory() for t in (q, k, v))
    host = cuda_ctx.sparse_attention_layer_host(qh, kh, vh, budgets,
                                                out=torch.empty_like(q).pin_memory())
    assert torch.equal(host, dev.cpu())
    if hkv >= 3:  # a head-parallel shard: q heads 1, 2, 5 read kv heads 0, 1, 2 (monotone map)
        heads, kvs = [1, 2, 5], [0, 1, 2]
        shard = cuda_ctx.sparse_attention_layer_host(
            q[heads].contiguous().pin_memory(), k[kvs].contiguous().pin_memory(),
            v[kvs].contiguous().pin_memory(), budgets[heads], kv_map=[0, 1, 2],
            out=torch.empty((3,) + tuple(q.shape[1:]), dtype=q.dtype).pin_memory())
        assert torch.equal(shard, dev.cpu()[heads])


def test_deterministic(cuda_ctx):
    """Bit-identical results for identical inputs (test_attention.cpp:315-324)."""
    spec = LayerSpec(num_q_heads=4, num_kv_heads=2, seq_len=2048, seed=8)
    q, k, v = (t.cuda() for t in make_layer(spec, "cpu"))
    b = [256, 512, 1024, 128]
    a = cuda_ctx.sparse_attention_layer(q, k, v, b)
    c = cuda_ctx.sparse_attention_layer(q, k, v, b)
    torch.cuda.synchronize()
    assert torch.equal(a, c)


@pytest.mark.parametrize("bq", [256, 128])
def test_c1_shape_two_heads_full_oracle(cuda_ctx, bq):
    """Llama-3-8B-shaped (d=128) 8K prefill, two q heads of one GQA group,
    heterogeneous budgets; full oracle comparison."""
    spec = LayerSpec(num_q_heads=2, num_kv_heads=1, seq_len=8192, seed=2603)
    run_case(cuda_ctx, spec, [4, 24], causal=True, bq=bq)


# BASELINE.json configs at full size: (q heads, kv heads, n, requests stacked on the head axis).
AT_SIZE = {
    "C3": (32, 8, 131072, 1),    # Llama-3-8B layer at 128K
    "C4": (28, 4, 65536, 1),     # Qwen2.5-7B layer at 64K (GQA 7)
    "C5x2": (64, 8, 131072, 2),  # Llama-3-70B layer at 128K, two requests batched (128 q / 16 kv heads)
}


def at_size_layer(cfg: str, device="cuda"):
    hq, hkv, n, reqs = AT_SIZE[cfg]
    parts = [make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=2603 + 101 * r), device)
             for r in range(reqs)]
    return tuple(torch.cat([p[i] for p in parts]) if reqs > 1 else parts[0][i] for i in range(3))


@pytest.mark.slow
@pytest.mark.parametrize("cfg,bq", [("C3", 256), ("C3", 128), ("C4", 256), ("C4", 128), ("C5x2", 256)])
def test_at_size_sampled_rows(cuda_ctx, cfg, bq):
    """A whole BASELINE config layer at full size through the layer call:
    size-independent checks on every (head, query block) row (count = min(k_h,
    visible), ascending in-range indices), then bit-exact selection against the
    C restatement and fp64 outputs (bf16-floor gate) on sampled (head, query
    block) rows, in the style of the reference's oracle comparison
    (test_attention.cpp:143-177)."""
    q, k, v = at_size_layer(cfg)
    hq, n, _ = q.shape
    group = hq // k.shape[0]
    rng = np.random.default_rng(hash(cfg) % 2**32 + bq)
    budgets = rng.choice([128, 1024, 8192, n // 4], size=hq).astype(np.int64)
    out = cuda_ctx.sparse_attention_layer(q, k, v, budgets, causal=True, block_q=bq)
    torch.cuda.synchronize()
    idx, cnt = cuda_ctx.last_selection(hq, n)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    nqb = n // bq
    vis = (bq // 128) * np.arange(1, nqb + 1)
    kb = (budgets + 127) // 128
    assert np.array_equal(cnt, np.minimum(kb[:, None], vis[None, :]))
    live = np.arange(idx.shape[2])[None, None, :] < cnt[:, :, None]  # every row at once
    assert (idx[~live] == -1).all(), "padding past the count must be -1"
    assert (idx[live] >= 0).all() and (idx < vis[None, :, None])[live].all(), "index outside the causal range"
    assert (idx[:, :, 1:] > idx[:, :, :-1])[live[:, :, 1:]].all(), "selection not strictly ascending"
    for h in sorted(rng.choice(hq, 4, replace=False).tolist()):
        g = h // group
        qbits, kbits, vbits = bf16_bits(q[h]), bf16_bits(k[g]), bf16_bits(v[g])
        kp = O.pool_blocks(kbits, 128)
        qbs = sorted(set(rng.choice(nqb, 3, replace=False).tolist() + [0, nqb - 1]))
        sc = O.pooled_scores_rows(qbits, kp, qbs, bq=bq)
        for r, qbk in enumerate(qbs):
            c = cnt[h, qbk]
            sel = idx[h, qbk, :c]
            want = np.sort(O.topk_row(sc[r, :vis[qbk]].astype(np.float64), c))
            assert np.array_equal(sel, want), (cfg, h, qbk)
            rows = sorted({qbk * bq, qbk * bq + 77, qbk * bq + bq // 2, qbk * bq + bq - 1})
            ref = O.sparse_rows(qbits, kbits, vbits, rows, sel.tolist())
            check_output(out[h, rows], ref, f"{cfg} bq {bq} head {h} qb {qbk}")


@pytest.mark.parametrize("bq", [256, 128])
def test_split_plan_shards_reassemble_the_layer(cuda_ctx, bq):
    """Sub-head plan: every rank computes only its heads' query-block ranges;
    stitching the ranks' rows back together gives exactly the whole-layer call."""
    from paper_2603_10353_b200.head_parallel import rank_segments
    spec = LayerSpec(num_q_heads=6, num_kv_heads=2, seq_len=2000, seed=41)
    q, k, v = (t.cuda() for t in make_layer(spec, "cpu"))
    budgets = np.array([128, 1024, 384, 2000, 256, 768], np.int64)
    full = cuda_ctx.sparse_attention_layer(q, k, v, budgets, block_q=bq)
    sp = P.split_assign(budgets, 4, 2000, block_q=bq)
    got = torch.zeros_like(full)
    for r in range(4):
        seg = rank_segments(sp, r, 3, budgets)
        if not seg.heads:
            continue
        part = cuda_ctx.sparse_attention_layer(
            q[seg.heads].contiguous(), k[seg.kv_heads].contiguous(), v[seg.kv_heads].contiguous(),
            seg.budgets, kv_map=seg.kv_map, q_block_range=seg.q_block_range, block_q=bq)
        for i, h in enumerate(seg.heads):
            r0, r1 = seg.q_block_range[i] * bq
            got[h, r0:r1] = part[i, r0:r1]
    torch.cuda.synchronize()
    assert torch.equal(got, full)


def test_async_host_entry_matches_sync_over_layers(cuda_ctx):
    """shplb_sparse_attention_layer_host_async over several layers (two staging
    slots alternate) gives the synchronous call's outputs."""
    outs_sync, outs_async, inputs = [], [], []
    for li in range(3):
        q, k, v = make_layer(LayerSpec(num_q_heads=4, num_kv_heads=2, seq_len=777 + 256 * li, seed=40 + li), "cpu")
        b = np.array([128, 384, 777, 256], np.int64)
        hq_, hk_, hv_ = (t.contiguous().pin_memory() for t in (q, k, v))
        inputs.append((hq_, hk_, hv_, b))
        outs_sync.append(cuda_ctx.sparse_attention_layer_host(hq_, hk_, hv_, b).clone())
    stream = torch.cuda.Stream()
    for hq_, hk_, hv_, b in inputs:
        o = torch.empty(hq_.shape, dtype=hq_.dtype, pin_memory=True)
        outs_async.append(cuda_ctx.sparse_attention_layer_host(hq_, hk_, hv_, b, stream=stream, out=o,
                                                               asynchronous=True))
    stream.synchronize()
    for a, s_ in zip(outs_async, outs_sync):
        assert torch.equal(a, s_)


def test_async_host_entry_shape_shrinks_and_grows(cuda_ctx):
    """Chained async host calls whose layer shrinks, then grows within the staging
    buffer, then shrinks again: every call's two-slot staging must stay disjoint
    from the in-flight previous call's (a per-call slot stride let slot 1
    of a smaller layer overlap slot 0 of a larger one). Outputs == sync calls."""
    sizes = [(8, 4, 2304), (4, 2, 1024), (4, 2, 640), (8, 4, 1536), (2, 1, 896), (8, 4, 2304), (4, 2, 384)]
    layers, want = [], []
    for li, (hq, hk, n) in enumerate(sizes):
        q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hk, seq_len=n, seed=500 + li), "cpu")
        b = np.array([min(n, 128 * (1 + (3 * h + li) % 7)) for h in range(hq)], np.int64)
        q, k, v = (t.contiguous().pin_memory() for t in (q, k, v))
        layers.append((q, k, v, b))
    for q, k, v, b in layers:
        want.append(cuda_ctx.sparse_attention_layer_host(q, k, v, b).clone())
    stream = torch.cuda.Stream()
    for rep in range(2):
        outs = []
        for q, k, v, b in layers:
            o = torch.full(q.shape, float("nan"), dtype=q.dtype).pin_memory()
            outs.append(cuda_ctx.sparse_attention_layer_host(q, k, v, b, stream=stream, out=o, asynchronous=True))
        stream.synchronize()
        for i, (o, w) in enumerate(zip(outs, want)):
            assert torch.equal(o, w), f"rep {rep} layer {i} {sizes[i]}"


def test_host_entry_leaves_whole_layer_selection(cuda_ctx):
    """After a host-buffer call (run in KV-head chunks) last_selection describes
    the whole layer, equal to the device call's selection, and last_selection_work
    counts every chunk's tiles."""
    q, k, v = make_layer(LayerSpec(num_q_heads=8, num_kv_heads=4, seq_len=2048, seed=77), "cpu")
    b = np.array([128, 2048, 384, 640, 1024, 256, 128, 1536], np.int64)
    cuda_ctx.sparse_attention_layer(q.cuda(), k.cuda(), v.cuda(), b)
    torch.cuda.synchronize()
    idx_d, cnt_d = (t.clone() for t in cuda_ctx.last_selection(8, 2048))
    work_d = cuda_ctx.last_selection_work()
    cuda_ctx.sparse_attention_layer_host(q.contiguous(), k.contiguous(), v.contiguous(), b)
    idx_h, cnt_h = cuda_ctx.last_selection(8, 2048)
    assert torch.equal(cnt_h, cnt_d)
    assert torch.equal(idx_h, idx_d)
    assert cuda_ctx.last_selection_work() == work_d


def test_host_entry_budget_count_checked(cuda_ctx):
    q, k, v = make_layer(LayerSpec(num_q_heads=4, num_kv_heads=2, seq_len=512, seed=3), "cpu")
    with pytest.raises(P.InvalidArgument, match="need one budget per query head"):
        cuda_ctx.sparse_attention_layer_host(q, k, v, np.array([128, 128], np.int64))
    with pytest.raises(P.InvalidArgument, match="head 3: budget k = 0 out of range"):
        cuda_ctx.sparse_attention_layer_host(q, k, v, np.array([128, 128, 128, 0], np.int64))


def test_async_host_entry_interleaved_with_device_calls(cuda_ctx):
    """Async host calls run their kernels on the context's own stream; device
    calls on the caller's stream in between (sharing the context workspace)
    must stay ordered with them. Six layers, chains of 1-3 async calls broken by device
    calls, every output checked against the synchronous device call."""
    stream = torch.cuda.Stream()
    layers = []
    for li in range(6):
        q, k, v = make_layer(LayerSpec(num_q_heads=4, num_kv_heads=2, seq_len=1024 + 128 * li, seed=60 + li), "cpu")
        b = np.array([128, 384, 1024, 256], np.int64)
        layers.append((q, k, v, b))
    want = []
    for q, k, v, b in layers:
        want.append(cuda_ctx.sparse_attention_layer(q.cuda(), k.cuda(), v.cuda(), b).cpu())
    torch.cuda.synchronize()
    got, dev_got = {}, {}
    plan = ["a", "a", "d", "a", "a", "a", "d", "a"]  # async host / device call, cycling the layers
    with torch.cuda.stream(stream):
        for i, kind in enumerate(plan):
            q, k, v, b = layers[i % 6]
            if kind == "a":
                o = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
                got[i] = cuda_ctx.sparse_attention_layer_host(q.pin_memory(), k.pin_memory(), v.pin_memory(), b,
                                                              stream=stream, out=o, asynchronous=True)
            else:
                dev_got[i] = cuda_ctx.sparse_attention_layer(q.cuda(), k.cuda(), v.cuda(), b, stream=stream)
    stream.synchronize()
    for i, o in got.items():
        assert torch.equal(o, want[i % 6]), f"async call {i}"
    for i, o in dev_got.items():
        assert torch.equal(o.cpu(), want[i % 6]), f"device call {i}"


def test_max_heads_per_call(cuda_ctx):
    """256 q heads (kMaxHeads: the per-launch head table) in one call, against the
    oracle; 257 is refused with NotSupported."""
    spec = LayerSpec(num_q_heads=256, num_kv_heads=32, seq_len=384, seed=99)
    kb = (np.arange(256) % 3) + 1
    run_case(cuda_ctx, spec, kb, causal=True, bq=256)
    q = torch.zeros((257, 128, 128), dtype=torch.bfloat16, device="cuda")
    k = torch.zeros((1, 128, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(P.NotSupported, match="at most 256 query heads per call"):
        cuda_ctx.sparse_attention_layer(q, k, k, np.full(257, 128, np.int64))


def test_sequence_length_limit_is_reported(cuda_ctx):
    """Kernel 2's shared-memory score rows bound n (380,416 tokens); longer
    sequences are refused up front with NotSupported, not a launch failure."""
    q = torch.zeros((1, 383104, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(P.NotSupported, match="exceeds the selector's limit of 380416 tokens"):
        cuda_ctx.sparse_attention_layer(q, q, q, [128])


def test_zero_q_gives_uniform_weights_over_kept_keys(cuda_ctx):
    """test_attention.cpp:44-61 at block granularity: Q = 0 makes every score 0,
    all blocks tie and the lowest k block indices are kept; each output row is
    the plain mean of V over its kept, causally visible keys."""
    n, kblk = 512, 2
    spec = LayerSpec(num_q_heads=1, num_kv_heads=1, seq_len=n, seed=17)
    _, k, v = make_layer(spec, "cpu")
    q = torch.zeros((1, n, 128), dtype=torch.bfloat16)
    out = cuda_ctx.sparse_attention_layer(q.cuda(), k.cuda(), v.cuda(), [kblk * 128], causal=True)
    torch.cuda.synchronize()
    vf = v[0].double().numpy()
    ref = np.empty((n, 128))
    for i in range(n):
        last = min(i, kblk * 128 - 1)  # kept blocks 0..kblk-1, causal
        ref[i] = vf[: last + 1].mean(0)
    check_output(out[0], ref, "zero q")


@pytest.mark.parametrize("bq", [256, 128])
@pytest.mark.parametrize("gain", [3.0, 12.0, 60.0])
def test_score_jumps_between_blocks(cuda_ctx, gain, bq):
    """Later key blocks score far above the first kept one (K of every third
    block scaled by `gain`): the running max of a row must move — kernel 3's
    lazy rescale (and, for jumps past 2^32 or to +inf in fp32, its exact-max
    fallback) — and the output still match the fp64 kept-set softmax."""
    n = 2048
    spec = LayerSpec(num_q_heads=2, num_kv_heads=1, seq_len=n, seed=int(gain) + bq)
    q, k, v = make_layer(spec, "cpu")
    k = k.float()
    for b in range(1, n // 128, 3):
        k[:, b * 128:(b + 1) * 128] *= gain
    k = k.to(torch.bfloat16)
    qb, kb, vb = bf16_bits(q), bf16_bits(k), bf16_bits(v)
    k_blocks = np.array([6, 16], np.int64)
    _, idx_o, cnt_o, out_o = O.layer(qb, kb, vb, k_blocks, bq=bq, causal=True, kmax=16)
    out = cuda_ctx.sparse_attention_layer(q.cuda(), k.cuda(), v.cuda(), k_blocks * 128, causal=True, block_q=bq)
    torch.cuda.synchronize()
    idx, cnt = cuda_ctx.last_selection(2, n)
    assert np.array_equal(cnt.cpu().numpy(), cnt_o) and np.array_equal(idx.cpu().numpy(), idx_o)
    check_output(out, out_o, f"score jumps x{gain}")


@pytest.mark.parametrize("group", ["1", "3"])
def test_kernel2_group_sizes(group):
    """Kernel 2 scores up to 4 q heads of one kv head per CTA (64 row slots =
    G heads x 64 / 32 / 16 / 16 query blocks for G = 1..4); SHPLB_K2_GROUP
    caps G, so 1 (64 query blocks of one head) and 3 (16 query blocks, 16
    slots idle, GQA-4 groups split 3 + 1) run the other row mappings on the parity cases of this file,
    in a subprocess (the switch is read once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-q", "-x",
                        "-k", "small_gqa_layer or ragged_lengths or mha_and_wide or ties or c1_shape or kv_map"],
                       cwd=root, env=dict(os.environ, SHPLB_K2_GROUP=group), capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("bq", [256, 128])
@pytest.mark.parametrize("n,causal", [(32769, True), (33000, False), (40000, True)])
def test_kernel2_key_split_partial_chunk(cuda_ctx, n, causal, bq):
    """Rows longer than one 256-block pooled-K chunk take the key-split kernel 2
    (grid.z over chunks, then the selector): 32769 tokens leave a last chunk of
    one key block, 33000 a ragged one, non-causal rows see every chunk."""
    spec = LayerSpec(num_q_heads=2, num_kv_heads=1, seq_len=n, seed=n + bq + int(causal))
    run_case(cuda_ctx, spec, [2, 3], causal=causal, bq=bq)


def test_kernel2_fused_single_kernel():
    """Kernel 2 splits the pooled-K chunks of a long row over grid.z and selects
    in a second kernel (the default when a row has more than 256 key blocks);
    SHPLB_K2_SPLIT=0 keeps the fused score + select kernel. The at-size C4 case
    (64K: 2 key chunks, GQA 7) under the fused kernel, in a subprocess."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-q", "-x",
                        "-k", "at_size_sampled_rows and C4"],
                       cwd=root, env=dict(os.environ, SHPLB_K2_SPLIT="0"), capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("bq", [256, 128])
def test_caller_selection_with_empty_rows(cuda_ctx, causal, bq):
    """shplb_block_sparse_attention on a caller-made selection (random counts,
    zeros included, ascending random visible blocks): rows whose query block
    keeps nothing are zero (attention.cpp:40-41), the others match the fp64
    oracle on their kept sets — kernel 3 runs every tile, empty ones included
    (the persistent kernel's tile handshakes must hold without any P·V)."""
    n = 1500
    spec = LayerSpec(num_q_heads=3, num_kv_heads=1, seq_len=n, seed=41 + bq + int(causal))
    q, k, v = make_layer(spec, "cpu")
    qbits, kbits, vbits = bf16_bits(q), bf16_bits(k), bf16_bits(v)
    nqb, nkb = (n + bq - 1) // bq, (n + 127) // 128
    rng = np.random.default_rng(bq + 2 * int(causal))
    kmax = nkb
    idx = np.full((3, nqb, kmax), -1, np.int32)
    cnt = np.zeros((3, nqb), np.int32)
    for h in range(3):
        for qb in range(nqb):
            vis = min(nkb, (min((qb + 1) * bq, n) - 1) // 128 + 1) if causal else nkb
            c = 0 if rng.random() < 0.35 else int(rng.integers(1, vis + 1))
            cnt[h, qb] = c
            idx[h, qb, :c] = np.sort(rng.choice(vis, c, replace=False))
    out = cuda_ctx.block_sparse_attention(q.cuda(), k.cuda(), v.cuda(), torch.from_numpy(idx).cuda(),
                                          torch.from_numpy(cnt).cuda(), causal=causal, block_q=bq)
    torch.cuda.synchronize()
    o = out.float().cpu()
    assert (cnt == 0).any() and (cnt > 0).any()
    for h in range(3):
        for qb in range(nqb):
            rows = list(range(qb * bq, min(n, (qb + 1) * bq)))
            if cnt[h, qb] == 0:
                assert torch.count_nonzero(o[h, rows]) == 0, (h, qb)
                continue
            ref = O.sparse_rows(qbits[h], kbits[0], vbits[0], rows, idx[h, qb, :cnt[h, qb]].tolist(), causal=causal)
            check_output(out[h, rows], ref, f"caller selection h {h} qb {qb}")


def test_single_cta_kernel3_variant():
    """The single-CTA kernel (fa_sm100.cu, SHPLB_K3=single — also the block_q =
    128 kernel) on the parity cases of this file and the fused-gather tests, in a
    subprocess (the switch is read once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "tests/test_gpu_gather.py", "-q",
                        "-x", "-k", "small_gqa_layer or ragged_lengths or mha_and_wide or kv_map or zero_q or "
                                    "single_kept or full_budget or c1_shape or fused_gather or caller_selection"],
                       cwd=root, env=dict(os.environ, SHPLB_K3="single"), capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_ticket_ring_reuse_over_many_launches(cuda_ctx):
    """The persistent kernel 3 takes tiles with a per-launch ticket counter from
    a ring of 64 and resets it itself (its last draw): 150 launches with three
    different tile counts, alternating between two (ordered) streams, wrap the
    ring twice; every output equals a fresh context's."""
    spec = LayerSpec(num_q_heads=4, num_kv_heads=2, seq_len=1536, seed=12)
    q, k, v = (t.cuda() for t in make_layer(spec, "cpu"))
    tables = [np.array(b, np.int64) for b in ([128, 256, 384, 512], [1536, 128, 640, 256], [768, 768, 768, 768])]
    fresh = P.Context(0)
    want = [fresh.sparse_attention_layer(q, k, v, b) for b in tables]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for i in range(150):
        s_ = streams[i % 2]
        with torch.cuda.stream(s_):
            outs.append((i % 3, cuda_ctx.sparse_attention_layer(q, k, v, tables[i % 3], stream=s_)))
        streams[(i + 1) % 2].wait_stream(s_)  # the context's workspace is shared: keep the launches ordered
    torch.cuda.synchronize()
    for t, o in outs:
        assert torch.equal(o, want[t])
    fresh.close()


def test_work_list_cache_eviction(monkeypatch):
    """Kernel-3 work lists are LRU-evicted (SHPLB_WORKLIST_CACHE entries) with
    stream-ordered frees: cycling more distinct budget tables than the cache
    holds, asynchronously on one stream, gives the same outputs as a context
    that never evicts."""
    monkeypatch.setenv("SHPLB_WORKLIST_CACHE", "2")
    small = P.Context(0)
    monkeypatch.delenv("SHPLB_WORKLIST_CACHE")
    big = P.Context(0)
    q, k, v = (t.cuda() for t in make_layer(LayerSpec(num_q_heads=4, num_kv_heads=2, seq_len=1536, seed=8), "cpu"))
    tables = [np.array([128 * (1 + (i + h) % 5) for h in range(4)], np.int64) for i in range(7)]
    stream = torch.cuda.Stream()
    want = [big.sparse_attention_layer(q, k, v, b).clone() for b in tables]
    outs = []
    for rep in range(3):
        for b in tables:
            outs.append(small.sparse_attention_layer(q, k, v, b, stream=stream))
    stream.synchronize()
    for i, o in enumerate(outs):
        assert torch.equal(o, want[i % len(tables)]), i
    small.close()
    big.close()
