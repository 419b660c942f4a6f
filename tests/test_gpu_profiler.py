"""GPU recovery-curve profiler (shplb_profile_curves[_kind])
against the host restatement and the compiled reference's build_profiles
(profiler.cpp:157-196, recovery_ratio attention.cpp:151-184) for both
PerQueryTopK and ColumnAggregateTopK.

Curves are fp64; the reference sums each top-k in nth_element's arbitrary
order, so agreement is to rounding (1e-12 absolute). The max-min budget
table computed from the GPU curves must equal the one from the host curves
(integer decisions on those curves).
"""
import numpy as np
import pytest
import torch

import paper_2603_10353_b200 as P
from oracle import oracle as O
from paper_2603_10353_b200.workload import LayerSpec, bf16_bits, make_layer

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _rand_bf16(rng, shape, scale=1.0):
    return torch.from_numpy((rng.standard_normal(shape) * scale).astype(np.float32)).to(torch.bfloat16)


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("hq,hkv,rows,n_k,stride", [(4, 2, 6, 300, 32), (8, 8, 3, 1000, 64),
                                                    (4, 1, 16, 4096, 128), (2, 1, 1, 129, 1)])
def test_gpu_profile_matches_host(cuda_ctx, hq, hkv, rows, n_k, stride, kind):
    rng = np.random.default_rng(hq * 1000 + n_k)
    q = _rand_bf16(rng, (hq, rows, 128)) * torch.from_numpy(
        rng.uniform(0.05, 0.5, (hq, 1, 1)).astype(np.float32)).to(torch.bfloat16)
    k = _rand_bf16(rng, (hkv, n_k, 128))
    grid = P.default_budget_grid(n_k, stride)
    host = P.profile_curves(bf16_bits(q), bf16_bits(k), grid, kind=kind)
    gpu = cuda_ctx.profile_curves(q.cuda(), k.cuda(), grid, kind=kind)
    for h in range(hq):
        assert np.abs(gpu[h].recovery - host[h].recovery).max() < TOL, f"head {h}"
        assert gpu[h].recovery[0] == 0.0 and abs(gpu[h].recovery[-1] - 1.0) < 1e-9


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built")
@pytest.mark.parametrize("kind", [0, 1])
def test_gpu_profile_matches_reference_build_profiles(cuda_ctx, kind):
    rng = np.random.default_rng(11)
    hq, hkv, rows, n_k = 4, 2, 5, 700
    q = _rand_bf16(rng, (hq, rows, 128), 0.3)
    k = _rand_bf16(rng, (hkv, n_k, 128))
    grid = P.default_budget_grid(n_k, 64)
    gpu = cuda_ctx.profile_curves(q.cuda(), k.cuda(), grid, kind=kind)
    Q = q.float().numpy().astype(np.float64)
    K = np.repeat(k.float().numpy().astype(np.float64), hq // hkv, axis=0)
    ref = O.ref.build_profiles(Q, K, np.zeros_like(K), grid, kind=kind)
    for h in range(hq):
        assert np.abs(gpu[h].recovery - ref[h]).max() < TOL


def test_gpu_profile_budget_table_equals_host(cuda_ctx):
    """The bench's calibration (last 16 rows of a structured 8K layer) ->
    max-min budgets: identical from GPU and host curves."""
    spec = LayerSpec(num_q_heads=32, num_kv_heads=8, seq_len=8192, seed=2603)
    q, k, _ = make_layer(spec, "cpu")
    n = spec.seq_len
    grid = P.default_budget_grid(n, 128)
    host = P.profile_curves(bf16_bits(q[:, n - 16:, :]), bf16_bits(k), grid)
    gpu = cuda_ctx.profile_curves(q[:, n - 16:, :].cuda(), k.cuda(), grid)
    worst = max(np.abs(g.recovery - h.recovery).max() for g, h in zip(gpu, host))
    assert worst < TOL
    total = int(0.25 * 32 * n)
    a = P.maxmin_allocate(host, total, quantum=128, floor=128).budgets
    b = P.maxmin_allocate(gpu, total, quantum=128, floor=128).budgets
    assert np.array_equal(a, b)


def test_gpu_profile_errors(cuda_ctx):
    q = torch.zeros((2, 2, 128), dtype=torch.bfloat16, device="cuda")
    k = torch.zeros((1, 64, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(P.InvalidArgument, match="budget grid must include the full context length"):
        cuda_ctx.profile_curves(q, k, [0, 32])
    with pytest.raises(P.InvalidArgument, match="strictly increasing"):
        cuda_ctx.profile_curves(q, k, [0, 32, 32, 64])
    with pytest.raises(P.InvalidArgument, match=r"budget grid entry 65 out of \[0, 64\]"):
        cuda_ctx.profile_curves(q, k, [0, 65])
    with pytest.raises(P.InvalidArgument, match="multiple of num_kv_heads"):
        cuda_ctx.profile_curves(torch.zeros((3, 2, 128), dtype=torch.bfloat16, device="cuda"),
                                torch.zeros((2, 64, 128), dtype=torch.bfloat16, device="cuda"), [0, 64])


@pytest.mark.parametrize("hq,hkv,n,bq,causal,nrows", [(4, 2, 1000, 128, True, 7), (4, 2, 1000, 256, True, 5),
                                                      (2, 1, 300, 256, False, 3), (8, 2, 4096, 256, True, 16),
                                                      (3, 3, 129, 128, True, 2)])
def test_block_selection_profile_matches_oracle(cuda_ctx, hq, hkv, n, bq, causal, nrows):
    """shplb_profile_curves_block against the numpy/C restatement
    (oracle.block_selection_profile): same kept blocks (kernel 2's fp32 ranking),
    fp64 masses to rounding."""
    q, k, _ = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=n + bq), "cpu")
    rows = np.unique(np.linspace(0, n - 1, nrows).round().astype(np.int64))
    grid = P.default_budget_grid(n, 128)
    gpu = cuda_ctx.profile_curves_block(q.cuda(), k.cuda(), rows, grid, block_q=bq, causal=causal)
    want = O.block_selection_profile(bf16_bits(q), bf16_bits(k), rows, grid, bq=bq, causal=causal)
    for h in range(hq):
        assert np.abs(gpu[h].recovery - want[h]).max() < TOL, f"head {h}"
        assert gpu[h].recovery[0] == 0.0 and abs(gpu[h].recovery[-1] - 1.0) < 1e-9
        assert (np.diff(gpu[h].recovery) >= 0).all()


def test_block_selection_profile_is_the_layers_kept_mass(cuda_ctx):
    """At a budget b the curve equals the softmax mass (fp64) of the calibration
    rows inside the blocks the LAYER CALL actually selected with every head at b
    — the profile describes the kernels' own selection, not a restatement of it."""
    hq, hkv, n, bq = 4, 2, 2048, 256
    q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=5), "cpu")
    rows = np.array([100, 700, 1300, 2047], np.int64)
    grid = P.default_budget_grid(n, 128)
    curves = cuda_ctx.profile_curves_block(q.cuda(), k.cuda(), rows, grid, block_q=bq)
    for b in (128, 384, 1024):
        cuda_ctx.sparse_attention_layer(q.cuda(), k.cuda(), v.cuda(), np.full(hq, b), block_q=bq)
        idx, cnt = (t.cpu().numpy() for t in cuda_ctx.last_selection(hq, n))
        for h in range(hq):
            K = k[h // (hq // hkv)].double().numpy()
            got = 0.0
            for p in rows:
                s = q[h, p].double().numpy() @ K[: p + 1].T / np.sqrt(128)
                w = np.exp(s - s.max())
                w /= w.sum()
                sel = idx[h, p // bq, : cnt[h, p // bq]]
                got += sum(w[blk * 128:(blk + 1) * 128].sum() for blk in sel)
            assert abs(curves[h].recovery_at(b) - got / rows.size) < 1e-12, (b, h)
