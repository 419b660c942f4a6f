"""Randomised parity sweep of the layer call against the oracle: random head
counts, GQA ratios and explicit (non-contiguous) kv maps, ragged lengths,
both query-block sizes, causal and not, both selection kinds, per-head budgets
and sub-head query-block ranges. Selections bit-exact, outputs within the
kernel-3 tolerance, rows outside a head's range untouched.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2603_10353_b200.workload import LayerSpec, bf16_bits, make_layer
from tolerance import check_output

pytestmark = pytest.mark.gpu

SENTINEL = 4096.0  # bf16-exact; never an attention output (|out| <= max |v|)


def _case(seed):
    rng = np.random.default_rng(seed)
    hkv = int(rng.integers(1, 5))
    hq = hkv * int(rng.choice([1, 2, 4, 7]))
    n = int(rng.choice([int(rng.integers(1, 300)), int(rng.integers(300, 2600))]))
    bq = int(rng.choice([128, 256]))
    causal = bool(rng.integers(0, 2))
    kind = int(rng.integers(0, 2))
    nkb, nqb = (n + 127) // 128, (n + bq - 1) // bq
    k_blocks = rng.integers(1, nkb + 1, hq).astype(np.int64)
    kv_map = rng.integers(0, hkv, hq).astype(np.int32)
    kv_map[:hkv] = np.arange(hkv)  # every kv head used at least once (hq >= hkv)
    rng.shuffle(kv_map)
    ranges = None
    if rng.integers(0, 2):
        lo = rng.integers(0, nqb + 1, hq)
        hi = rng.integers(0, nqb + 1, hq)
        ranges = np.stack([np.minimum(lo, hi), np.maximum(lo, hi)], 1).astype(np.int32)
    return dict(hq=hq, hkv=hkv, n=n, bq=bq, causal=causal, kind=kind, k_blocks=k_blocks, kv_map=kv_map,
                ranges=ranges)


@pytest.mark.parametrize("seed", range(64))
def test_random_layer(cuda_ctx, seed):
    c = _case(1000 + seed)
    hq, hkv, n, bq = c["hq"], c["hkv"], c["n"], c["bq"]
    q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=seed), "cpu")
    kv_map = c["kv_map"]
    # oracle: one kv head per q head (k[kv_map[h]]), so its grouping is the identity
    qb, kb, vb = bf16_bits(q), bf16_bits(k)[kv_map], bf16_bits(v)[kv_map]
    nkb = (n + 127) // 128
    kmax = int(min(nkb, c["k_blocks"].max()))
    _, idx_o, cnt_o, out_o = O.layer(qb, kb, vb, c["k_blocks"], bq=bq, causal=c["causal"], kmax=kmax,
                                     kind=c["kind"])
    out = torch.full(q.shape, SENTINEL, dtype=torch.bfloat16, device="cuda")
    budgets = np.minimum(c["k_blocks"] * 128, n)
    cuda_ctx.sparse_attention_layer(q.cuda(), k.cuda(), v.cuda(), budgets, causal=c["causal"], out=out,
                                    kv_map=kv_map, block_q=bq, q_block_range=c["ranges"], kind=c["kind"])
    torch.cuda.synchronize()
    idx, cnt = cuda_ctx.last_selection(hq, n)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    assert np.array_equal(cnt, cnt_o), c
    assert np.array_equal(idx, idx_o), c
    g = out.float().cpu().numpy().astype(np.float64)
    mask = np.zeros((hq, n), bool)
    for h in range(hq):
        lo, hi = (0, (n + bq - 1) // bq) if c["ranges"] is None else c["ranges"][h]
        mask[h, lo * bq:min(hi * bq, n)] = True
    assert np.all(g[~mask] == SENTINEL), "rows outside the query-block range were written"
    if mask.any():
        check_output(g[mask], out_o[mask], str(c))
