"""Step-by-step GPU diagnostics for kernels 1-3 on tiny shapes (dev tool).

Prints, per case, whether scores/selection are bit-exact and the kernel-3
error against the fp64 oracle, so a failing stage is localised quickly.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_10353_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2603_10353_b200.workload import LayerSpec, bf16_bits, make_layer  # noqa: E402


def case(ctx, hq, hkv, n, kblocks, causal, seed=1):
    spec = LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=seed)
    q, k, v = make_layer(spec, "cpu")
    qb, kb, vb = bf16_bits(q), bf16_bits(k), bf16_bits(v)
    kblocks = np.asarray(kblocks, np.int64)
    nkb = (n + 127) // 128
    kmax = int(min(nkb, kblocks.max()))
    sc_o, idx_o, cnt_o, out_o = O.layer(qb, kb, vb, kblocks, bq=256, causal=causal, kmax=kmax)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    sc = ctx.block_scores(qd, kd, causal=causal)
    torch.cuda.synchronize()
    s_ok = np.array_equal(sc.cpu().numpy().view(np.uint32), sc_o.view(np.uint32))
    idx, cnt = ctx.select_blocks(sc, kblocks, n, causal=causal, kmax=kmax)
    torch.cuda.synchronize()
    i_ok = np.array_equal(idx.cpu().numpy(), idx_o) and np.array_equal(cnt.cpu().numpy(), cnt_o)
    t0 = time.time()
    out = ctx.block_sparse_attention(qd, kd, vd, idx, cnt, causal=causal)
    torch.cuda.synchronize()
    dt = time.time() - t0
    g = out.float().cpu().numpy().astype(np.float64)
    d = np.abs(g - out_o)
    rel = d.sum() / np.abs(out_o).sum()
    print(f"hq={hq} hkv={hkv} n={n} k={kblocks.tolist()} causal={causal}: scores_exact={s_ok} "
          f"select_exact={i_ok} fa max_abs={d.max():.3e} mean_rel={rel:.3e} ({dt*1e3:.1f} ms)",
          flush=True)
    if d.max() > 2e-2:
        worst = np.unravel_index(np.argmax(d), d.shape)
        print("   worst at", worst, "gpu", g[worst], "ref", out_o[worst])
        rows = d.max(axis=2)
        bad = np.argwhere(rows > 2e-2)
        print("   bad rows:", len(bad), "first:", bad[:8].tolist())
        print("   gpu row0[:8]", g[0, 0, :8], "\n   ref row0[:8]", out_o[0, 0, :8])
    return d.max()


def main():
    ctx = P.Context(0)
    case(ctx, 1, 1, 128, [1], False)
    case(ctx, 1, 1, 128, [1], True)
    case(ctx, 1, 1, 256, [2], False)
    case(ctx, 1, 1, 512, [3], True)
    case(ctx, 2, 1, 1024, [2, 8], True)
    case(ctx, 4, 2, 1000, [1, 3, 8, 5], True)
    case(ctx, 2, 1, 8192, [4, 24], True)


if __name__ == "__main__":
    main()
