"""Seeded synthetic attention layers with heterogeneous per-head sparsity.

The reference's own generator (profiler.cpp:93-155) realises target weights
through Q = sqrt(d)[I|0], which needs head_dim >= num_queries and cannot
express an 8K-128K prefill at d=128. This generator instead
draws bf16 Q [Hq, n, d] and K/V [Hkv, n, d] with structure that block pooling
can see:

* every key block b of KV head g has a centroid c[g,b] ~ N(0, I); its keys are
  ``alpha * c[g,b] + N(0, I)``;
* query i of head h mixes its own block's centroid (locality), the centroid
  of one random earlier "target" block, and noise, scaled by a per-head
  temperature ``tau_h`` drawn log-uniformly from ``tau_range`` — large tau
  makes a head sparse (mass concentrates on few blocks), small tau makes it
  dense. So different heads need different budgets, which is what the max-min
  allocator and the balancer act on.

``targets="per_head"`` (the accuracy study, not the bench default): each head
h has its own set of m_h "hot" key blocks, m_h log-uniform in [1, hot_max];
a query targets a random visible hot block of its head (its own block if none
is visible yet). Heads then differ in how many *blocks* they need — the
block-level heterogeneity the head-adaptive budget is meant to exploit.

Generation runs with torch on the target device (plumbing, not the product);
the same seed gives the same tensors on CPU and GPU generators separately, so
tests generate on CPU and copy, and the bench generates on the GPU.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

BLOCK = 128


@dataclass
class LayerSpec:
    num_q_heads: int = 32
    num_kv_heads: int = 8
    seq_len: int = 8192
    head_dim: int = 128
    seed: int = 2603
    tau_range: tuple = (0.15, 1.2)
    key_alpha: float = 1.0
    local_weight: float = 0.5
    target_weight: float = 1.0
    layer: int = 0
    targets: str = "per_query"  # or "per_head" (hot key blocks per head, see module doc)
    hot_max: int = 256


def head_temperatures(spec: LayerSpec) -> torch.Tensor:
    g = torch.Generator().manual_seed(spec.seed * 1000003 + spec.layer * 7919 + 11)
    lo, hi = (math.log(t) for t in spec.tau_range)
    u = torch.rand(spec.num_q_heads, generator=g, dtype=torch.float64)
    return torch.exp(lo + (hi - lo) * u).to(torch.float32)


@torch.no_grad()
def make_layer(spec: LayerSpec, device="cpu"):
    """Returns (q, k, v) bf16 tensors on `device`: [Hq,n,d], [Hkv,n,d], [Hkv,n,d]."""
    n, d, hq, hkv = spec.seq_len, spec.head_dim, spec.num_q_heads, spec.num_kv_heads
    nb = (n + BLOCK - 1) // BLOCK
    dev = torch.device(device)
    g = torch.Generator(device=dev).manual_seed(spec.seed * 1000003 + spec.layer)
    cent = torch.randn(hkv, nb, d, generator=g, device=dev)
    blk = torch.arange(n, device=dev) // BLOCK
    k = spec.key_alpha * cent[:, blk, :] + torch.randn(hkv, n, d, generator=g, device=dev)
    v = torch.randn(hkv, n, d, generator=g, device=dev)
    tau = head_temperatures(spec).to(dev)
    group = hq // hkv
    q = torch.empty(hq, n, d, device=dev)
    if spec.targets == "per_head":
        gh_ = torch.Generator().manual_seed(spec.seed * 1000003 + spec.layer * 7919 + 23)
        lo, hi = 0.0, math.log(max(1, min(spec.hot_max, nb)))
        m = torch.exp(lo + (hi - lo) * torch.rand(hq, generator=gh_, dtype=torch.float64)).round().long().clamp(min=1)
    for h in range(hq):
        gh = h // group
        u = torch.rand(n, generator=g, device=dev)
        if spec.targets == "per_head":
            # m_h hot blocks per head; a query picks a random visible one (else its own block)
            hot = torch.sort(torch.randperm(nb, generator=g, device=dev)[: int(m[h])]).values
            nvis = torch.searchsorted(hot, blk, right=True)  # hot blocks <= own block
            pick = torch.floor(u * nvis.clamp(min=1).to(u.dtype)).to(torch.int64)
            tgt = torch.where(nvis > 0, hot[pick.clamp(max=hot.numel() - 1)], blk)
        else:
            # one random earlier (or same) block per query: uniform in [0, own block]
            tgt = torch.floor(u * (blk + 1).to(u.dtype)).to(torch.int64)
        qh = (spec.local_weight * cent[gh, blk, :] + spec.target_weight * cent[gh, tgt, :]
              + torch.randn(n, d, generator=g, device=dev))
        q[h] = tau[h] * qh
    return (q.to(torch.bfloat16).contiguous(), k.to(torch.bfloat16).contiguous(),
            v.to(torch.bfloat16).contiguous())


def bf16_bits(t: torch.Tensor):
    """bf16 tensor -> numpy uint16 bit patterns (host copy)."""
    return t.detach().to("cpu").contiguous().view(torch.int16).numpy().view("uint16")
