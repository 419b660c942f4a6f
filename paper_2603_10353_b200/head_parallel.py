"""Head parallelism (HP): shard a layer's heads over ranks by a plan and
reassemble per-head outputs.

The plan is the reference's Assignment::device_of_head
(partitioner.hpp:16-22) from greedy_assign (S-HPLB) or naive_assign (even
HP). Each rank runs the hot path on its q heads and only the kv heads they
read (GQA: q head h reads kv head h // group); `kv_map` tells the kernels
which local kv head each local q head uses. Outputs are reassembled with one
all-gather over the process group (NCCL over NVLink on B200; gloo in the CPU
tests). Ranks hold different head counts, so each contributes a buffer padded
to the largest count and the receiver drops the padding.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class RankShard:
    heads: list        # global q heads on this rank, ascending
    kv_heads: list     # global kv heads those q heads read, ascending
    kv_map: list       # local kv index of each local q head
    budgets: np.ndarray


def rank_shard(device_of_head, rank: int, group: int, budgets) -> RankShard:
    plan = np.asarray(device_of_head)
    heads = np.nonzero(plan == rank)[0].tolist()
    kv_heads = sorted({h // group for h in heads})
    kv_map = [kv_heads.index(h // group) for h in heads]
    return RankShard(heads, kv_heads, kv_map, np.asarray(budgets, np.int64)[heads])


@dataclass
class RankSegments(RankShard):
    q_block_range: np.ndarray  # [len(heads), 2] query blocks [begin, end) per local head


def rank_segments(split_plan, rank: int, group: int, budgets) -> RankSegments:
    """The rank's part of a sub-head plan (api.split_assign): its heads, each
    with the query-block range it computes."""
    sel = np.nonzero(np.asarray(split_plan.device) == rank)[0]
    heads = [int(split_plan.head[i]) for i in sel]
    rng = np.array([[split_plan.qb_begin[i], split_plan.qb_end[i]] for i in sel],
                   np.int32).reshape(-1, 2)
    order = np.argsort(heads, kind="stable")
    heads = [heads[i] for i in order]
    rng = rng[order]
    kv_heads = sorted({h // group for h in heads})
    kv_map = [kv_heads.index(h // group) for h in heads]
    return RankSegments(heads, kv_heads, kv_map, np.asarray(budgets, np.int64)[heads], rng)


def head_counts(device_of_head, world: int) -> list:
    plan = np.asarray(device_of_head)
    return [int((plan == r).sum()) for r in range(world)]


def gather_segments(local_out, split_plan, world: int, group=None, block_q: int = 256):
    """All-gather for a sub-head plan: rank r's local_out holds its heads
    (ordered like rank_segments(...).heads) with valid rows only inside each
    head's query-block range; returns [Hq, n, ...] with every row taken from
    the rank that computed it."""
    import torch
    import torch.distributed as dist
    dev = np.asarray(split_plan.device)
    counts = [int((dev == r).sum()) for r in range(world)]
    hmax = max(counts)
    hq = int(np.asarray(split_plan.head).max()) + 1
    n = local_out.shape[1]
    tail = tuple(local_out.shape[1:])
    bq = block_q
    send = torch.zeros((hmax,) + tail, dtype=local_out.dtype, device=local_out.device)
    send[:local_out.shape[0]] = local_out
    recv = torch.empty((world * hmax,) + tail, dtype=local_out.dtype, device=local_out.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    full = torch.empty((hq,) + tail, dtype=local_out.dtype, device=local_out.device)
    for r in range(world):
        sel = np.nonzero(dev == r)[0]
        order = np.argsort(np.asarray(split_plan.head)[sel], kind="stable")
        for slot, i in enumerate(sel[order]):
            h = int(split_plan.head[i])
            r0, r1 = int(split_plan.qb_begin[i]) * bq, min(n, int(split_plan.qb_end[i]) * bq)
            full[h, r0:r1] = recv[r * hmax + slot, r0:r1]
    return full


def gather_heads(local_out, device_of_head, world: int, group=None):
    """All-gather per-rank outputs [h_r, ...] into [Hq, ...] in global head order.

    Every rank passes its own shard's outputs (rows ordered like
    RankShard.heads). Returns the full tensor on every rank.
    """
    import torch
    import torch.distributed as dist
    plan = np.asarray(device_of_head)
    counts = head_counts(plan, world)
    hmax = max(counts)
    tail = tuple(local_out.shape[1:])
    send = torch.zeros((hmax,) + tail, dtype=local_out.dtype, device=local_out.device)
    send[:local_out.shape[0]] = local_out
    recv = torch.empty((world * hmax,) + tail, dtype=local_out.dtype, device=local_out.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    full = torch.empty((plan.size,) + tail, dtype=local_out.dtype, device=local_out.device)
    for r in range(world):
        heads = np.nonzero(plan == r)[0]
        if heads.size:
            full[torch.as_tensor(heads, device=full.device)] = recv[r * hmax:r * hmax + heads.size]
    return full
