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


@dataclass
class GatherMap:
    """Where every row of the all-gathered buffer goes. Rank r contributes a
    buffer of `hmax` head slots (its heads in ascending order, padded); after
    the all-gather slot r*hmax + i holds its i-th head. Whole heads move with
    one index copy (src_slots -> dst_heads); heads a sub-head plan split
    across ranks move as row ranges (slot, head, row0, row1)."""
    hmax: int
    num_heads: int
    src_slots: np.ndarray
    dst_heads: np.ndarray
    partial: list


def gather_map(plan, world: int, seq_len: int, block_q: int = 256) -> GatherMap:
    """GatherMap of a whole-head plan (device_of_head array) or a sub-head
    plan (api.split_assign result)."""
    src, dst, partial = [], [], []
    if isinstance(plan, np.ndarray) or isinstance(plan, (list, tuple)):
        p = np.asarray(plan)
        hmax = max(1, max(int((p == r).sum()) for r in range(world)))
        for r in range(world):
            heads = np.nonzero(p == r)[0]
            src += [r * hmax + i for i in range(heads.size)]
            dst += heads.tolist()
        return GatherMap(hmax, int(p.size), np.asarray(src, np.int64), np.asarray(dst, np.int64), partial)
    dev = np.asarray(plan.device)
    hmax = max(1, max(int((dev == r).sum()) for r in range(world)))
    nqb = -(-seq_len // block_q)
    for r in range(world):
        sel = np.nonzero(dev == r)[0]
        segs = sorted((int(plan.head[i]), int(plan.qb_begin[i]), int(plan.qb_end[i])) for i in sel)
        for i, (h, b0, b1) in enumerate(segs):
            if b0 == 0 and b1 >= nqb:
                src.append(r * hmax + i)
                dst.append(h)
            else:
                partial.append((r * hmax + i, h, b0 * block_q, min(b1 * block_q, seq_len)))
    return GatherMap(hmax, int(np.asarray(plan.head).max()) + 1, np.asarray(src, np.int64),
                     np.asarray(dst, np.int64), partial)


def apply_gather(recv, full, gm: GatherMap, src_t=None, dst_t=None) -> None:
    """full[head rows] <- recv[slots] per the map (on the current stream).
    src_t / dst_t: the index tensors already on recv's device (optional)."""
    import torch
    if gm.dst_heads.size:
        s = src_t if src_t is not None else torch.as_tensor(gm.src_slots, device=recv.device)
        d = dst_t if dst_t is not None else torch.as_tensor(gm.dst_heads, device=recv.device)
        full.index_copy_(0, d, recv.index_select(0, s))
    for slot, h, r0, r1 in gm.partial:
        full[h, r0:r1].copy_(recv[slot, r0:r1])


def _gather(local_out, gm: GatherMap, world: int, group=None):
    import torch
    import torch.distributed as dist
    tail = tuple(local_out.shape[1:])
    send = torch.zeros((gm.hmax,) + tail, dtype=local_out.dtype, device=local_out.device)
    send[:local_out.shape[0]] = local_out
    recv = torch.empty((world * gm.hmax,) + tail, dtype=local_out.dtype, device=local_out.device)
    dist.all_gather_into_tensor(recv, send, group=group)
    full = torch.empty((gm.num_heads,) + tail, dtype=local_out.dtype, device=local_out.device)
    apply_gather(recv, full, gm)
    return full


def gather_segments(local_out, split_plan, world: int, group=None, block_q: int = 256):
    """All-gather for a sub-head plan: rank r's local_out holds its heads
    (ordered like rank_segments(...).heads) with valid rows only inside each
    head's query-block range; returns [Hq, n, ...] with every row taken from
    the rank that computed it."""
    return _gather(local_out, gather_map(split_plan, world, local_out.shape[1], block_q), world, group)


def gather_heads(local_out, device_of_head, world: int, group=None):
    """All-gather per-rank outputs [h_r, ...] into [Hq, ...] in global head order.

    Every rank passes its own shard's outputs (rows ordered like
    RankShard.heads). Returns the full tensor on every rank.
    """
    return _gather(local_out, gather_map(np.asarray(device_of_head), world, local_out.shape[1]), world, group)


def agree_outcomes(ok: bool, payload, world: int, group=None) -> list:
    """[(ok, payload)] of every rank (all_gather_object): a setup step that can
    fail on one rank only (IPC export / open) is judged collectively, so a
    failure anywhere makes ALL ranks raise and fall back together instead of
    one rank entering a collective the others never reach."""
    if world == 1:
        return [(ok, payload)]
    import torch.distributed as dist
    res = [None] * world
    dist.all_gather_object(res, (ok, payload), group=group)
    return res


class PeerOutputs:
    """Full-layer output buffers [Hq, n, d] on every rank, mapped into every
    other rank (CUDA IPC over NVLink) for the fused gather: kernel 3 stores each
    output row straight into every rank's buffer (shplb_layer_shape.out_peers),
    so reassembly needs no all-gather and no reorder, only a barrier.

    All `sets` buffers of a rank are one allocation (one IPC handle, opened
    once per peer); ptrs(b) lists set b's device pointers as seen from this
    rank, own buffer first, then the other ranks in rank order.
    """

    HANDLE_BYTES = 72  # SHPLB_IPC_HANDLE_BYTES

    def __init__(self, num_heads: int, seq_len: int, head_dim: int, world: int, rank: int, device,
                 sets: int = 2, group=None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from ._native import ShplbError, check, lib
        self.world, self.rank, self.device = world, rank, torch.device(device)
        self.buffer = torch.empty((sets, num_heads, seq_len, head_dim), dtype=torch.bfloat16, device=self.device)
        self.local = [self.buffer[b] for b in range(sets)]
        set_bytes = num_heads * seq_len * head_dim * 2
        self._opened = []

        def agree(ok: bool, payload):
            return agree_outcomes(ok, payload, world, group)

        hnd = (C.c_char * self.HANDLE_BYTES)()
        try:
            check(lib().shplb_ipc_handle(C.c_void_p(self.buffer.data_ptr()), hnd, self.HANDLE_BYTES))
            mine = (True, bytes(hnd))
        except ShplbError as e:
            mine = (False, f"rank {rank}: {e}")
        handles = agree(*mine)
        bad = [m for ok, m in handles if not ok]
        if bad:
            raise ShplbError("; ".join(bad))
        bases = [self.buffer.data_ptr()]
        err = None
        for r in range(world):
            if r == rank:
                continue
            out = C.c_void_p()
            buf = (C.c_char * self.HANDLE_BYTES).from_buffer_copy(handles[r][1])
            try:
                check(lib().shplb_ipc_open(self.device.index or 0, buf, self.HANDLE_BYTES, C.byref(out)))
            except ShplbError as e:
                err = f"rank {rank} opening rank {r}'s buffer: {e}"
                break
            self._opened.append(out.value)
            bases.append(out.value)
        bad = [m for ok, m in agree(err is None, err) if not ok]
        if bad:
            self.close()
            raise ShplbError("; ".join(bad))
        self._ptrs = [[base + b * set_bytes for base in bases] for b in range(sets)]

    def ptrs(self, b: int) -> list:
        return self._ptrs[b % len(self._ptrs)]

    def close(self) -> None:
        import ctypes as C

        from ._native import lib
        for p in self._opened:
            lib().shplb_ipc_close(self.device.index or 0, C.c_void_p(p))
        self._opened = []
