"""Head-parallel plumbing on CPU with gloo, world_size 2 (the N>1 path of
bench.py without the GPU kernels): plan -> per-rank shards -> uneven
all-gather -> heads back in global order; budget broadcast; max-over-ranks
barrier metric."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2603_10353_b200 as P
from paper_2603_10353_b200.head_parallel import (agree_outcomes, gather_heads, gather_segments,
                                                  head_counts, rank_segments, rank_shard)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, budgets, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hq, group = len(budgets), 4
        # rank 0 owns the budget table; everyone receives it (bench.make_budgets)
        b = torch.tensor(budgets if rank == 0 else [0] * hq, dtype=torch.int64)
        dist.broadcast(b, 0)
        b = b.numpy()
        for name, plan in (("greedy", P.greedy_assign(b, world)),
                           ("naive", P.naive_assign(b, world))):
            sh = rank_shard(plan, rank, group, b)
            assert all(plan[h] == rank for h in sh.heads)
            assert [sh.kv_heads[m] for m in sh.kv_map] == [h // group for h in sh.heads]
            # stand-in for the rank's kernel output: head h filled with h
            local = torch.stack([torch.full((3, 2), float(h)) for h in sh.heads]) if sh.heads \
                else torch.zeros((0, 3, 2))
            full = gather_heads(local, plan, world)
            expect = torch.arange(hq, dtype=torch.float32)[:, None, None].expand(hq, 3, 2)
            assert torch.equal(full, expect), name
            # per-rank "latency" proportional to the rank's load; max over ranks
            load = float(b[sh.heads].sum())
            lat = torch.tensor([load])
            gathered = [torch.zeros(1) for _ in range(world)]
            dist.all_gather(gathered, lat)
            lats = [float(x) for x in gathered]
            res = P.barrier(lats)
            rep = P.imbalance(b, plan, world)
            assert res.barrier_latency == float(rep.loads.max())
            if rank == 0:
                results[name] = (res.barrier_latency, res.bubble_fraction, head_counts(plan, world))
        # sub-head plan: rows of a split head come from different ranks
        n, bq = 1000, 256
        sp = P.split_assign(b, world, n, block_q=bq)
        seg = rank_segments(sp, rank, group, b)
        local = torch.full((len(seg.heads), n, 2), -1.0)
        for i, h in enumerate(seg.heads):
            r0, r1 = seg.q_block_range[i] * bq
            local[i, r0:min(r1, n)] = h * 10000 + torch.arange(r0, min(r1, n))[:, None].float()
        full = gather_segments(local, sp, world, block_q=bq)
        want = (torch.arange(hq)[:, None] * 10000 + torch.arange(n)[None, :]).float()[..., None]
        assert torch.equal(full, want.expand(hq, n, 2))
        if rank == 0:
            results["split_heads"] = len(sp.head) - len(set(sp.head.tolist()))
    finally:
        dist.destroy_process_group()


def test_head_parallel_world2_gloo():
    budgets = [64 * 128, 128, 128, 32 * 128, 2 * 128, 128, 16 * 128, 128,
               8 * 128, 128, 4 * 128, 128]  # 12 heads, 3 kv groups of 4
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), budgets, results), nprocs=2, join=True)
    g_T, g_bub, g_counts = results["greedy"]
    n_T, n_bub, n_counts = results["naive"]
    assert n_counts == [6, 6]            # even HP splits by head count
    assert g_T <= n_T and g_bub <= n_bub  # the balancer never does worse here
    assert g_T == max(P.imbalance(budgets, P.greedy_assign(budgets, 2), 2).loads)
    assert results["split_heads"] <= 1  # at most D-1 heads are split


def _agree_worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank 1 fails its (IPC) setup step, rank 0 succeeds: both must see it
        out = agree_outcomes(rank != 1, "h0" if rank != 1 else "rank 1: open failed", world)
        results[rank] = [ok for ok, _ in out], [m for ok, m in out if not ok]
        # and the ranks stay in lock-step afterwards (the NCCL fallback's collectives)
        t = torch.tensor([rank + 1.0])
        dist.all_reduce(t)
        results[("sum", rank)] = float(t)
    finally:
        dist.destroy_process_group()


def test_fused_gather_setup_failure_is_collective():
    """PeerOutputs judges IPC setup collectively (agree_outcomes): a failure on
    one rank makes every rank fall back to the NCCL gather together."""
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_agree_worker, args=(2, _free_port(), results), nprocs=2, join=True)
    for r in range(2):
        assert results[r] == ([True, False], ["rank 1: open failed"])
        assert results[("sum", r)] == 3.0


@pytest.mark.parametrize("world", [2, 3, 8])
def test_plan_segments_match_rank_shards(world):
    """The segment list handed to shplb_gather_segments / shplb_gather_heads
    (api.plan_segments) names, for every rank, exactly the heads and rows that
    rank's shard computes, at the local index its layer-call output holds them."""
    import paper_2603_10353_b200 as P
    from paper_2603_10353_b200.head_parallel import rank_segments, rank_shard
    rng = np.random.default_rng(world)
    hq, n, group = 28, 5000, 7
    budgets = rng.choice([128, 1024, 2048, 5000], size=hq).astype(np.int64)
    for plan in (P.greedy_assign(budgets, world), P.naive_assign(budgets, world), P.split_assign(budgets, world, n)):
        segs = list(P.plan_segments(plan, world, hq, n))
        rows = np.zeros((hq, n), np.int32)
        for s in segs:
            rows[s.head, s.row_begin:s.row_end] += 1
        assert (rows == 1).all(), "every output row exactly once"
        for r in range(world):
            mine = [s for s in segs if s.owner == r]
            if isinstance(plan, P.api.SplitPlan):
                sh = rank_segments(plan, r, group, budgets)
                want = [(h, i, min(int(a) * 256, n), min(int(b) * 256, n))
                        for i, (h, (a, b)) in enumerate(zip(sh.heads, sh.q_block_range))]
                want = [w for w in want if w[3] > w[2]]
            else:
                sh = rank_shard(plan, r, group, budgets)
                want = [(h, i, 0, n) for i, h in enumerate(sh.heads)]
            assert [(s.head, s.local_head, s.row_begin, s.row_end) for s in mine] == want
