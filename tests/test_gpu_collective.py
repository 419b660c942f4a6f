"""Multi-rank C ABI (include/shplb.h "Head parallelism across ranks"): the
library's NCCL communicator, shplb_gather_segments / shplb_gather_heads and
shplb_comm_barrier, and the C++ host tool that runs a head-parallel layer over
them (tools/hp_layer.cpp).

One B200 is available: NCCL refuses two ranks on one device, so these run a
world-1 communicator. Every reassembly path is still exercised — segments with
arbitrary local slots and row ranges (what a rank's peers send), whole-head
plans, split plans — and checked bit-exact; the rank-to-rank transport is
NCCL's own. The plan/segment logic for world > 1 is covered on CPU
(tests/test_distributed.py)."""
import os
import subprocess

import numpy as np
import pytest
import torch

import paper_2603_10353_b200 as P
from paper_2603_10353_b200.workload import LayerSpec, make_layer

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def comm():
    c = P.NcclComm(0, 1, 0, P.NcclComm.unique_id())
    yield c
    c.close()


def _layer(hq=8, hkv=2, n=1000):
    q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=12), "cuda")
    budgets = np.array([128, 384, 1000, 256, 640, 128, 896, 512][:hq], np.int64)
    return q, k, v, budgets


def test_gather_segments_arbitrary_slots_and_rows(cuda_ctx, comm):
    """Every head cut into 1-3 row ranges, each held at its own local slot in a
    permuted order: the gather must put every row back at (head, row)."""
    q, k, v, budgets = _layer()
    ref = cuda_ctx.sparse_attention_layer(q, k, v, budgets)
    hq, n, d = ref.shape
    rng = np.random.default_rng(0)
    pieces = []
    for h in range(hq):
        cuts = sorted(set(rng.integers(1, n, size=rng.integers(0, 3)).tolist()))
        bounds = [0] + cuts + [n]
        pieces += [(h, bounds[i], bounds[i + 1]) for i in range(len(bounds) - 1)]
    order = rng.permutation(len(pieces))
    local = torch.full((len(pieces), n, d), float("nan"), dtype=torch.bfloat16, device="cuda")
    segs = (P.OutSegment * len(pieces))()
    for slot, i in enumerate(order):
        h, r0, r1 = pieces[i]
        local[slot, r0:r1] = ref[h, r0:r1]
        segs[slot] = P.OutSegment(h, 0, slot, 0, r0, r1)
    out = torch.zeros_like(ref)
    comm.gather_segments(cuda_ctx, out, local, segs)
    comm.barrier()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


@pytest.mark.parametrize("plan_kind", ["greedy", "split"])
def test_gather_reassembles_plan_shards(cuda_ctx, comm, plan_kind):
    """The rank's shard computed with the plan's kv map / query ranges, then the
    gather: bit-identical to the whole-layer call."""
    from paper_2603_10353_b200.head_parallel import rank_segments, rank_shard
    q, k, v, budgets = _layer(n=2000)
    ref = cuda_ctx.sparse_attention_layer(q, k, v, budgets)
    hq, n, d = ref.shape
    group = hq // k.shape[0]
    plan = P.greedy_assign(budgets, 1) if plan_kind == "greedy" else P.split_assign(budgets, 1, n)
    sh = rank_shard(plan, 0, group, budgets) if plan_kind == "greedy" else rank_segments(plan, 0, group, budgets)
    local = cuda_ctx.sparse_attention_layer(q[sh.heads].contiguous(), k[sh.kv_heads].contiguous(),
                                            v[sh.kv_heads].contiguous(), sh.budgets, kv_map=sh.kv_map,
                                            q_block_range=getattr(sh, "q_block_range", None))
    out = torch.zeros_like(ref)
    if plan_kind == "greedy":
        comm.gather_heads(cuda_ctx, out, local, plan)
    else:
        comm.gather_segments(cuda_ctx, out, local, P.plan_segments(plan, 1, hq, n))
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_gather_argument_errors(cuda_ctx, comm):
    out = torch.zeros((2, 256, 128), dtype=torch.bfloat16, device="cuda")
    local = torch.zeros_like(out)
    with pytest.raises(P.InvalidArgument, match="head 1 assigned to invalid device 1"):
        comm.gather_heads(cuda_ctx, out, local, np.array([0, 1], np.int32))
    segs = (P.OutSegment * 3)(P.OutSegment(0, 0, 0, 0, 0, 256), P.OutSegment(1, 0, 1, 0, 0, 128),
                              P.OutSegment(1, 0, 1, 0, 100, 256))
    with pytest.raises(P.InvalidArgument, match="head 1: segments must cover every output row exactly once"):
        comm.gather_segments(cuda_ctx, out, local, segs)
    segs = (P.OutSegment * 1)(P.OutSegment(0, 0, 0, 0, 0, 256))
    with pytest.raises(P.InvalidArgument, match="head 1: segments must cover"):
        comm.gather_segments(cuda_ctx, out, local, segs)
    dup = (P.OutSegment * 3)(P.OutSegment(0, 0, 0, 0, 0, 256), P.OutSegment(1, 0, 1, 0, 0, 256),
                             P.OutSegment(1, 0, 1, 0, 0, 256))
    with pytest.raises(P.InvalidArgument, match="exactly once"):
        comm.gather_segments(cuda_ctx, out, local, dup)
    with pytest.raises(P.InvalidArgument, match="rank 1 out of range"):
        P.NcclComm(0, 1, 1, P.NcclComm.unique_id())


@pytest.mark.parametrize("plan", ["greedy", "naive", "refined", "split"])
def test_cpp_host_head_parallel_layer(plan, tmp_path):
    """tools/hp_layer: plan -> shard layer -> NCCL gather, C ABI only, from a C++
    process; the reassembled layer is bit-identical to the single call."""
    exe = os.path.join(ROOT, "tools", "bin", "hp_layer")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools")], check=True)
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", SHPLB_ID_FILE=str(tmp_path / "id"))
    r = subprocess.run([exe, plan, "4096", "16", "4"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    assert '"bit_identical": true' in r.stdout, r.stdout
