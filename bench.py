#!/usr/bin/env python
"""bench.py — S-HPLB sparse-attention hot path on B200.

Metric (BASELINE.json): attention ms/layer at 128K context, max over ranks, at
1/2/4/8 B200; bubble %; TFLOP/s.

Workload (config C3, the configuration the metric is quoted on): the
Llama-3-8B-shaped 32-layer attention stack — per layer 32 query / 8 KV heads,
d=128, 131072-token causal prefill, bf16 synthetic inputs
(paper_2603_10353_b200.workload), each layer with its own seed. Per-head
budgets per layer: recovery curves profiled on calibration rows (GPU
profiler) -> max-min allocation at B = 0.25*Hq*n tokens (the reference
default budget fraction, commands.hpp:28), quantum = floor = 128. Heads are
placed on ranks by the greedy (LPT) plan per layer; the even-HP (naive
contiguous) and sub-head (split) plans are timed beside it when N > 1.

A step = the whole stack: for every layer kernel 1 (pool) + kernel 2
(score+select) + kernel 3 (block-sparse FA) over the rank's heads, inputs
resident in HBM (48 GiB for 32 layers; every layer's 1.5 GiB exceeds the
126 MB L2). `value` = step time / layers (ms per layer), max over ranks;
at N > 1 it includes each layer's output all-gather, overlapped with the next
layer's compute (`compute_only_ms` without it). Timing: W warm-up steps, then
K steps bracketed by barrier + synchronize, CUDA events on the launching
stream. `e2e` runs the stack (or its first --e2e-layers layers) through the public
host-buffer API with inputs copied host(pinned)->device and the output
device->host inside the timed region, every step (ms per layer).

`--impl reference` times the reference's own CPU implementation
(headbal::sparse_attention, compiled unmodified into oracle/_ref) on the box's
host cores on a bounded sample of the same workload and extrapolates to
ms/layer.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse_args():
    p = argparse.ArgumentParser(description=__doc__.split("\n")[1])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["shplb", "reference"], default="shplb")
    p.add_argument("--seq-len", type=int, default=131072)
    p.add_argument("--q-heads", type=int, default=32)
    p.add_argument("--kv-heads", type=int, default=8)
    p.add_argument("--budget-fraction", type=float, default=0.25)
    p.add_argument("--calib-rows", type=int, default=128,
                   help="calibration rows per head, evenly spaced through the sequence (SURVEY d2)")
    p.add_argument("--profile-kind", choices=["token", "block"], default="token",
                   help="recovery curves of the budget table: 'token' = the reference's build_profiles "
                        "(PerQueryTopK, per-token top-k mass), 'block' = the kernels' own block selection "
                        "(shplb_profile_curves_block, causal rows)")
    p.add_argument("--seed", type=int, default=2603)
    p.add_argument("--layers", type=int, default=32,
                   help="distinct attention layers per step (C3: the 32-layer stack); each has its "
                        "own inputs, budget table and head plan")
    p.add_argument("--e2e-layers", type=int, default=0,
                   help="layers timed through the host-buffer entry for e2e (ms/layer); 0 = the whole "
                        "stack (--layers), i.e. the same step as `value`")
    p.add_argument("--allocation-json", default=None,
                   help="budget table from an allocation.json (reference format) instead of profiling")
    p.add_argument("--assignment-json", default=None,
                   help="S-HPLB head plan from an assignment.json (reference format) instead of greedy_assign")
    p.add_argument("--project-degrees", type=int, nargs="*", default=[2, 4, 8],
                   help="N=1 only: time every rank's shard of layer 0 under the naive / greedy / split "
                        "plans for these GPU counts on this GPU (per-rank compute of a D-GPU run)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0,
                   help="target CPU time of the bounded reference sample")
    p.add_argument("--c1-repeats", type=int, default=1,
                   help="--impl reference: time the whole C1 layer (8K) this many times, best reported "
                        "(0 = skip)")
    p.add_argument("--gather", choices=["nccl", "p2p"], default="p2p",
                   help="N>1 output reassembly: the C ABI's NCCL gather (shplb_gather_segments, one "
                        "broadcast per output segment, no padding or reorder) on a comm stream, or the "
                        "fused gather (kernel 3 stores rows into every rank's buffer over NVLink)")
    p.add_argument("--policy", choices=["per_query_topk", "column_aggregate_topk"], default="per_query_topk",
                   help="selection policy (SelectionKind) of the profile and the layer: per (head, query "
                        "block) top-k blocks, or one kept block set per head (block granularity)")
    p.add_argument("--placement", choices=["greedy", "greedy_refined", "split"], default="greedy",
                   help="N>1 headline plan: 'greedy' = the reference's whole-head greedy_assign (LPT on "
                        "budgets, bit-exact); 'greedy_refined' = greedy on tile cost + whole-head local "
                        "search (shplb_plan_refine); 'split' = the sub-head balancer (shplb_plan_split). "
                        "All plans are timed and reported either way")
    p.add_argument("--force-gather", action="store_true",
                   help="validation: run the overlapped all-gather pipeline even at N=1 (1-rank NCCL group)")
    p.add_argument("--debug-one-device", action="store_true",
                   help="debug only: run every rank on cuda:0 with gloo (exercise the N>1 path "
                        "on a 1-GPU box; timings are not meaningful)")
    return p.parse_args()


DEBUG_GLOO = False  # set by --debug-one-device: collectives on CPU tensors over gloo


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return FALLBACK_PEAKS, "fallback"


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"shplb_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx.append(float(parts[2]))
                except ValueError:
                    continue
                try:
                    pw.append(float(parts[3]))
                except ValueError:
                    pass
                for nm, val in zip(names, parts[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return None
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
               "samples": len(sm)}
        if pw:
            out["power_w_median"] = statistics.median(pw)
        return out


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------

def dist_setup(n_gpus, debug_one_device=False):
    import torch
    global DEBUG_GLOO
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}: launch N>1 under torchrun")
    if world > 1 and debug_one_device:
        import torch.distributed as dist
        DEBUG_GLOO = True
        local = 0
        torch.cuda.set_device(0)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
    elif world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def init_single_rank_group(local):
    """A 1-rank NCCL group (--force-gather at N=1): exercises the gather pipeline."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))


def make_hp_comm(world, rank, local):
    """The library's NCCL communicator (shplb_nccl_comm_init) for the layer-output
    gathers and barriers; its unique id travels over the torch.distributed
    group (plumbing only). None in the one-device gloo debug mode."""
    import torch
    import paper_2603_10353_b200 as P
    if DEBUG_GLOO:
        return None
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(P.NcclComm.unique_id()), dtype=torch.uint8))
    if world > 1:
        import torch.distributed as dist
        dist.broadcast(uid, 0)
    return P.NcclComm(local, world, rank, bytes(uid.cpu().numpy().tobytes()))


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allgather_float(x: float, world):
    if world == 1:
        return [x]
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if DEBUG_GLOO else "cuda")
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [float(o.item()) for o in out]


# ---------------------------------------------------------------------------
# budgets
# ---------------------------------------------------------------------------

def make_budgets(q, k, args, world, rank, pctx=None):
    """Max-min budget table from calibration rows (rank 0), broadcast to all ranks."""
    import paper_2603_10353_b200 as P
    from paper_2603_10353_b200 import calibrate
    n, hq = args.seq_len, args.q_heads
    total = int(round(args.budget_fraction * hq * n))
    info = {}
    if args.allocation_json:  # a budget table written by the reference CLI (allocator.cpp:240-273)
        la = P.formats.load_allocation(args.allocation_json)
        if la.budgets.size != hq:
            raise SystemExit(f"{args.allocation_json}: {la.budgets.size} budgets for {hq} heads")
        return la.budgets.astype(np.int64), la.total, {"source": args.allocation_json,
                                                       "digest": calibrate.table_digest(la.budgets)}
    if rank == 0:
        kind = "colagg" if args.policy == "column_aggregate_topk" else args.profile_kind
        budgets, info, _ = calibrate.layer_budgets(q, k, args.budget_fraction, kind=kind, rows=args.calib_rows,
                                                   quantum=128, floor=128, ctx=pctx)
    else:
        budgets = np.zeros(hq, np.int64)
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.from_numpy(budgets)
        t = t if DEBUG_GLOO else t.cuda()
        dist.broadcast(t, 0)
        budgets = t.cpu().numpy()
    return budgets, total, info


# ---------------------------------------------------------------------------
# timed loops
# ---------------------------------------------------------------------------

class LayerShard:
    """One layer's work on this rank: its q heads (contiguous), the kv heads
    they read, the local kv map, budgets and optional query-block ranges."""

    def __init__(self, q, k, v, shard, ranges, full: bool):
        if full:  # every head on this rank: no copy
            self.q, self.k, self.v = q, k, v
        else:
            self.q = q[shard.heads].contiguous()
            self.k, self.v = k[shard.kv_heads].contiguous(), v[shard.kv_heads].contiguous()
        self.heads, self.kv_map, self.budgets, self.ranges = shard.heads, shard.kv_map, shard.budgets, ranges
        self.flops = 0.0


KIND = 0  # selection kind of every layer call (--policy)


def run_layer(ctx, ls, out, stream):
    if not ls.heads:
        return
    ctx.sparse_attention_layer(ls.q, ls.k, ls.v, ls.budgets, causal=True, out=out, kv_map=ls.kv_map,
                               stream=stream, q_block_range=ls.ranges, kind=KIND)


def board_energy_mj(index):
    """The board's total energy counter (mJ, NVML), or None."""
    try:
        import pynvml
        pynvml.nvmlInit()
        return pynvml.nvmlDeviceGetTotalEnergyConsumption(pynvml.nvmlDeviceGetHandleByIndex(index))
    except Exception:  # noqa: BLE001 - no NVML: the line simply carries no energy
        return None


def time_stack(ctx, shards, steps, warmup, world, stream):
    """K timed steps of the whole stack (every layer's kernels 1-3 back to back
    on one stream, inputs resident). Returns ms per layer, mean per-call stage
    ms, launches per step, one output buffer, and the board energy per layer
    over the timed region (J, NVML; None without it)."""
    import torch
    hmax = max(1, max(len(ls.heads) for ls in shards))
    ref = next((ls.q for ls in shards if ls.heads), shards[0].q)
    out = torch.empty((hmax,) + tuple(ref.shape[1:]), dtype=ref.dtype, device=ref.device)
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            for ls in shards:
                run_layer(ctx, ls, out[:len(ls.heads)], stream)
    torch.cuda.synchronize()
    for ls in shards:  # exact tiles / FLOPs of each layer's selection (untimed)
        if ls.heads:
            run_layer(ctx, ls, out[:len(ls.heads)], stream)
            ls.flops = ctx.last_selection_work()[1]
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    ctx.set_timing(True)
    launches0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mj0 = board_energy_mj(torch.cuda.current_device())
    e0.record(stream)
    for _ in range(steps):
        for ls in shards:
            run_layer(ctx, ls, out[:len(ls.heads)], stream)
    e1.record(stream)
    torch.cuda.synchronize()
    mj1 = board_energy_mj(torch.cuda.current_device())
    joules = None if mj0 is None or mj1 is None else (mj1 - mj0) / 1e3 / (steps * len(shards))
    launches = (ctx.launches - launches0) // max(1, steps)
    stages = ctx.read_timing(max_calls=steps * len(shards) + 8)
    ctx.set_timing(False)
    barrier(world)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (steps * len(shards))
    st = stages.mean(axis=0) if len(stages) else np.zeros(3)
    return ms, st, launches, out, joules


def time_stack_gathered(ctx, shards, plans, hq, steps, warmup, world, stream, hp_comm):
    """The stack with every layer's outputs reassembled on every rank through the
    C ABI's NCCL gather (shplb_gather_segments: one ncclBroadcast per output
    segment from its owner straight into every rank's [Hq, n, d] buffer, one
    NCCL group per layer; no padding, no reorder) on a communication stream
    while layer l+1 computes; two output buffer sets alternate, the compute of
    layer l+2 waits for layer l's gather. Returns ms per layer (max over
    ranks) of the whole pipeline."""
    import torch

    import paper_2603_10353_b200 as P
    n_l = len(shards)
    ref = next(ls.q for ls in shards if ls.heads)
    tail = tuple(ref.shape[1:])
    segs = [P.plan_segments(plans[l], world, hq, tail[0]) for l in range(n_l)]
    hmax = max(max(len(ls.heads) for ls in shards), 1)
    local = [torch.zeros((hmax,) + tail, dtype=ref.dtype, device=ref.device) for _ in range(2)]
    full = [torch.empty((hq,) + tail, dtype=ref.dtype, device=ref.device) for _ in range(2)]
    comm = torch.cuda.Stream()
    done = [torch.cuda.Event() for _ in range(2)]
    computed = [torch.cuda.Event() for _ in range(2)]

    def one_step():
        for l, ls in enumerate(shards):
            b = l % 2
            stream.wait_event(done[b])  # layer l-2's gather has released local/full[b]
            run_layer(ctx, ls, local[b][:len(ls.heads)], stream)
            computed[b].record(stream)
            comm.wait_event(computed[b])
            hp_comm.gather_segments(ctx, full[b], local[b], segs[l], stream=comm)
            done[b].record(comm)
        stream.wait_stream(comm)

    with torch.cuda.stream(stream):
        for _ in range(warmup):
            one_step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(steps):
            one_step()
        e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    return max(allgather_float(e0.elapsed_time(e1) / (steps * n_l), world))


def time_stack_p2p(ctx, shards, hq, steps, warmup, world, rank, stream, hp_comm=None):
    """The stack with the fused gather: kernel 3 of every rank stores each output
    row straight into every rank's full [Hq, n, d] buffer (CUDA IPC peer
    pointers over NVLink), so a layer needs no all-gather or reorder — only a
    cross-rank barrier (shplb_comm_barrier: a 1-element all-reduce on the
    library's NCCL communicator, on a communication stream) before its buffer
    set is reused two layers later. ms per layer, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2603_10353_b200.head_parallel import PeerOutputs
    ref = next(ls.q for ls in shards if ls.heads)
    po = PeerOutputs(hq, ref.shape[1], ref.shape[2], world, rank, ref.device, sets=2)
    comm = torch.cuda.Stream()
    done = [torch.cuda.Event() for _ in range(2)]
    computed = [torch.cuda.Event() for _ in range(2)]

    def one_step():
        for l, ls in enumerate(shards):
            b = l % 2
            stream.wait_event(done[b])
            if ls.heads:
                ctx.sparse_attention_layer(ls.q, ls.k, ls.v, ls.budgets, causal=True, kv_map=ls.kv_map,
                                           stream=stream, q_block_range=ls.ranges,
                                           gather=(po.ptrs(b), ls.heads, hq), kind=KIND)
            if DEBUG_GLOO:  # exercising the path with every rank on one GPU: host barrier
                torch.cuda.synchronize()
                dist.barrier()
                continue
            computed[b].record(stream)
            comm.wait_event(computed[b])
            if world > 1:
                hp_comm.barrier(stream=comm)
            done[b].record(comm)
        stream.wait_stream(comm)

    with torch.cuda.stream(stream):
        for _ in range(warmup):
            one_step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(steps):
            one_step()
        e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    po.close()
    return max(allgather_float(e0.elapsed_time(e1) / (steps * len(shards)), world))


def e2e_layer_budget(shards, wanted: int, local_ranks: int = 1) -> int:
    """Layers the e2e leg can pin on this host: each needs its Q/K/V and output
    in pinned host memory; stay within half of MemAvailable shared by the
    ranks of the node (at least 2 layers, so the async pipeline still overlaps)."""
    per_layer = [sum(t.numel() * t.element_size() for t in (ls.q, ls.k, ls.v)) + ls.q.numel() * ls.q.element_size()
                 for ls in shards if ls.heads]
    if not per_layer:
        return 0
    try:
        with open("/proc/meminfo") as f:
            avail = next(int(x.split()[1]) * 1024 for x in f if x.startswith("MemAvailable:"))
    except (OSError, StopIteration, ValueError):
        return min(wanted, len(per_layer))
    budget = avail // 2 // max(1, local_ranks)
    n, used = 0, 0
    for b in per_layer[:wanted]:
        if n >= 2 and used + b > budget:
            break
        used += b
        n += 1
    return n


def time_e2e(ctx, shards, steps, warmup, world, stream):
    """End to end through the reference-facing C-ABI call with HOST buffers
    (shplb_sparse_attention_layer_host): for every layer of `shards`, pinned
    host Q/K/V -> device, kernels 1-3, output -> pinned host, stream
    synchronised — every step. Returns ms per layer and bytes per layer."""
    import torch
    shards = [ls for ls in shards if ls.heads]
    def pinned(t):  # device -> pinned host by DMA (no pageable staging copy)
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h

    host = [tuple(pinned(t) for t in (ls.q, ls.k, ls.v)) for ls in shards]

    outs = [torch.empty(ls.q.shape, dtype=ls.q.dtype, pin_memory=True) for ls in shards]  # per layer

    def step():  # layer l+1's H2D overlaps layer l's kernels and D2H (async host entry)
        for ls, (hq_, hk_, hv_), o in zip(shards, host, outs):
            ctx.sparse_attention_layer_host(hq_, hk_, hv_, ls.budgets, causal=True, out=o,
                                            stream=stream, kv_map=ls.kv_map, q_block_range=ls.ranges,
                                            asynchronous=True, kind=KIND)
        stream.synchronize()

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    # bytes per layer (the e2e value is ms per layer), averaged over the timed layers
    h2d = sum(t.numel() * t.element_size() for hs in host for t in hs) // len(host)
    d2h = sum(o.numel() * o.element_size() for o in outs) // len(outs)
    return e0.elapsed_time(e1) / (steps * len(shards)), h2d, d2h


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref = the reference library, unmodified)
# ---------------------------------------------------------------------------

class RefKV:
    """fp64 K / V of every kv head (the reference's HeadData holds fp64), built
    once and shared by every sample step (the bf16 -> fp64 conversion is
    harness work, not the reference's)."""

    def __init__(self, k, v):
        from paper_2603_10353_b200.workload import bf16_bits
        self.k = [_ref_f64(bf16_bits(k[g])) for g in range(k.shape[0])]
        self.v = [_ref_f64(bf16_bits(v[g])) for g in range(v.shape[0])]


def cpu_reference_sample(q, k, v, budgets, group, target_s, rng_seed=0, kv=None, rows_per_call=None):
    """Time headbal::sparse_attention (PerQueryTopK, fp64, OpenMP over rows) on
    a bounded sample of (head, query-row) pairs and extrapolate to ms/layer.
    Per-row cost is O(n_k*d) whatever the budget or causal mask (scores are
    computed before masking, attention.cpp:22-30), so the sample rows are run
    without the mask and the time scales linearly with the row count. Each
    call takes 16 rows per thread so OpenMP's fixed cost per call stays small
    against the rows (checked against a whole measured C1 layer in the
    reference arm's c1_full_layer)."""
    from oracle import oracle as O
    from paper_2603_10353_b200.workload import bf16_bits
    hq, n, d = q.shape
    threads = O.ref.max_threads()
    rows_per_call = rows_per_call or min(n, 16 * max(threads, 4))
    kv = kv or RefKV(k, v)
    rng = np.random.default_rng(rng_seed)
    heads = list(rng.permutation(hq))
    per_row = []  # seconds per (head,row) for each call
    spent = 0.0
    calls = 0
    for h in heads:
        g = h // group
        rows = np.sort(rng.choice(n, rows_per_call, replace=False))
        qq = _ref_f64(bf16_bits(q[h][rows]))
        _, sec = O.ref.sparse_attention_timed(qq, kv.k[g], kv.v[g], int(budgets[h]), causal=False)
        per_row.append(sec / rows_per_call)
        spent += sec
        calls += 1
        if spent >= target_s:
            break
    ms_layer = float(np.mean(per_row)) * hq * n * 1e3
    sample = (f"{calls} heads x {rows_per_call} query rows of the {hq}x{n} layer "
              f"(headbal::sparse_attention, PerQueryTopK, fp64, budgets b_h), "
              f"{spent:.1f} s timed, extrapolated linearly to {hq}x{n} rows")
    return ms_layer, threads, sample


def cpu_reference_serial_head(q, k, v, budgets, group, rows=8):
    """The bench_attention pattern (bench_attention.cpp:71-80): the serial
    reference::sparse_attention on one head, timed on `rows` query rows and
    extrapolated to the head's n rows (ms)."""
    import time as _t

    from oracle import oracle as O
    from paper_2603_10353_b200.workload import bf16_bits
    hq, n, d = q.shape
    h = int(np.argmax(budgets))
    kk = (bf16_bits(k[h // group]).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    vv = (bf16_bits(v[h // group]).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    sel = np.linspace(0, n - 1, rows).astype(np.int64)
    qq = (bf16_bits(q[h][sel]).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    t0 = _t.time()
    O.ref.sparse_attention(qq, kk, vv, int(budgets[h]), causal=False, serial=True)
    return (_t.time() - t0) / rows * n * 1e3


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _ref_f64(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def committed_reference_table(hq, hkv, n, seed, calib_rows, fraction):
    """(budgets, path) of a reference-written allocation.json for this layer
    under oracle/tables (tools/ref_budget_table.py), or None."""
    from oracle import oracle as O
    from paper_2603_10353_b200 import calibrate
    pos = calibrate.calibration_rows(n, calib_rows)
    name = f"hq{hq}_kv{hkv}_n{n}_seed{seed}_rows{pos.size}_q128.f{fraction}.allocation.json"
    path = os.path.join(ROOT, "oracle", "tables", name)
    if not os.path.exists(path) or not O.ref_available():
        return None
    b, _, tot, _ = O.ref.load_allocation(path)
    if tot != int(round(fraction * hq * n)) or b.size != hq:
        return None
    return b.astype(np.int64), f"oracle/tables/{name}"


def reference_table(q, k, v, args, seed, fraction=None):
    """The layer's max-min budget table as the REFERENCE builds it:
    headbal::build_profiles (PerQueryTopK, the calibration rows, grid stride
    128) -> headbal::maxmin_allocate (quantum 128, floor 128). Read from the
    reference-written files under oracle/tables/ (tools/ref_budget_table.py;
    headbal::save_allocation / save_profiles) when present — the reference's
    profile of a 128K layer takes minutes — else computed here by the reference.
    Returns (budgets, source)."""
    from oracle import oracle as O
    from paper_2603_10353_b200 import calibrate
    from paper_2603_10353_b200.workload import bf16_bits
    hq, n, _ = q.shape
    f = args.budget_fraction if fraction is None else fraction
    total = int(round(f * hq * n))
    pos = calibrate.calibration_rows(n, args.calib_rows)
    tag = f"hq{hq}_kv{k.shape[0]}_n{n}_seed{seed}_rows{pos.size}_q128"
    tables = os.path.join(ROOT, "oracle", "tables")
    prof = os.path.join(tables, f"{tag}.profiles.json")
    hit = committed_reference_table(hq, k.shape[0], n, seed, args.calib_rows, f)
    if hit is not None:
        return hit[0], f"{hit[1]} (headbal::load_allocation)"
    if os.path.exists(prof):
        curves = O.ref.load_profiles(prof)[0]
        src = f"headbal::maxmin_allocate on oracle/tables/{os.path.basename(prof)} (headbal::load_profiles)"
    else:
        import torch
        group = hq // k.shape[0]
        idx = torch.as_tensor(pos, device=q.device)
        Q = np.stack([_ref_f64(bf16_bits(q[h].index_select(0, idx))) for h in range(hq)])
        K = np.stack([_ref_f64(bf16_bits(k[h // group])) for h in range(hq)])
        V = np.stack([_ref_f64(bf16_bits(v[h // group])) for h in range(hq)])
        grid = np.asarray(list(range(0, n, 128)) + [n], np.int64)
        rec = O.ref.build_profiles(Q, K, V, grid, causal=False, kind=0)
        curves = [(grid, r) for r in rec]
        src = "headbal::build_profiles -> headbal::maxmin_allocate, computed in this run"
    b, _, _ = O.ref.maxmin_allocate(curves, n, total, quantum=128, floor=128)
    return b.astype(np.int64), src


def c1_full_layer(args, repeats=1):
    """C1 (BASELINE.json configs[0], the reference's own CPU-runnable case):
    one Llama-3-8B-shaped layer (32 q / 8 kv heads, d = 128) of 8192 tokens,
    causal, every head through headbal::sparse_attention with its own budget
    (the run_skyline loop, commands.cpp:464-470) — timed in full, no
    extrapolation, best of `repeats` (bench_attention.cpp:71-90). Budgets: the
    reference's build_profiles -> maxmin_allocate at the bench's fraction. Also
    the bench's sampled estimator on the same layer, to check the
    extrapolation C3's value relies on."""
    import torch
    from oracle import oracle as O
    from paper_2603_10353_b200.workload import LayerSpec, bf16_bits, make_layer
    hq, hkv, n = 32, 8, 8192
    q, k, v = make_layer(LayerSpec(num_q_heads=hq, num_kv_heads=hkv, seq_len=n, seed=args.seed), "cuda")
    budgets, src = reference_table(q, k, v, args, args.seed)
    group = hq // hkv
    Qh = [_ref_f64(bf16_bits(q[h])) for h in range(hq)]
    Kg = [_ref_f64(bf16_bits(k[g])) for g in range(hkv)]
    Vg = [_ref_f64(bf16_bits(v[g])) for g in range(hkv)]
    runs = []
    for _ in range(max(1, repeats)):
        t0 = time.perf_counter()
        for h in range(hq):
            O.ref.sparse_attention(Qh[h], Kg[h // group], Vg[h // group], int(budgets[h]), causal=True)
        runs.append((time.perf_counter() - t0) * 1e3)
    est, _, est_sample = cpu_reference_sample(q, k, v, budgets, group, 3.0, rng_seed=7)
    del q, k, v
    torch.cuda.empty_cache()
    return {"what": ("C1: 32 q / 8 kv heads x 8192 tokens, causal, headbal::sparse_attention per head "
                     "(PerQueryTopK, fp64) with its max-min budget, whole layer timed, no extrapolation"),
            "ms": round(min(runs), 1), "runs_ms": [round(x, 1) for x in runs], "best_of": len(runs),
            "budget_table": src, "budgets_min_max": [int(budgets.min()), int(budgets.max())],
            "sampled_estimate_ms": round(est, 1), "sampled_estimate_over_measured": round(est / min(runs), 4),
            "sampled_estimate": est_sample}


def run_reference(args):
    """The reference arm: headbal::sparse_attention (compiled unmodified into
    oracle/_ref) on the box's host cores. A step = a bounded sample of (head,
    row) pairs of layer 0 of the C3 stack with the budgets the reference's own
    build_profiles -> maxmin_allocate produced for that layer; `value` is that
    sample extrapolated linearly to ms per layer (per-row cost is O(n_k d)
    whatever the budget or mask, attention.cpp:22-30), `ms_per_step` the
    sample's measured wall time. `cpu_baseline.c1_full_layer` is a measured,
    unextrapolated whole C1 layer."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2603_10353_b200.workload import LayerSpec, make_layer
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libheadbal_ref.so not built (make -C oracle with /root/reference)"}))
        return
    c1 = c1_full_layer(args, args.c1_repeats) if args.c1_repeats > 0 else None
    spec = LayerSpec(num_q_heads=args.q_heads, num_kv_heads=args.kv_heads, seq_len=args.seq_len,
                     seed=args.seed)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    q, k, v = make_layer(spec, dev)
    budgets, table_src = reference_table(q, k, v, args, args.seed)
    from paper_2603_10353_b200 import calibrate
    group = args.q_heads // args.kv_heads
    per_step = max(1.0, args.cpu_seconds / max(1, args.steps))
    vals, walls = [], []
    threads, sample = 1, ""
    kv = RefKV(k, v)
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        ms, threads, sample = cpu_reference_sample(q, k, v, budgets, group, per_step, rng_seed=i, kv=kv)
        if i >= args.warmup:
            vals.append(ms)
            walls.append((time.perf_counter() - t0) * 1e3)
    value = float(np.mean(vals))
    step_ms = float(np.mean(walls))
    cpu = {"value": round(value, 3), "unit": "ms", "cores": threads, "kind": "reference",
           "cpu_model": cpu_model(),
           "sample": (f"per step: {sample}; layer 0 of the stack, whose per-layer CPU cost stands for every "
                      f"layer (budget- and mask-independent); step wall time = ms_per_step"),
           "budget_table": table_src, "budget_table_digest": calibrate.table_digest(budgets)}
    if c1:
        cpu["c1_full_layer"] = c1
    line = {
        "impl": "reference",
        "metric": "attention ms/layer at 128K ctx (max over ranks)",
        "value": round(value, 3), "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(step_ms, 3), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, budgets_desc(args), args.placement if world > 1 else "greedy"),
        "cpu_baseline": cpu,
        "e2e": {"value": round(value, 3), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def budgets_desc(args):
    """The budget table both arms use (the same string in both lines' config)."""
    if args.allocation_json:
        return f"from {args.allocation_json} (reference allocation.json)"
    kind = ("ColumnAggregateTopK" if args.policy == "column_aggregate_topk"
            else "PerQueryTopK (token level)" if args.profile_kind == "token" else "block selection")
    return (f"max-min at {args.budget_fraction} x Hq x n tokens, quantum 128, floor 128, on {kind} recovery "
            f"curves of {args.calib_rows} evenly spaced calibration rows per head, grid stride 128")


PLACEMENTS = {
    "greedy": ("greedy (LPT) whole-head plan (greedy_assign, bit-exact with the reference); even head "
               "parallelism (naive_even_hp), greedy on tile cost (greedy_tile_cost), its whole-head "
               "refinement (greedy_refined) and the sub-head balancer (split_subhead) are timed alongside"),
    "greedy_refined": ("whole-head plan: greedy_assign on kernel 3's tile cost per head (+ 4 tiles per visited "
                       "query tile), refined by moves / "
                       "swaps of heads off the most loaded rank (shplb_plan_refine); the reference's greedy plan, "
                       "even head parallelism and the sub-head balancer are timed alongside"),
    "split": ("sub-head balancer (shplb_plan_split): heads in index order with exact tile costs, cut "
              "McNaughton-style at query-block boundaries, at most D-1 heads split; the reference's "
              "whole-head greedy plan is timed alongside (greedy_whole_head)"),
}


def k3_traffic():
    """DRAM bytes (read + write) of one kernel-3 launch from the newest ncu
    --set full capture of the bench's layer 0 committed under profiles/
    (profiles/rNN/ncu_k3_summary.json), and where the number comes from."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_k3_summary.json")), reverse=True):
        try:
            d = json.load(open(path))
            return d["dram_bytes_per_launch"], (f"{os.path.relpath(path, ROOT)}: {d.get('what', '')}").strip()
        except Exception:
            continue
    return None, "no ncu capture committed"


def measure_fp32_peak():
    """FFMA throughput of this GPU, measured now (tools/bin/fp32_peak), or None."""
    exe = os.path.join(ROOT, "tools", "bin", "fp32_peak")
    if not os.path.exists(exe):
        return None
    try:
        r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
        return json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else None
    except Exception:
        return None


def stage_rooflines(layers, plans, rank, group, n, stages, peaks, fp32_peak, split):
    """Kernel 1 against HBM bandwidth (algorithmic bytes: Q and K read once,
    pooled means written) and kernel 2 against FP32 FFMA throughput
    (algorithmic FLOPs: 2*d per visible (query block, key block) pair of the
    rank's heads), per layer averaged over the stack, with this run's stage
    times."""
    from paper_2603_10353_b200.head_parallel import rank_segments, rank_shard
    d, bq = 128, 256
    nqb, nkb = n // bq, n // 128
    vis = np.minimum(((np.arange(nqb) + 1) * bq - 1) // 128 + 1, nkb)
    k1_bytes, k2_flops = [], []
    for (q, k, v), plan, b in zip(layers, plans, [None] * len(layers)):
        sh = rank_segments(plan, rank, group, np.zeros(q.shape[0], np.int64)) if split else \
            rank_shard(plan, rank, group, np.zeros(q.shape[0], np.int64))
        hq_r, hkv_r = len(sh.heads), len(sh.kv_heads)
        k1_bytes.append(2.0 * n * d * (hq_r + hkv_r) + 4.0 * d * (nqb * hq_r + nkb * hkv_r))
        k2_flops.append(2.0 * d * hq_r * float(vis.sum()))
    k1_ms, k2_ms = float(stages[0]), float(stages[1])
    out = {}
    if k1_ms > 0:
        gbs = np.mean(k1_bytes) / (k1_ms * 1e-3) / 1e9
        out["k1_pool"] = {"bound": "hbm", "achieved": round(gbs, 1), "peak": peaks.get("hbm_gbs"),
                          "unit": "GB/s", "frac": round(gbs / float(peaks.get("hbm_gbs", 1)), 4),
                          "bytes_per_layer": float(np.mean(k1_bytes)),
                          "bytes_formula": "2*n*d*(Hq+Hkv) bf16 read + 4*d*(nqb*Hq + nkb*Hkv) fp32 written"}
    if k2_ms > 0 and fp32_peak:
        tf = np.mean(k2_flops) / (k2_ms * 1e-3) / 1e12
        out["k2_score_select"] = {"bound": "fp32", "achieved": round(tf, 2),
                                  "peak": fp32_peak["fp32_tflops_burst"], "unit": "TFLOP/s",
                                  "frac": round(tf / fp32_peak["fp32_tflops_burst"], 4),
                                  "flops_per_layer": float(np.mean(k2_flops)),
                                  "flops_formula": "2*d per visible (query block, key block) pair (fp32 FFMA "
                                                   "pooled product; the selection's bisection not counted)",
                                  "peak_source": f"tools/bin/fp32_peak measured in this run ({fp32_peak})"}
    return out


def config_dict(args, budgets_desc, headline="greedy"):
    return {
        "workload": (f"C3: Llama-3-8B-shaped {args.layers}-layer attention stack ({args.q_heads} Q / "
                     f"{args.kv_heads} KV heads, d=128), {args.seq_len}-token causal prefill, "
                     f"block-sparse top-k (128x128 key blocks, 256-row query blocks); every layer has "
                     f"its own inputs, budget table and head plan"),
        "layers": args.layers,
        "seq_len": args.seq_len, "q_heads": args.q_heads, "kv_heads": args.kv_heads,
        "head_dim": 128, "budget_fraction": args.budget_fraction, "budgets": budgets_desc,
        "policy": args.policy,
        "placement": PLACEMENTS[headline],
        "l2": "each layer's inputs (1.5 GiB at 128K) exceed the 126 MB L2; layers run back to back",
    }


# ---------------------------------------------------------------------------
# main arm
# ---------------------------------------------------------------------------

def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch

    import paper_2603_10353_b200 as P
    from paper_2603_10353_b200.head_parallel import rank_segments, rank_shard
    from paper_2603_10353_b200.workload import LayerSpec, make_layer

    global KIND
    KIND = P.selection_kind(args.policy)
    world, rank, local = dist_setup(args.gpus, args.debug_one_device)
    if args.force_gather and world == 1:
        init_single_rank_group(local)
    peaks, peaks_src = load_peaks()
    fp32_peak = measure_fp32_peak() if rank == 0 else None
    hq, n, group = args.q_heads, args.seq_len, args.q_heads // args.kv_heads
    L = max(1, args.layers)
    layers, budgets_l, binfo = [], [], {}
    ctx = P.Context(local)
    for li in range(L):  # distinct layers: own seeds, own budget tables
        spec = LayerSpec(num_q_heads=hq, num_kv_heads=args.kv_heads, seq_len=n,
                         seed=args.seed + 7919 * li)
        q, k, v = make_layer(spec, "cuda")
        b_l, total, info_l = make_budgets(q, k, args, world, rank, pctx=ctx)
        layers.append((q, k, v))
        budgets_l.append(b_l)
        if li == 0:
            binfo = info_l
    torch.cuda.synchronize()
    budgets = budgets_l[0]
    stream = torch.cuda.Stream()

    plans_l = {"greedy": [P.greedy_assign(b, world) for b in budgets_l]}
    if args.assignment_json:  # a head plan written by the reference CLI (partitioner.cpp:288-334)
        la = P.formats.load_assignment(args.assignment_json)
        if la.devices != world or la.device_of_head.size != args.q_heads:
            raise SystemExit(f"{args.assignment_json}: plan for {la.devices} devices / "
                             f"{la.device_of_head.size} heads, run has {world} / {args.q_heads}")
        plans_l["greedy"] = [la.device_of_head.astype(np.int32)] * L
    hp_comm = make_hp_comm(world, rank, local) if (world > 1 or args.force_gather) else None
    if world > 1:
        plans_l["naive"] = [P.naive_assign(b, world) for b in budgets_l]
        plans_l["greedy_tiles"] = [P.greedy_assign(P.tile_costs(b, n), world) for b in budgets_l]
        wcosts = [P.tile_costs(b, n, query_tile_weight=P.api.QUERY_TILE_WEIGHT) for b in budgets_l]
        plans_l["greedy_refined"] = [P.refine_assign(c, world, P.greedy_assign(c, world)) for c in wcosts]
        plans_l["split"] = [P.split_assign(b, world, n, query_tile_weight=P.api.QUERY_TILE_WEIGHT) for b in budgets_l]
    headline = args.placement if world > 1 else "greedy"  # at N = 1 every plan is the whole layer
    results = {}
    for name, plans in plans_l.items():
        shards = []
        for (q, k, v), b, plan in zip(layers, budgets_l, plans):
            if name == "split":
                sh = rank_segments(plan, rank, group, b)
                shards.append(LayerShard(q, k, v, sh, sh.q_block_range, False))
            else:
                sh = rank_shard(plan, rank, group, b)
                shards.append(LayerShard(q, k, v, sh, None, len(sh.heads) == hq))
        sampler = ClockSampler(local) if (name == headline) else None
        if sampler:
            sampler.start()
        ms, stages, launches, _, joules = time_stack(ctx, shards, args.steps, args.warmup, world, stream)
        clocks = sampler.stop() if sampler else None
        flops = sum(ls.flops for ls in shards) / L  # per layer, this rank
        per_rank = allgather_float(ms, world)
        per_rank_k3 = allgather_float(float(stages[2]), world)
        res = {"ms": max(per_rank), "per_rank_ms": per_rank, "stages": stages, "launches": launches,
               "clocks": clocks, "flops_local": flops, "joules": joules,
               "flops_total": sum(allgather_float(flops, world)),
               "bubble": P.barrier(per_rank).bubble_fraction,
               "k3_bubble": P.barrier(per_rank_k3).bubble_fraction,
               "load_imbalance": float(np.mean([
                   (float(p.loads.max() * world / p.loads.sum()) if name == "split"
                    else P.imbalance(b, p, world).imbalance) for b, p in zip(budgets_l, plans)]))}
        if (world > 1 or args.force_gather) and (not DEBUG_GLOO or args.gather == "p2p"):
            if args.gather == "p2p":
                try:
                    res["ms_with_gather"] = time_stack_p2p(ctx, shards, hq, max(2, args.steps // 2), 1, world,
                                                           rank, stream, hp_comm)
                    res["gather_kind"] = "p2p"
                except P.ShplbError as e:  # IPC / peer access unavailable: NCCL all-gather instead
                    torch.cuda.synchronize()
                    res["gather_kind"] = f"nccl (fused p2p unavailable: {e})"
                    res["ms_with_gather"] = time_stack_gathered(ctx, shards, plans, hq, max(2, args.steps // 2),
                                                                1, world, stream, hp_comm)
            else:
                res["gather_kind"] = "nccl"
                res["ms_with_gather"] = time_stack_gathered(ctx, shards, plans, hq, max(2, args.steps // 2),
                                                            1, world, stream, hp_comm)
        if name == headline and not args.no_e2e:
            n_e2e = e2e_layer_budget(shards, args.e2e_layers or L, local_ranks=world)
            e2e_ms, h2d, d2h = time_e2e(ctx, shards[:n_e2e], max(2, args.steps // 2), 1, world, stream)
            res["e2e"] = (max(allgather_float(e2e_ms, world)), h2d, d2h, n_e2e)
        results[name] = res
        del shards
        torch.cuda.empty_cache()

    q, k, v = layers[0]
    dense_ms = None
    if world == 1:  # the paper's "vs full attention" axis: dense causal layer 0 on the same kernel 3
        from paper_2603_10353_b200 import experiments as X
        dense_ms = X._time(lambda: ctx.dense_attention_layer(q, k, v, causal=True), 2)  # current stream
    projection = None
    if world == 1 and args.project_degrees:
        from paper_2603_10353_b200 import experiments as X
        rows = X.measured_sweep(ctx, {n: (q, k, v, budgets)}, args.project_degrees, steps=6)
        projection = {}
        for r in rows:
            projection.setdefault(str(r.degree), {})[r.assigner] = {
                "barrier_ms": round(r.barrier_latency, 3), "bubble": round(r.bubble_fraction, 4),
                "speedup_vs_naive": round(r.speedup_vs_naive, 4),
                "per_rank_ms": [round(x, 3) for x in r.per_rank_ms]}
    g = results[headline]
    flops_total = g["flops_total"]
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            ms_cpu, cores, sample = cpu_reference_sample(q, k, v, budgets, group, args.cpu_seconds)
            cpu = {"value": round(ms_cpu, 1), "unit": "ms", "cores": cores, "kind": "reference",
                   "sample": sample, "cpu_model": cpu_model(),
                   "serial_one_head_ms": round(cpu_reference_serial_head(q, k, v, budgets, group), 1),
                   "serial_one_head_note": ("reference::sparse_attention (serial) on the largest-budget "
                                            "head, 8 rows timed, extrapolated to n rows")}
            # The reference's own table for layer 0 (oracle/tables, written by headbal), if committed:
            # same config as the reference arm iff this run's table equals it.
            if not args.allocation_json and args.profile_kind == "token" and args.policy == "per_query_topk":
                from paper_2603_10353_b200 import calibrate
                hit = committed_reference_table(hq, args.kv_heads, n, args.seed, args.calib_rows,
                                                args.budget_fraction)
                if hit is not None:
                    cpu["reference_table"] = {"file": hit[1], "digest": calibrate.table_digest(hit[0]),
                                              "equal_to_this_run": bool(np.array_equal(hit[0], budgets))}
        except Exception as e:  # reference library missing: report, do not fail the bench
            cpu = {"value": None, "unit": "ms", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {e}"}
    if rank != 0:
        return
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
    k3_ms = float(g["stages"][2])
    k3_tflops = g["flops_local"] / (k3_ms * 1e-3) / 1e12
    traffic, traffic_src = k3_traffic()
    stage_roofs = stage_rooflines(layers, plans_l[headline], rank, group, n, g["stages"], peaks, fp32_peak,
                                  headline == "split")
    # Headline: per-layer time of the stack. At N > 1 it includes every
    # layer's output all-gather (overlapped with the next layer's compute).
    value = g.get("ms_with_gather", g["ms"])
    line = {
        "metric": "attention ms/layer at 128K ctx (max over ranks)",
        "value": round(value, 3), "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(value * args.layers, 3), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded bf16 Q/K/V with per-head temperature, block-local structure)",
        "config": config_dict(args, budgets_desc(args), headline),
        "tflops": round(flops_total / (value * 1e-3) / 1e12, 1),
        "layers_per_step": args.layers,
        "compute_only_ms": round(g["ms"], 3),
        "bubble": round(g["bubble"], 4),
        "per_rank_ms": [round(x, 3) for x in g["per_rank_ms"]],
        "stages_ms": {"k1_pool": round(float(g["stages"][0]), 3),
                      "k2_score_select": round(float(g["stages"][1]), 3),
                      "k3_sparse_fa": round(k3_ms, 3)},
        "budget_table": {"layer0": {"total_tokens": total, "min": int(budgets.min()),
                                    "max": int(budgets.max()),
                                    "blocks_selected": int(P.layer_work(hq, args.kv_heads, n, budgets)[0]),
                                    **binfo},
                         "per_layer_max_min_budget": [[int(b.max()), int(b.min())] for b in budgets_l]},
        "roofline": {"kernel": "k3 block-sparse FA (tcgen05)", "bound": "tensor",
                     "achieved": round(k3_tflops, 1),
                     "peak": peak, "unit": "TFLOP/s", "frac": round(k3_tflops / peak, 4),
                     "peak_source": f"{peaks_src} bf16 dense "
                                    f"{'sustained' if 'bf16_tflops_sustained' in peaks else 'burst'}",
                     "flops_per_launch": g["flops_local"],
                     "flops_formula": "4*d*128*128*computed (query half, key block) tiles, counted "
                                      "from the selection (diagonal tiles counted in full)",
                     "traffic": traffic, "traffic_source": traffic_src},
        "stage_rooflines": stage_roofs,
        "gpu_launches": g["launches"],
        "clocks": g["clocks"],
    }
    if g.get("joules"):
        # This rank's board over the timed region (NVML): under sw_power_cap the
        # layer time is this energy over the cap.
        line["energy"] = {"joules_per_layer": round(g["joules"], 3),
                          "avg_power_w": round(g["joules"] / (g["per_rank_ms"][0] / 1e3), 1),
                          "pj_per_flop": round(g["joules"] / g["flops_local"] * 1e12, 4),
                          "what": "board energy (NVML total-energy counter) over the timed region / "
                                  "layers timed; rank 0's board; pJ per algorithmic FLOP of its layer"}
    if "e2e" in g:
        e2e_ms, h2d, d2h, n_e2e = g["e2e"]
        line["e2e"] = {"value": round(e2e_ms, 3), "unit": "ms", "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h, "layers": n_e2e}
    if world > 1:
        nv = results["naive"]
        def _vg(r):
            return r.get("ms_with_gather", r["ms"])
        line["naive_even_hp"] = {"ms": round(_vg(nv), 3), "compute_only_ms": round(nv["ms"], 3),
                                 "bubble": round(nv["bubble"], 4),
                                 "per_rank_ms": [round(x, 3) for x in nv["per_rank_ms"]],
                                 "load_imbalance": round(nv["load_imbalance"], 4)}
        line["speedup_vs_even_hp"] = round(_vg(nv) / value, 4)
        line["speedup_vs_even_hp_compute_only"] = round(nv["ms"] / g["ms"], 4)
        gr = results["greedy"]
        line["greedy_whole_head"] = {"ms": round(_vg(gr), 3), "compute_only_ms": round(gr["ms"], 3),
                                     "bubble": round(gr["bubble"], 4),
                                     "per_rank_ms": [round(x, 3) for x in gr["per_rank_ms"]],
                                     "speedup_vs_even_hp": round(_vg(nv) / _vg(gr), 4),
                                     "load_imbalance": round(gr["load_imbalance"], 4),
                                     "plan": "the reference's greedy_assign (LPT on budgets), bit-exact"}
        spl = results["split"]
        line["split_subhead"] = {"ms": round(_vg(spl), 3), "compute_only_ms": round(spl["ms"], 3),
                                 "bubble": round(spl["bubble"], 4),
                                 "per_rank_ms": [round(x, 3) for x in spl["per_rank_ms"]],
                                 "speedup_vs_even_hp": round(_vg(nv) / _vg(spl), 4),
                                 "plan": "sub-head balancer (shplb_plan_split), an extension "
                                         "beyond the reference's whole-head greedy_assign"}
        gt = results["greedy_tiles"]
        line["greedy_tile_cost"] = {"ms": round(_vg(gt), 3), "compute_only_ms": round(gt["ms"], 3),
                                    "bubble": round(gt["bubble"], 4),
                                    "per_rank_ms": [round(x, 3) for x in gt["per_rank_ms"]],
                                    "speedup_vs_even_hp": round(_vg(nv) / _vg(gt), 4),
                                    "plan": "greedy_assign on kernel 3's causal tile cost per head "
                                            "(api.tile_costs) instead of budgets (SURVEY a11 extension)"}
        grf = results["greedy_refined"]
        line["greedy_refined"] = {"ms": round(_vg(grf), 3), "compute_only_ms": round(grf["ms"], 3),
                                  "bubble": round(grf["bubble"], 4),
                                  "per_rank_ms": [round(x, 3) for x in grf["per_rank_ms"]],
                                  "speedup_vs_even_hp": round(_vg(nv) / _vg(grf), 4),
                                  "plan": "greedy_assign on tile cost + 4 tiles per visited query tile, refined "
                                          "by whole-head moves / swaps off the most loaded rank "
                                          "(shplb_plan_refine), an extension"}
        line["gather"] = ("every layer's [Hq, n, d] output reassembled on every rank by shplb_gather_segments "
                          "(one NCCL broadcast per output segment from its owner, one group per layer) on a "
                          "communication stream, overlapped with the next layer's compute"
                          if g.get("gather_kind", "nccl").startswith("nccl") else
                          "fused: kernel 3 stores every output row into every rank's [Hq, n, d] buffer over "
                          "NVLink (CUDA IPC peer pointers); one shplb_comm_barrier per layer on a comm stream")
        line["gather_kind"] = g.get("gather_kind")
        line["load_imbalance"] = round(g["load_imbalance"], 4)
    if dense_ms is not None:
        line["dense_comparator"] = {"ms": round(dense_ms, 3), "speedup_sparse_vs_dense": round(dense_ms / value, 3),
                                    "what": "layer 0, every causally visible key block (shplb_dense_attention_layer)"}
    if projection:
        line["per_rank_projection"] = {
            "what": ("layer 0: every rank's shard timed in turn on this GPU (CUDA events, 6 back-to-back calls, "
                     "3 rounds interleaved over the ranks, median per rank); "
                     "barrier = max over ranks, bubble = 1 - mean/max (simulator.cpp:40-44); "
                     "naive = even head parallelism, greedy = S-HPLB greedy_assign, greedy_tiles = greedy_assign on tile cost, greedy_refined = greedy_tiles + "
                     "whole-head local search (shplb_plan_refine), split = sub-head "
                     "balancer; gathers excluded"),
            "degrees": projection}
    line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
