"""bench.py end to end at small size: the N=1 line keeps the driver's contract,
and the N>1 head-parallel path (both ranks on cuda:0 over gloo,
--debug-one-device; timings not meaningful) runs every plan, the fused gather
and the host-buffer e2e leg and prints one line from rank 0 only."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = ["--seq-len", "8192", "--layers", "2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
         "--calib-rows", "16"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _lines(out):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def test_bench_single_gpu_contract():
    r = subprocess.run([sys.executable, "bench.py", *SMALL], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    (line,) = _lines(r.stdout)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks",
                "gpu_launches"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["higher_is_better"] is False
    assert line["gpu_launches"] == 3 * 2  # pool q+k, score+select, attention per layer (8K: one key chunk)
    assert 0 < line["roofline"]["frac"] < 1.2
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0


def test_bench_two_ranks_debug_path():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--debug-one-device", *SMALL]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    (line,) = _lines(r.stdout)  # rank 0 only
    assert line["n_gpus"] == 2 and len(line["per_rank_ms"]) == 2
    assert line["gather_kind"] == "p2p"
    assert "sub-head balancer" in line["config"]["placement"]
    for k in ("naive_even_hp", "greedy_whole_head", "greedy_tile_cost", "greedy_refined", "split_subhead"):
        assert line[k]["ms"] > 0, k
    assert line["e2e"]["value"] > 0


def test_cpp_host_driver():
    """tools/bench_layer (C++ over the C ABI only): profile -> max-min table ->
    layer call on device and host buffers, one JSON line."""
    binary = os.path.join(ROOT, "tools", "bin", "bench_layer")
    if not os.path.exists(binary):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools")], check=True)
    r = subprocess.run([binary, "8192", "2", "2"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    (line,) = _lines(r.stdout)
    assert line["tool"] == "bench_layer" and line["launches_per_layer"] == 3
    assert 0 < line["device_ms_per_layer"] < line["host_buffers_ms_per_layer"] * 10
