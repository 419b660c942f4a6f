"""ctypes binding of libshplb.so (the C ABI declared in include/shplb.h).

The shared library is built in-tree by ``paper_2603_10353_b200/csrc/Makefile``
(``build()`` below, or ``__graft_entry__.build()``). There is no fallback: if
the library is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SHPLB_LIB") or os.path.join(PKG_DIR, "lib", "libshplb.so")
CSRC_DIR = os.path.join(PKG_DIR, "csrc")

# Every symbol include/shplb.h declares (checked by the CPU test suite).
EXPORTS = (
    "shplb_last_error", "shplb_version",
    "shplb_uniform_allocate", "shplb_maxmin_allocate", "shplb_recovery_at", "shplb_budget_for_recovery",
    "shplb_profile_curves_host", "shplb_profile_curves",
    "shplb_profile_curves_host_kind", "shplb_profile_curves_kind", "shplb_profile_curves_block",
    "shplb_plan_naive", "shplb_plan_greedy", "shplb_plan_optimal", "shplb_plan_refine", "shplb_plan_split", "shplb_plan_split_weighted", "shplb_imbalance",
    "shplb_simulate", "shplb_barrier",
    "shplb_ctx_create", "shplb_ctx_destroy", "shplb_ctx_launch_count",
    "shplb_ctx_set_timing", "shplb_ctx_read_timing",
    "shplb_block_scores", "shplb_select_blocks", "shplb_block_sparse_attention",
    "shplb_sparse_attention_layer", "shplb_sparse_attention_layer_host", "shplb_dense_attention_layer",
    "shplb_sparse_attention_layer_host_async",
    "shplb_last_selection", "shplb_copy_last_selection",
    "shplb_layer_work", "shplb_last_selection_work",
    "shplb_ipc_handle", "shplb_ipc_open", "shplb_ipc_close",
    "shplb_nccl_get_unique_id", "shplb_nccl_comm_init", "shplb_nccl_comm_destroy", "shplb_nccl_comm_size",
    "shplb_gather_segments", "shplb_gather_heads", "shplb_comm_barrier",
)

SHPLB_OK = 0
SHPLB_INVALID_ARGUMENT = 1
SHPLB_RUNTIME_ERROR = 2
SHPLB_LOGIC_ERROR = 3
SHPLB_CUDA_ERROR = 4
SHPLB_NOT_SUPPORTED = 5
SHPLB_NCCL_ERROR = 6


class ShplbError(RuntimeError):
    """Base class of errors raised through the C ABI."""


class InvalidArgument(ShplbError, ValueError):
    """The reference's std::invalid_argument (bad shapes, budgets, totals)."""


class ShplbRuntimeError(ShplbError):
    """The reference's std::runtime_error (I/O and file-schema errors)."""


class LogicError(ShplbError):
    """The reference's std::logic_error."""


class CudaError(ShplbError):
    """A CUDA runtime/driver failure."""


class NotSupported(ShplbError, NotImplementedError):
    """A shape or policy the sm_100a kernels do not implement."""


class NcclError(ShplbError):
    """An NCCL failure (or libnccl.so.2 not loadable) in a multi-rank call."""


_ERRORS = {
    SHPLB_INVALID_ARGUMENT: InvalidArgument,
    SHPLB_RUNTIME_ERROR: ShplbRuntimeError,
    SHPLB_LOGIC_ERROR: LogicError,
    SHPLB_CUDA_ERROR: CudaError,
    SHPLB_NOT_SUPPORTED: NotSupported,
    SHPLB_NCCL_ERROR: NcclError,
}


class LayerShape(C.Structure):
    """shplb_layer_shape."""
    _fields_ = [
        ("num_q_heads", C.c_int32),
        ("num_kv_heads", C.c_int32),
        ("seq_len", C.c_int64),
        ("head_dim", C.c_int32),
        ("block_q", C.c_int32),
        ("block_k", C.c_int32),
        ("causal", C.c_int32),
        ("kind", C.c_int32),
        ("validate", C.c_int32),
        ("kv_head_of_q", C.c_void_p),
        ("q_block_range", C.c_void_p),
        ("out_peers", C.c_void_p),
        ("n_out_peers", C.c_int32),
        ("out_head_of_q", C.c_void_p),
        ("out_heads_total", C.c_int32),
    ]


class MaxminDiag(C.Structure):
    """shplb_maxmin_diag."""
    _fields_ = [
        ("transfers", C.c_int64),
        ("hit_iteration_cap", C.c_int32),
        ("off_grid_evaluations", C.c_int64),
        ("min_recovery_start", C.c_double),
        ("min_recovery_end", C.c_double),
    ]


def build(verbose: bool = False) -> None:
    """Compile libshplb.so for sm_100a in-tree (nvcc + g++)."""
    r = subprocess.run(["make", "-C", CSRC_DIR, "-j8"], capture_output=True, text=True)
    if verbose or r.returncode != 0:
        print(r.stdout[-4000:], r.stderr[-4000:])
    if r.returncode != 0:
        raise RuntimeError("building libshplb.so failed")


_lib = None


def lib() -> C.CDLL:
    """Load libshplb.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FileNotFoundError(
            f"{LIB_PATH} not found: the CUDA extension is not built "
            "(run paper_2603_10353_b200._native.build() or __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    P = C.POINTER
    L.shplb_last_error.restype = C.c_char_p
    L.shplb_version.restype = C.c_char_p
    L.shplb_uniform_allocate.argtypes = [i64, i64, i64, i64, vp]
    L.shplb_maxmin_allocate.argtypes = [i32, i64, vp, vp, vp, i64, i64, i64, i64, vp,
                                        P(MaxminDiag)]
    L.shplb_recovery_at.argtypes = [i64, vp, vp, i64, P(f64)]
    L.shplb_budget_for_recovery.argtypes = [i64, vp, vp, i64, f64, P(i64)]
    L.shplb_profile_curves_host.argtypes = [vp, vp, i32, i32, i64, i64, i32, vp, i64, vp]
    L.shplb_profile_curves.argtypes = [vp, vp, vp, i32, i32, i64, i64, i32, vp, i64, vp, vp]
    L.shplb_profile_curves_host_kind.argtypes = [vp, vp, i32, i32, i64, i64, i32, vp, i64, i32, vp]
    L.shplb_profile_curves_kind.argtypes = [vp, vp, vp, i32, i32, i64, i64, i32, vp, i64, i32, vp, vp]
    L.shplb_profile_curves_block.argtypes = [vp, vp, vp, i32, i32, i64, i32, i32, i32, vp, i64, vp, i64, vp, vp]
    L.shplb_plan_naive.argtypes = [vp, i32, i32, i32, vp]
    L.shplb_plan_greedy.argtypes = [vp, i32, i32, vp]
    L.shplb_plan_optimal.argtypes = [vp, i32, i32, vp]
    L.shplb_plan_refine.argtypes = [vp, i32, i32, vp, vp]
    L.shplb_plan_split.argtypes = [vp, i32, i64, i32, i32, i32, i32, vp, vp, vp, vp, P(i32), vp]
    L.shplb_plan_split_weighted.argtypes = [vp, i32, i64, i32, i32, i32, i64, i32, vp, vp, vp, vp, P(i32), vp]
    L.shplb_imbalance.argtypes = [vp, i32, vp, i32, vp, P(i64), P(f64), P(i32)]
    L.shplb_simulate.argtypes = [vp, i32, f64, f64, vp, P(f64), P(f64)]
    L.shplb_barrier.argtypes = [vp, i32, P(f64), P(f64)]
    L.shplb_ctx_create.argtypes = [C.c_int, P(vp)]
    L.shplb_ctx_destroy.argtypes = [vp]
    L.shplb_ctx_launch_count.argtypes = [vp]
    L.shplb_ctx_launch_count.restype = i64
    L.shplb_ctx_set_timing.argtypes = [vp, C.c_int]
    L.shplb_ctx_read_timing.argtypes = [vp, vp, C.c_int, P(C.c_int)]
    L.shplb_block_scores.argtypes = [vp, P(LayerShape), vp, vp, vp, vp]
    L.shplb_select_blocks.argtypes = [vp, P(LayerShape), vp, vp, i64, vp, vp, vp]
    L.shplb_block_sparse_attention.argtypes = [vp, P(LayerShape), vp, vp, vp, vp, vp, i64, vp,
                                               vp]
    L.shplb_sparse_attention_layer.argtypes = [vp, P(LayerShape), vp, vp, vp, vp, vp, vp]
    L.shplb_sparse_attention_layer_host.argtypes = [vp, P(LayerShape), vp, vp, vp, vp, vp, vp]
    L.shplb_dense_attention_layer.argtypes = [vp, P(LayerShape), vp, vp, vp, vp, vp]
    L.shplb_sparse_attention_layer_host_async.argtypes = [vp, P(LayerShape), vp, vp, vp, vp, vp, vp]
    L.shplb_ipc_handle.argtypes = [vp, vp, C.c_size_t]
    L.shplb_ipc_open.argtypes = [C.c_int, vp, C.c_size_t, P(vp)]
    L.shplb_ipc_close.argtypes = [C.c_int, vp]
    L.shplb_nccl_get_unique_id.argtypes = [vp, C.c_size_t]
    L.shplb_nccl_comm_init.argtypes = [C.c_int, i32, i32, vp, C.c_size_t, P(vp)]
    L.shplb_nccl_comm_destroy.argtypes = [vp]
    L.shplb_nccl_comm_size.argtypes = [vp, P(i32), P(i32)]
    L.shplb_gather_segments.argtypes = [vp, vp, vp, i32, i32, i64, i32, vp, vp, vp]
    L.shplb_gather_heads.argtypes = [vp, vp, i32, i64, i32, vp, vp, vp, vp]
    L.shplb_comm_barrier.argtypes = [vp, vp]
    L.shplb_last_selection.argtypes = [vp, P(vp), P(vp), P(i64)]
    L.shplb_copy_last_selection.argtypes = [vp, vp, i64, vp, i64, vp]
    L.shplb_layer_work.argtypes = [P(LayerShape), vp, P(i64), P(f64)]
    L.shplb_last_selection_work.argtypes = [vp, P(i64), P(f64)]
    _lib = L
    return L


def check(status: int) -> None:
    """Translate a shplb_status into the matching Python exception."""
    if status != SHPLB_OK:
        msg = lib().shplb_last_error().decode()
        raise _ERRORS.get(status, ShplbError)(msg)
