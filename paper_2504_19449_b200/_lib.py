"""ctypes binding of include/rsparse_b200.h (the product's C ABI).

Loading fails loudly when librsparse_b200.so is missing: there is no CPU or
eager-PyTorch fallback for any operator in this package.
"""
from __future__ import annotations

import ctypes as ct
import os

from .build import LIB

RSP_OK, RSP_E_NUMERIC, RSP_E_USAGE, RSP_E_IO, RSP_E_CUDA, RSP_E_UNSUPPORTED = range(6)
RSP_F32, RSP_BF16, RSP_F64 = 0, 1, 2
RSP_MEM_HOST, RSP_MEM_DEVICE = 0, 1
RSP_W_ROW_MAJOR, RSP_W_COL_MAJOR = 0, 1

# Every symbol include/rsparse_b200.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "rsp_abi_version", "rsp_last_error", "rsp_keep_count", "rsp_plan_for", "rsp_shard_rows",
    "rsp_linear_create", "rsp_linear_destroy", "rsp_linear_info_get",
    "rsp_linear_workspace_size", "rsp_workspace_init", "rsp_linear_forward",
    "rsp_linear_forward_host", "rsp_linear_dense_forward", "rsp_gather_matvec",
    "rsp_linear_selected", "rsp_linear_io_cost", "rsp_linear_export",
    "rsp_top_k_by_magnitude", "rsp_threshold_sparsify", "rsp_stack_create", "rsp_stack_create_ex",
    "rsp_stack_launch", "rsp_stack_destroy", "rsp_device_sm_count", "rsp_debug_forward_trace",
    "rsp_debug_stack_trace", "rsp_debug_batch_trace", "rsp_debug_set_batch_trace", "rsp_stack_io_spans",
    "rsp_stack_launch_host", "rsp_stack_create_ops", "rsp_stack_create_spec", "rsp_rspl_read", "rsp_linear_load_rspl", "rsp_linear_save_rspl", "rsp_linear_components",
    "rsp_aggregate_scores", "rsp_select_components", "rsp_split_factors", "rsp_linear_set_components",
    "rsp_stack_exchange_words", "rsp_stack_grids", "rsp_ipc_alloc", "rsp_ipc_free", "rsp_ipc_export",
    "rsp_ipc_open", "rsp_ipc_close", "rsp_stack_launch_direct",
]
RSP_IPC_HANDLE_BYTES = 64


class LinearDesc(ct.Structure):
    _fields_ = [
        ("m_in", ct.c_uint32), ("m_out", ct.c_uint32), ("rank", ct.c_uint32),
        ("keep_fraction", ct.c_double), ("k_override", ct.c_int64),
        ("weight_dtype", ct.c_int), ("src_dtype", ct.c_int), ("src_memory", ct.c_int),
        ("w_layout", ct.c_int), ("w", ct.c_void_p), ("a_r", ct.c_void_p), ("b_r", ct.c_void_p),
        ("device", ct.c_int), ("shard_rank", ct.c_uint32), ("shard_count", ct.c_uint32),
        ("flags", ct.c_uint32),
    ]


RSP_FLAG_DETERMINISTIC = 1
RSP_FLAG_BATCH_TCGEN05 = 2
RSP_XOP_NONE, RSP_XOP_SILU_GATE = 0, 1
RSP_PATH_PERSISTENT, RSP_PATH_BATCH_MMA, RSP_PATH_BATCH_TCGEN05, RSP_PATH_DETERMINISTIC = 1, 2, 4, 8


class LinearInfo(ct.Structure):
    _fields_ = [
        ("m_in", ct.c_uint32), ("m_out", ct.c_uint32), ("rank", ct.c_uint32), ("k", ct.c_uint32),
        ("row_begin", ct.c_uint32), ("row_end", ct.c_uint32), ("m_pad", ct.c_uint32),
        ("r_pad", ct.c_uint32), ("col_tiles", ct.c_uint32), ("k_splits", ct.c_uint32),
        ("grid", ct.c_uint32), ("smem_bytes", ct.c_uint32), ("weight_dtype", ct.c_int),
        ("device_bytes", ct.c_uint64), ("path", ct.c_uint32),
    ]


class IoReport(ct.Structure):
    _fields_ = [
        ("dense_bytes", ct.c_uint64), ("touched_bytes", ct.c_uint64),
        ("relative_cost", ct.c_double), ("kernel_weight_bytes", ct.c_uint64),
        ("kernel_total_bytes", ct.c_uint64), ("dense_weight_bytes", ct.c_uint64),
    ]


class StackSpec(ct.Structure):
    _fields_ = [
        ("layers", ct.POINTER(ct.c_void_p)), ("count", ct.c_uint32), ("x_devs", ct.POINTER(ct.c_void_p)),
        ("x_dtype", ct.c_int), ("y_devs", ct.POINTER(ct.c_void_p)), ("dense", ct.c_int),
        ("wait_prev", ct.POINTER(ct.c_uint8)), ("x_ops", ct.POINTER(ct.c_uint8)), ("npeer", ct.c_uint32),
        ("y_peers", ct.POINTER(ct.c_void_p)), ("max_ctas", ct.c_uint32),
        ("xrank", ct.c_uint32), ("xself", ct.c_uint32), ("xctr", ct.POINTER(ct.c_void_p)),
    ]


class RsplHeader(ct.Structure):
    _fields_ = [("m_in", ct.c_uint32), ("m_out", ct.c_uint32), ("rank", ct.c_uint32),
                ("kept_width", ct.c_uint32), ("keep_fraction", ct.c_double)]


class RspError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[rsp status {status}] {msg}")
        self.status = status


class UsageError(RspError, ValueError):
    """rsparse::usage_error (include/rsparse/errors.hpp:10-12)."""


class NumericError(RspError):
    """rsparse::numeric_error (errors.hpp:14-17)."""


class IoError(RspError):
    """rsparse::io_error (errors.hpp:19-22)."""


class CudaError(RspError):
    pass


_ERR = {RSP_E_USAGE: UsageError, RSP_E_NUMERIC: NumericError, RSP_E_IO: IoError,
        RSP_E_CUDA: CudaError}

_lib = None


def lib() -> ct.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        raise ImportError(f"{LIB} is missing: run `python -m paper_2504_19449_b200.build` "
                          "(no CPU fallback exists for this operator)")
    L = ct.CDLL(LIB)
    vp, u32, i32p = ct.c_void_p, ct.c_uint32, ct.POINTER(ct.c_int32)
    sig = {
        "rsp_abi_version": (ct.c_int, []),
        "rsp_last_error": (ct.c_char_p, []),
        "rsp_keep_count": (ct.c_int, [ct.c_double, u32, ct.POINTER(u32)]),
        "rsp_plan_for": (ct.c_int, [ct.c_double, ct.c_double, u32, u32,
                                    ct.POINTER(ct.c_double), ct.POINTER(u32)]),
        "rsp_shard_rows": (ct.c_int, [u32, u32, u32, ct.POINTER(u32), ct.POINTER(u32)]),
        "rsp_linear_create": (ct.c_int, [ct.POINTER(LinearDesc), ct.POINTER(vp)]),
        "rsp_linear_destroy": (None, [vp]),
        "rsp_linear_info_get": (ct.c_int, [vp, ct.POINTER(LinearInfo)]),
        "rsp_linear_workspace_size": (ct.c_size_t, [vp, u32]),
        "rsp_workspace_init": (ct.c_int, [vp, ct.c_size_t, vp]),
        "rsp_linear_forward": (ct.c_int, [vp, vp, ct.c_int, vp, u32, vp, ct.c_size_t, vp]),
        "rsp_linear_forward_host": (ct.c_int, [vp, vp, ct.c_int, vp, ct.c_int, u32]),
        "rsp_linear_dense_forward": (ct.c_int, [vp, vp, ct.c_int, vp, vp, ct.c_size_t, vp]),
        "rsp_gather_matvec": (ct.c_int, [vp, vp, ct.c_int, ct.POINTER(ct.c_int64), u32, vp,
                                         ct.POINTER(ct.c_uint64), vp]),
        "rsp_linear_selected": (ct.c_int, [vp, vp, ct.c_int, i32p, ct.POINTER(u32)]),
        "rsp_linear_io_cost": (ct.c_int, [vp, ct.POINTER(IoReport)]),
        "rsp_linear_export": (ct.c_int, [vp, ct.c_int, ct.POINTER(ct.c_double)]),
        "rsp_top_k_by_magnitude": (ct.c_int, [vp, ct.c_int, u32, u32, vp, vp, vp]),
        "rsp_threshold_sparsify": (ct.c_int, [vp, ct.c_int, u32, ct.c_double, vp, vp,
                                              ct.POINTER(u32), vp]),
        "rsp_stack_create": (ct.c_int, [ct.POINTER(vp), u32, ct.POINTER(vp), ct.c_int,
                                        ct.POINTER(vp), ct.c_int, ct.POINTER(vp)]),
        "rsp_stack_create_ex": (ct.c_int, [ct.POINTER(vp), u32, ct.POINTER(vp), ct.c_int,
                                           ct.POINTER(vp), ct.c_int, ct.POINTER(ct.c_uint8), ct.POINTER(vp)]),
        "rsp_stack_create_ops": (ct.c_int, [ct.POINTER(vp), u32, ct.POINTER(vp), ct.c_int,
                                            ct.POINTER(vp), ct.c_int, ct.POINTER(ct.c_uint8), ct.POINTER(ct.c_uint8),
                                            ct.POINTER(vp)]),
        "rsp_stack_create_spec": (ct.c_int, [ct.POINTER(StackSpec), ct.POINTER(vp)]),
        "rsp_stack_launch": (ct.c_int, [vp, vp]),
        "rsp_stack_destroy": (None, [vp]),
        "rsp_device_sm_count": (ct.c_int, [ct.c_int]),
        "rsp_stack_exchange_words": (ct.c_size_t, [ct.c_uint32]),
        "rsp_stack_grids": (ct.c_int, [vp, ct.POINTER(ct.c_uint32), ct.c_uint32]),
        "rsp_stack_launch_direct": (ct.c_int, [vp, vp]),
        "rsp_ipc_alloc": (ct.c_int, [ct.c_int, ct.c_size_t, ct.POINTER(vp)]),
        "rsp_ipc_free": (ct.c_int, [vp]),
        "rsp_ipc_export": (ct.c_int, [vp, ct.c_char_p]),
        "rsp_ipc_open": (ct.c_int, [ct.c_int, ct.c_char_p, ct.POINTER(vp)]),
        "rsp_ipc_close": (ct.c_int, [vp]),
        "rsp_debug_forward_trace": (ct.c_int, [vp, vp, ct.c_int, vp, vp, ct.c_size_t, vp, ct.c_int, vp]),
        "rsp_debug_stack_trace": (ct.c_int, [vp, vp, ct.POINTER(u32), vp]),
        "rsp_debug_batch_trace": (ct.c_int, [vp, u32]),
        "rsp_debug_set_batch_trace": (ct.c_int, [ct.c_int]),
        "rsp_stack_io_spans": (ct.c_int, [vp, ct.POINTER(ct.c_size_t), ct.POINTER(ct.c_size_t)]),
        "rsp_stack_launch_host": (ct.c_int, [vp, vp, ct.c_size_t, vp, ct.c_size_t, vp]),
        "rsp_rspl_read": (ct.c_int, [ct.c_char_p, ct.POINTER(RsplHeader), vp, vp, vp, vp]),
        "rsp_linear_load_rspl": (ct.c_int, [ct.c_char_p, ct.POINTER(LinearDesc), ct.POINTER(vp)]),
        "rsp_linear_save_rspl": (ct.c_int, [vp, ct.c_char_p]),
        "rsp_linear_components": (ct.c_int, [vp, ct.POINTER(u32)]),
        "rsp_aggregate_scores": (ct.c_int, [vp, u32, u32, vp, vp, u32, vp, vp]),
        "rsp_select_components": (ct.c_int, [vp, u32, u32, u32, vp, vp, vp]),
        "rsp_split_factors": (ct.c_int, [vp, u32, u32, vp, vp, u32, vp, u32, vp, vp, vp]),
        "rsp_linear_set_components": (ct.c_int, [vp, ct.POINTER(u32), u32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int, what: str = "") -> None:
    if status == RSP_OK:
        return
    msg = lib().rsp_last_error().decode(errors="replace")
    raise _ERR.get(status, RspError)(status, f"{what}: {msg}" if what else msg)
