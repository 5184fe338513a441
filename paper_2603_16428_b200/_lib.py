"""ctypes binding to libslf_lce.so (include/slf_lce.h).  Argument marshalling only.

The library is REQUIRED: if it is missing or fails to load, every call raises — there is no
CPU or PyTorch fallback on the product path.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libslf_lce.so")

SLF_OK = 0
STATUS_NAMES = {0: "SLF_OK", 1: "SLF_ERR_ARG", 2: "SLF_ERR_ALIGN", 3: "SLF_ERR_WORKSPACE", 4: "SLF_ERR_CUDA",
                5: "SLF_ERR_UNSUPPORTED", 6: "SLF_ERR_UNIMPLEMENTED", 7: "SLF_ERR_COMM"}
REDUCTIONS = {"sum": 0, "mean": 1, "none": 2}
SCHEDULES = {"auto": 0, "R": 1, "S": 2}

# Every symbol include/slf_lce.h declares.
EXPORTS = ["slf_lce_version", "slf_last_error_string", "slf_lce_workspace_bytes", "slf_lce_plan_describe",
           "slf_lce_fwd_bwd", "slf_lce_fwd", "slf_lce_fwd_shard_stats", "slf_lce_stats_combine", "slf_lce_bwd",
           "slf_lce_status", "slf_debug_gemm", "slf_lce_dx_finalize", "slf_profile_begin", "slf_profile_end",
           "slf_lce_s_plan", "slf_lce_s_begin", "slf_lce_s_chunk_stats", "slf_lce_s_chunk_bwd", "slf_lce_s_end",
           "slf_lce_s_rowstat", "slf_rmsnorm_workspace_bytes", "slf_rmsnorm_fwd", "slf_rmsnorm_bwd",
           "slf_debug_trace_read", "slf_debug_max_active_clusters", "slf_lce_fwd_bwd_ex", "slf_scale_bf16",
           "slf_lce_fwd_bwd_host", "slf_comm_get_unique_id", "slf_comm_init", "slf_comm_init_callbacks",
           "slf_comm_destroy", "slf_comm_rank", "slf_shard_bounds", "slf_lce_sharded_workspace_bytes",
           "slf_lce_sharded_plan_describe", "slf_lce_sharded_chunk_table", "slf_lce_fwd_bwd_sharded", "slf_comm_set_p2p", "slf_comm_status",
           "slf_lce_fwd_bwd_dp", "slf_target_csr_scratch_bytes", "slf_target_csr",
           "slf_rmsnorm_lce_workspace_bytes", "slf_rmsnorm_lce_plan_describe", "slf_rmsnorm_lce_fwd_bwd",
           "slf_scale_bf16_dev", "slf_rowstat_scale",
           # include/slf_adam.h (Layer-Adam, host)
           "slf_adam_last_error_string", "slf_adam_simd_width", "slf_adam_create", "slf_adam_destroy",
           "slf_adam_set_config", "slf_adam_set_params", "slf_adam_get_state", "slf_adam_step_host",
           "slf_adam_step_device_async", "slf_adam_wait"]
PROF_KINDS = ["gemm_stats", "gemm_grad", "gemm_dw", "gemm_dx", "gemm_debug", "prep", "local_combine", "final_combine",
              "dx_finalize", "gemm_group", "combine_transform", "csr", "onehot", "loss_reduce", "rmsnorm", "transpose",
              "comm_allgather", "comm_allreduce"]

_lock = threading.Lock()
_lib = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
INT = ctypes.c_int
F32 = ctypes.c_float
SZ = ctypes.c_size_t


# slf_allgather_fn / slf_allreduce_f32_fn (include/slf_lce.h)
ALLGATHER_FN = ctypes.CFUNCTYPE(INT, P, P, SZ, P, P)
ALLREDUCE_FN = ctypes.CFUNCTYPE(INT, P, SZ, P, P)


class SlfError(RuntimeError):
    pass


def _declare(lib):
    sig = {
        "slf_lce_version": (INT, []),
        "slf_last_error_string": (ctypes.c_char_p, []),
        "slf_lce_workspace_bytes": (SZ, [I64, I64, I64, INT, SZ]),
        "slf_lce_plan_describe": (INT, [I64, I64, I64, INT, SZ, ctypes.c_char_p, SZ]),
        "slf_lce_fwd_bwd": (INT, [P, P, P, I64, I64, I64, I32, INT, F32, P, P, P, P, SZ, INT, SZ, P]),
        "slf_lce_fwd": (INT, [P, P, P, I64, I64, I64, I32, INT, F32, P, P, P, SZ, SZ, P]),
        "slf_lce_fwd_shard_stats": (INT, [P, P, P, I64, I64, I64, I64, I32, P, P, SZ, SZ, P]),
        "slf_lce_stats_combine": (INT, [P, INT, P, I64, I64, I64, I64, I32, INT, F32, P, P, P, SZ, P]),
        "slf_lce_bwd": (INT, [P, P, P, P, I64, I64, I64, F32, P, INT, P, P, SZ, SZ, P]),
        "slf_lce_status": (INT, [P, P, ctypes.POINTER(I32), ctypes.POINTER(I64)]),
        "slf_debug_gemm": (INT, [P, P, P, I64, I64, I64, INT, INT, P]),
        "slf_lce_dx_finalize": (INT, [P, P, P, I64, I64, P]),
        "slf_target_csr_scratch_bytes": (SZ, [I64, I64]),
        "slf_target_csr": (INT, [P, I64, I32, I64, I64, P, P, P, SZ, P]),
        "slf_scale_bf16_dev": (INT, [P, I64, P, P]),
        "slf_rowstat_scale": (INT, [P, P, INT, I64, P, P]),
        "slf_rmsnorm_lce_workspace_bytes": (SZ, [I64, I64, I64, SZ]),
        "slf_rmsnorm_lce_plan_describe": (INT, [I64, I64, I64, SZ, ctypes.c_char_p, SZ]),
        "slf_rmsnorm_lce_fwd_bwd": (INT, [P, P, F32, P, P, I64, I64, I64, I32, INT, F32, P, P, P, P, P, SZ, SZ, P]),
        "slf_profile_begin": (INT, []),
        "slf_profile_end": (INT, [P, P, P, P]),
        "slf_lce_s_plan": (INT, [I64, I64, I64, SZ, ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "slf_lce_s_begin": (INT, [P, I64, I64, I64, I64, I64, I32, INT, P, SZ, SZ, P]),
        "slf_lce_s_chunk_stats": (INT, [P, P, P, I64, I64, I64, I64, I64, I32, I64, P, P, SZ, SZ, P]),
        "slf_lce_s_chunk_bwd": (INT, [P, P, P, I64, I64, I64, I64, I64, I32, INT, F32, I64, P, INT, P, P, INT, P, P,
                                      SZ, SZ, P]),
        "slf_lce_s_end": (INT, [P, I64, I64, I64, INT, F32, P, P, P, SZ, SZ, P]),
        "slf_lce_s_rowstat": (INT, [I64, I64, I64, SZ, P, ctypes.POINTER(P)]),
        "slf_rmsnorm_workspace_bytes": (SZ, [I64, I64]),
        "slf_debug_trace_read": (INT, [P, I64]),
        "slf_scale_bf16": (INT, [P, I64, F32, P]),
        "slf_lce_fwd_bwd_ex": (INT, [P, P, P, I64, I64, I64, I32, INT, F32, P, P, P, P, SZ, INT, SZ,
                                     ctypes.c_uint32, P]),
        "slf_lce_fwd_bwd_host": (INT, [P, P, P, I64, I64, I64, I32, INT, F32, P, P, P, P, P, P, P, SZ, INT, SZ,
                                       ctypes.c_uint32, P]),
        "slf_debug_max_active_clusters": (INT, [INT, ctypes.POINTER(INT)]),
        "slf_rmsnorm_fwd": (INT, [P, P, I64, I64, F32, P, P, P]),
        "slf_rmsnorm_bwd": (INT, [P, P, P, P, I64, I64, P, P, P, SZ, P]),
        "slf_comm_get_unique_id": (INT, [P]),
        "slf_comm_init": (INT, [ctypes.POINTER(P), P, INT, INT, INT]),
        "slf_comm_init_callbacks": (INT, [ctypes.POINTER(P), INT, INT, ALLGATHER_FN, ALLREDUCE_FN, P]),
        "slf_comm_destroy": (INT, [P]),
        "slf_comm_rank": (INT, [P, ctypes.POINTER(INT), ctypes.POINTER(INT)]),
        "slf_comm_set_p2p": (INT, [P, INT]),
        "slf_comm_status": (INT, [P, ctypes.POINTER(I32)]),
        "slf_shard_bounds": (INT, [I64, INT, INT, ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "slf_lce_sharded_workspace_bytes": (SZ, [I64, I64, I64, INT, INT, SZ]),
        "slf_lce_sharded_plan_describe": (INT, [I64, I64, I64, INT, INT, SZ, ctypes.c_char_p, SZ]),
        "slf_lce_sharded_chunk_table": (INT, [I64, I64, I64, INT, INT, SZ, P, I64, ctypes.POINTER(I64)]),
        "slf_lce_fwd_bwd_sharded": (INT, [P, P, P, I64, I64, I64, I32, INT, F32, P, P, P, P, SZ, SZ, P, P]),
        "slf_lce_fwd_bwd_dp": (INT, [P, P, P, I64, I64, I64, I32, INT, F32, P, P, P, P, SZ, INT, SZ, INT, P, P]),
        "slf_adam_last_error_string": (ctypes.c_char_p, []),
        "slf_adam_simd_width": (INT, []),
        "slf_adam_create": (INT, [ctypes.POINTER(P), I64, P]),
        "slf_adam_destroy": (INT, [P]),
        "slf_adam_set_config": (INT, [P, P]),
        "slf_adam_set_params": (INT, [P, P, P]),
        "slf_adam_get_state": (INT, [P, P, P, P, ctypes.POINTER(I64)]),
        "slf_adam_step_host": (INT, [P, P, F32, P]),
        "slf_adam_step_device_async": (INT, [P, P, F32, P, P]),
        "slf_adam_wait": (INT, [P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args


def lib():
    """Load libslf_lce.so (built in-tree by paper_2603_16428_b200.build / __graft_entry__.build)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(SO_PATH):
                    raise SlfError(f"{SO_PATH} is missing: run `python -m paper_2603_16428_b200.build` "
                                   "(there is no fallback path)")
                l = ctypes.CDLL(SO_PATH)
                _declare(l)
                _lib = l
    return _lib


def check(status: int, what: str):
    if status != SLF_OK:
        msg = lib().slf_last_error_string().decode(errors="replace")
        raise SlfError(f"{what} failed with {STATUS_NAMES.get(status, status)}: {msg}")
