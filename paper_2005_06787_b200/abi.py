"""ctypes mirror of the C ABI in include/stn_exec.h.

This is the binding a Python caller of the executor uses (the same stub is
shown in INTEGRATION.md). It loads the in-tree ``libstn_exec.so`` and fails
loudly when it is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libstn_exec.so")

STN_SINGLE, STN_DOUBLE = 0, 1
STN_MODE_FAST, STN_MODE_EXACT = 0, 1

# stn_status: 1..19 mirror stemtn::ErrorKind (errors.hpp:8-30) as index + 1.
ERROR_KINDS = [
    "MalformedNetwork", "CapExceeded", "OpenEdgeSliced", "IndexOutOfRange", "MissingParams",
    "SyntaxError", "InvariantViolation", "QubitCoverage", "LayoutTooSmall", "Infeasible",
    "EdgeNotFound", "SchemaError", "Stuck", "HashMismatch", "WidthExceedsBudget",
    "SubtaskFailure", "MissingResult", "ChecksumMismatch", "EmptySamples",
]
EXECUTOR_ERRORS = {100: "CudaError", 101: "InvalidArgument", 102: "OutOfMemory",
                   103: "NoDevice", 104: "IOError"}


def status_name(code: int) -> str:
    if 1 <= code <= len(ERROR_KINDS):
        return ERROR_KINDS[code - 1]
    return EXECUTOR_ERRORS.get(code, "Unknown")


class StnError(RuntimeError):
    """Mirrors stemtn::Error (errors.hpp:60-70): message prefixed by the kind."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.kind = status_name(status)
        super().__init__(message if message.startswith(self.kind) else f"{self.kind}: {message}")


class StepDesc(C.Structure):
    _fields_ = [
        ("node", C.c_int32), ("lhs", C.c_int32), ("rhs", C.c_int32), ("is_branch", C.c_int32),
        ("nd", C.c_int32), ("nm", C.c_int32), ("nk", C.c_int32), ("nn", C.c_int32),
        ("D", C.c_int64), ("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64),
        ("mults", C.c_uint64),
        ("lrank", C.c_int32), ("rrank", C.c_int32), ("orank", C.c_int32),
        ("lperm", C.POINTER(C.c_int32)), ("rperm", C.POINTER(C.c_int32)),
        ("operm", C.POINTER(C.c_int32)), ("out_dims", C.POINTER(C.c_int32)),
    ]


class LeafDesc(C.Structure):
    _fields_ = [
        ("node", C.c_int32), ("vertex", C.c_int32), ("rank", C.c_int32),
        ("dims", C.POINTER(C.c_int32)), ("values", C.POINTER(C.c_double)),
        ("n_sliced", C.c_int32), ("sliced_axis", C.POINTER(C.c_int32)),
        ("sliced_index", C.POINTER(C.c_int32)),
        ("perm_rank", C.c_int32), ("perm", C.POINTER(C.c_int32)),
    ]


class PlanDesc(C.Structure):
    _fields_ = [
        ("precision", C.c_int32), ("merge_min_dim", C.c_int32), ("n_nodes", C.c_int32),
        ("root", C.c_int32), ("identity", C.c_uint64), ("subtasks", C.c_uint64),
        ("merged_groups", C.c_int32), ("exec_cw", C.c_int32),
        ("n_sliced", C.c_int32), ("sliced_dims", C.POINTER(C.c_int32)),
        ("n_open", C.c_int32), ("n_steps", C.c_int32), ("steps", C.POINTER(StepDesc)),
        ("n_leaves", C.c_int32), ("leaves", C.POINTER(LeafDesc)),
    ]


class SubtaskInfo(C.Structure):
    _fields_ = [("assignment", C.c_uint64), ("step_count", C.c_int32), ("mults", C.c_uint64),
                ("peak_elements", C.c_uint64)]


class RunReport(C.Structure):
    _fields_ = [
        ("subtasks", C.c_uint64), ("mult_count", C.c_uint64), ("branch_mults", C.c_uint64),
        ("wall_seconds", C.c_double), ("p50_ms", C.c_double), ("p90_ms", C.c_double),
        ("p99_ms", C.c_double), ("parallelism", C.c_int32), ("precision", C.c_int32),
        ("peak_elements", C.c_uint64), ("merged_groups", C.c_int32),
        ("slices_per_batch", C.c_int32), ("kernel_launches", C.c_int32),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("identity", C.c_uint64), ("subtasks", C.c_uint64), ("n_sliced", C.c_int32),
        ("out_rank", C.c_int32), ("out_elements", C.c_int64), ("out_dims", C.c_int32 * 64),
        ("per_slice_steps", C.c_int32), ("per_slice_mults", C.c_uint64),
        ("branch_mults", C.c_uint64), ("peak_elements", C.c_uint64),
        ("arena_bytes_per_slice", C.c_uint64), ("cache_bytes", C.c_uint64),
        ("steps_tensor_core", C.c_int32), ("steps_absorb", C.c_int32),
        ("steps_generic", C.c_int32), ("sweeps", C.c_int32), ("steps_in_sweeps", C.c_int32),
    ]


KERNEL_KINDS = ["generic", "absorb", "gemm_simt", "gemm_tc", "permute", "leaf", "root",
                "absorb_tc", "sweep"]


class KernelProfile(C.Structure):
    _fields_ = [("kind", C.c_int32), ("launches", C.c_int32), ("ms", C.c_double),
                ("bytes", C.c_double), ("flops", C.c_double)]


class StepProfile(C.Structure):
    _fields_ = [("step", C.c_int32), ("kind", C.c_int32), ("M", C.c_int64), ("N", C.c_int64),
                ("K", C.c_int64), ("launches", C.c_int32), ("ms", C.c_double),
                ("bytes", C.c_double), ("flops", C.c_double)]


# Every symbol include/stn_exec.h declares, with its ctypes signature.
_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
SIGNATURES = {
    "stn_version": (C.c_char_p, []),
    "stn_abi_version": (C.c_int, []),
    "stn_last_error": (C.c_char_p, []),
    "stn_status_name": (C.c_char_p, [C.c_int]),
    "stn_plan_load": (C.c_int, [C.c_char_p, C.POINTER(C.POINTER(PlanDesc))]),
    "stn_plan_save": (C.c_int, [C.POINTER(PlanDesc), C.c_char_p]),
    "stn_plan_desc_free": (None, [C.POINTER(PlanDesc)]),
    "stn_plan_create": (C.c_int, [C.POINTER(PlanDesc), C.c_int, C.c_int, _PP]),
    "stn_plan_destroy": (C.c_int, [_P]),
    "stn_plan_get_info": (C.c_int, [_P, C.POINTER(PlanInfo)]),
    "stn_plan_set_leaf_values": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_double), C.c_int64]),
    "stn_plan_set_max_batch": (C.c_int, [_P, C.c_int32]),
    "stn_plan_set_streams": (C.c_int, [_P, C.c_int32]),
    "stn_plan_set_profiling": (C.c_int, [_P, C.c_int]),
    "stn_plan_get_profile": (C.c_int, [_P, C.POINTER(KernelProfile)]),
    "stn_plan_reset_profile": (C.c_int, [_P]),
    "stn_plan_get_step_profile": (C.c_int, [_P, C.POINTER(StepProfile), C.c_int32,
                                            C.POINTER(C.c_int32)]),
    "stn_cache_build": (C.c_int, [_P, _P, _PP]),
    "stn_cache_destroy": (C.c_int, [_P]),
    "stn_cache_info": (C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_uint64)]),
    "stn_run_subtask": (C.c_int, [_P, C.c_uint64, _P, _P, C.POINTER(C.c_double),
                                  C.POINTER(SubtaskInfo)]),
    "stn_run_subtask_digits": (C.c_int, [_P, C.POINTER(C.c_int32), _P, _P,
                                         C.POINTER(C.c_double), C.POINTER(SubtaskInfo)]),
    "stn_run_slices": (C.c_int, [_P, _P, C.c_uint64, C.c_uint64, _P, _P, _P]),
    "stn_run_slices_digits": (C.c_int, [_P, _P, C.POINTER(C.c_int32), C.c_uint64, _P, _P, _P]),
    "stn_run_scheme": (C.c_int, [_P, C.c_int, C.POINTER(C.c_double), C.POINTER(RunReport)]),
    "stn_sum_slices_ordered": (C.c_int, [_P, C.c_uint64, C.c_int64, _P, _P]),
    "stn_fold_slices_ordered": (C.c_int, [_P, C.c_uint64, C.c_int64, _P, _P]),
    "stn_run_slices_host": (C.c_int, [_P, _P, C.POINTER(C.c_int32), C.c_uint64, C.c_uint64, _P,
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "stn_flush_block_cache": (C.c_int, []),
    "stn_device_count": (C.c_int, []),
    "stn_multi_create": (C.c_int, [C.POINTER(PlanDesc), C.c_int, C.POINTER(C.c_int32), C.c_int,
                                   _PP]),
    "stn_multi_destroy": (C.c_int, [_P]),
    "stn_multi_device_count": (C.c_int, [_P]),
    "stn_multi_plan": (_P, [_P, C.c_int]),
    "stn_multi_build_caches": (C.c_int, [_P]),
    "stn_multi_set_leaf_values": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_double), C.c_int64]),
    "stn_multi_run_scheme": (C.c_int, [_P, C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(RunReport)]),
    "stn_multi_run_slices": (C.c_int, [_P, C.POINTER(C.c_int32), C.c_uint64, C.c_uint64, C.c_int,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "stn_run_scheme_multi": (C.c_int, [C.POINTER(PlanDesc), C.c_int, C.POINTER(C.c_int32),
                                       C.c_int, C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(RunReport)]),
    "stn_selftest_chain_jit": (C.c_int, [C.c_int, C.c_char_p, C.c_int32]),
    "stn_selftest_bitperm": (C.c_int, [C.c_int32, C.POINTER(C.c_int32), C.c_int32,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       C.POINTER(C.c_int32)]),
    "stn_selftest_gemm_tc": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                       C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}

_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Loads libstn_exec.so (built by ``__graft_entry__.build()``); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"B200 executor library not built: {path} is missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != 0:
        msg = _lib.stn_last_error().decode() if _lib is not None else ""
        raise StnError(status, msg)
