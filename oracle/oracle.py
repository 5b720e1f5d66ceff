"""TEST INFRASTRUCTURE ONLY -- ctypes binding of the CPU oracle (oracle/liboracle.so).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline. The product (paper_2005_06787_b200) never imports it.

The oracle is the C restatement of the reference executor (oracle/stn_oracle.c),
bitwise equal to the reference CPU path; it is pinned against outputs of the
reference itself in tests/golden (tests/test_oracle_golden.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2005_06787_b200.abi import PlanDesc, SubtaskInfo, StnError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_TOOL = os.path.join(HERE, "_ref", "ref_tool")


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        P = C.c_void_p
        L.stn_plan_load.argtypes = [C.c_char_p, C.POINTER(C.POINTER(PlanDesc))]
        L.stn_plan_load.restype = C.c_int
        L.stn_plan_desc_free.argtypes = [C.POINTER(PlanDesc)]
        L.stn_plan_desc_free.restype = None
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_cache_build.argtypes = [C.POINTER(PlanDesc), C.c_int]
        L.oracle_cache_build.restype = P
        L.oracle_cache_free.argtypes = [P]
        L.oracle_cache_free.restype = None
        L.oracle_cache_info.argtypes = [P] + [C.POINTER(C.c_uint64)] * 3
        L.oracle_run_subtask.argtypes = [C.POINTER(PlanDesc), C.c_int, C.c_uint64, P,
                                         C.POINTER(C.c_double), C.c_int64,
                                         C.POINTER(SubtaskInfo)]
        L.oracle_run_subtask_digits.argtypes = [C.POINTER(PlanDesc), C.c_int,
                                                C.POINTER(C.c_int32), P, C.POINTER(C.c_double),
                                                C.c_int64, C.POINTER(SubtaskInfo)]
        L.oracle_run_subtask_digits_lean.argtypes = [C.POINTER(PlanDesc), C.c_int,
                                                     C.POINTER(C.c_int32), P,
                                                     C.POINTER(C.c_double), C.c_int64,
                                                     C.POINTER(SubtaskInfo), C.c_int]
        L.oracle_time_slice_lean.argtypes = [C.POINTER(PlanDesc), C.c_int, C.POINTER(C.c_int32),
                                             P, C.c_int, C.c_double, C.POINTER(C.c_double),
                                             C.c_int32, C.POINTER(C.c_int32),
                                             C.POINTER(C.c_int32), C.POINTER(C.c_double)]
        L.oracle_run_slices.argtypes = [C.POINTER(PlanDesc), C.c_int, P, C.c_uint64, C.c_uint64,
                                        C.c_int, C.c_int64, C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]
        L.oracle_out_elements.argtypes = [C.POINTER(PlanDesc)]
        L.oracle_out_elements.restype = C.c_int64
        L.oracle_decode_assignment.argtypes = [C.POINTER(PlanDesc), C.c_uint64,
                                               C.POINTER(C.c_int32)]
        _lib = L
    return _lib


def _check(st: int) -> None:
    if st != 0:
        raise StnError(st, lib().oracle_last_error().decode())


class OraclePlan:
    """A plan file executed by the CPU oracle."""

    def __init__(self, path: str, precision: int | None = None):
        L = lib()
        self._desc = C.POINTER(PlanDesc)()
        _check(L.stn_plan_load(path.encode(), C.byref(self._desc)))
        d = self._desc.contents
        self.precision = d.precision if precision is None else precision
        self.subtasks = d.subtasks
        self.n_sliced = d.n_sliced
        self.sliced_dims = [d.sliced_dims[i] for i in range(d.n_sliced)]
        self.out_elements = int(L.oracle_out_elements(self._desc))
        self._caches = []

    def __del__(self):
        try:
            for c in self._caches:
                lib().oracle_cache_free(c)
            lib().stn_plan_desc_free(self._desc)
        except Exception:
            pass

    @property
    def desc(self):
        return self._desc

    def build_cache(self):
        c = lib().oracle_cache_build(self._desc, self.precision)
        if not c:
            raise StnError(16, lib().oracle_last_error().decode())
        self._caches.append(c)
        return c

    def digits(self, assignment: int) -> list[int]:
        arr = (C.c_int32 * max(1, self.n_sliced))()
        lib().oracle_decode_assignment(self._desc, assignment, arr)
        return list(arr[: self.n_sliced])

    def run_subtask(self, assignment: int, cache=None):
        out = np.zeros(2 * self.out_elements, dtype=np.float64)
        info = SubtaskInfo()
        _check(lib().oracle_run_subtask(self._desc, self.precision, assignment, cache,
                                        out.ctypes.data_as(C.POINTER(C.c_double)),
                                        self.out_elements, C.byref(info)))
        return out.view(np.complex128), info

    def run_subtask_digits(self, digits, cache=None):
        out = np.zeros(2 * self.out_elements, dtype=np.float64)
        arr = (C.c_int32 * max(1, self.n_sliced))(*digits)
        info = SubtaskInfo()
        _check(lib().oracle_run_subtask_digits(self._desc, self.precision, arr, cache,
                                               out.ctypes.data_as(C.POINTER(C.c_double)),
                                               self.out_elements, C.byref(info)))
        return out.view(np.complex128), info

    def run_subtask_digits_lean(self, digits, cache=None, threads: int = 1):
        """Bitwise the same value as run_subtask_digits, computed without the
        reference's materialised transposes (oracle/stn_oracle.c gemm_lean) on
        `threads` host threads: the oracle for 2^33-element stems."""
        out = np.zeros(2 * self.out_elements, dtype=np.float64)
        arr = (C.c_int32 * max(1, self.n_sliced))(*digits)
        info = SubtaskInfo()
        _check(lib().oracle_run_subtask_digits_lean(self._desc, self.precision, arr, cache,
                                                    out.ctypes.data_as(C.POINTER(C.c_double)),
                                                    self.out_elements, C.byref(info), threads))
        return out.view(np.complex128), info

    def time_slice_lean(self, digits, cache=None, threads: int = 1, budget_s: float = 0.0,
                        with_value: bool = False):
        """Per-step wall-clock ms of the lean oracle on one slice (stops after
        the step during which budget_s passed; 0 = whole slice) -> (ms list,
        complete[, value when complete])."""
        arr = (C.c_int32 * max(1, self.n_sliced))(*digits)
        cap = 1 << 16
        ms = np.zeros(cap, np.float64)
        out = np.zeros(2 * self.out_elements, np.float64)
        n, done = C.c_int32(), C.c_int32()
        _check(lib().oracle_time_slice_lean(self._desc, self.precision, arr, cache, threads,
                                            budget_s, ms.ctypes.data_as(C.POINTER(C.c_double)),
                                            cap, C.byref(n), C.byref(done),
                                            out.ctypes.data_as(C.POINTER(C.c_double))))
        if with_value:
            return ms[: n.value].tolist(), bool(done.value), out.view(np.complex128)
        return ms[: n.value].tolist(), bool(done.value)

    def run_slices(self, lo: int, hi: int, cache=None, threads: int = 1):
        n = hi - lo
        vals = np.zeros((max(n, 1), 2 * self.out_elements), dtype=np.float64)
        s = np.zeros(2 * self.out_elements, dtype=np.float64)
        _check(lib().oracle_run_slices(self._desc, self.precision, cache, lo, hi, threads,
                                       self.out_elements,
                                       vals.ctypes.data_as(C.POINTER(C.c_double)),
                                       s.ctypes.data_as(C.POINTER(C.c_double))))
        return vals[:n].view(np.complex128), s.view(np.complex128)
