"""Host-side mirror of the reference executor API (runtime.hpp), on the B200.

The names, argument meanings and error behaviour follow
/root/reference/proj/include/stemtn/runtime.hpp so callers (and the parity
tests) read like the reference's own:

    reference (runtime.hpp)                 here
    ---------------------------------------  ------------------------------------------
    ExecutablePlan        (60-73)            ExecutablePlan.load(path) / .from_desc()
    build_branch_cache    (492-500)          build_branch_cache(plan)
    run_subtask           (502-514)          run_subtask(plan, assignment, cache)
    SubtaskResult         (75-81)            SubtaskResult
    run_scheme            (555-632)          run_scheme(plan, parallelism)
    RunReport             (516-550)          RunReport (+ to_json / deterministic_json)
    stemtn::Error         (errors.hpp:60)    abi.StnError (.kind is the ErrorKind name)

Every call goes through the C ABI of libstn_exec.so; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import abi
from .abi import check

MODES = {"fast": abi.STN_MODE_FAST, "exact": abi.STN_MODE_EXACT}


def _lib():
    return abi.load_library()


def _stream_handle(stream) -> C.c_void_p:
    """Accepts None, an int handle, or a torch.cuda.Stream."""
    if stream is None:
        return C.c_void_p(0)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(int(stream.cuda_stream))


class ExecutablePlan:
    """A flattened stemtn::ExecutablePlan resident on one GPU."""

    def __init__(self, handle: C.c_void_p, mode: int):
        self._h = handle
        self.mode = mode
        info = abi.PlanInfo()
        check(_lib().stn_plan_get_info(self._h, C.byref(info)))
        self.info = info
        self.identity = info.identity
        self.subtasks = info.subtasks
        self.n_sliced = info.n_sliced
        self.out_dims = tuple(info.out_dims[i] for i in range(info.out_rank))
        self.out_elements = info.out_elements

    @classmethod
    def load(cls, path: str, device: int = 0, mode: str = "fast") -> "ExecutablePlan":
        """Loads a plan file written by the reference-side adapter (flatten.hpp)."""
        lib = _lib()
        desc = C.POINTER(abi.PlanDesc)()
        check(lib.stn_plan_load(path.encode(), C.byref(desc)))
        try:
            return cls.from_desc(desc, device, mode)
        finally:
            lib.stn_plan_desc_free(desc)

    @classmethod
    def from_desc(cls, desc, device: int = 0, mode: str = "fast") -> "ExecutablePlan":
        h = C.c_void_p()
        m = MODES[mode] if isinstance(mode, str) else int(mode)
        check(_lib().stn_plan_create(desc, device, m, C.byref(h)))
        return cls(h, m)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib().stn_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def set_leaf_values(self, vertex: int, values) -> None:
        """Replaces a vertex tensor (what frugal_sample does to plan.net,
        sampler.hpp:206-213). Branch caches built before become stale."""
        v = np.ascontiguousarray(np.asarray(values, dtype=np.complex128).ravel())
        check(_lib().stn_plan_set_leaf_values(
            self._h, vertex, v.view(np.float64).ctypes.data_as(C.POINTER(C.c_double)), v.size))

    def set_max_batch(self, n: int) -> None:
        check(_lib().stn_plan_set_max_batch(self._h, n))

    def set_streams(self, n: int) -> None:
        """Streams (each with its own arena) that run_slices* rotate batches over."""
        check(_lib().stn_plan_set_streams(self._h, n))

    def set_profiling(self, enable: bool = True) -> None:
        check(_lib().stn_plan_set_profiling(self._h, 1 if enable else 0))

    def reset_profile(self) -> None:
        check(_lib().stn_plan_reset_profile(self._h))

    def get_profile(self) -> dict:
        """Per kernel class: launches, device ms, algorithmic bytes and flops."""
        arr = (abi.KernelProfile * len(abi.KERNEL_KINDS))()
        check(_lib().stn_plan_get_profile(self._h, arr))
        return {abi.KERNEL_KINDS[i]: {"launches": arr[i].launches, "ms": arr[i].ms,
                                      "bytes": arr[i].bytes, "flops": arr[i].flops}
                for i in range(len(abi.KERNEL_KINDS))}

    def get_step_profile(self) -> list:
        """Per plan step: kernel kind, shape, launches, device ms, bytes, flops."""
        n = C.c_int32()
        check(_lib().stn_plan_get_step_profile(self._h, None, 0, C.byref(n)))
        arr = (abi.StepProfile * max(1, n.value))()
        check(_lib().stn_plan_get_step_profile(self._h, arr, n.value, C.byref(n)))
        return [{"step": e.step, "kernel": abi.KERNEL_KINDS[e.kind], "M": e.M, "N": e.N,
                 "K": e.K, "launches": e.launches, "ms": e.ms, "bytes": e.bytes,
                 "flops": e.flops} for e in arr[: n.value]]

    def kernel_mix(self) -> dict:
        i = self.info
        return {"tensor_core": i.steps_tensor_core, "absorb": i.steps_absorb,
                "generic": i.steps_generic, "sweeps": i.sweeps,
                "steps_in_sweeps": i.steps_in_sweeps}


def load_desc(path: str):
    """Host-side plan descriptor (no device needed); free with free_desc."""
    desc = C.POINTER(abi.PlanDesc)()
    check(_lib().stn_plan_load(path.encode(), C.byref(desc)))
    return desc


def free_desc(desc) -> None:
    _lib().stn_plan_desc_free(desc)


def desc_leaf_bytes(desc) -> int:
    """Bytes of vertex-tensor data a plan upload copies host -> device."""
    d = desc.contents
    total = 0
    for i in range(d.n_leaves):
        L = d.leaves[i]
        n = 1
        for k in range(L.rank):
            n *= L.dims[k]
        total += 16 * n
    return total


class BranchCache:
    """Device-resident slice-invariant partial results (runtime.hpp:146-152)."""

    def __init__(self, handle: C.c_void_p, plan: ExecutablePlan):
        self._h = handle
        self._plan = plan  # keeps the plan alive
        ident, mults, elems = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(_lib().stn_cache_info(self._h, C.byref(ident), C.byref(mults), C.byref(elems)))
        self.plan_identity = ident.value
        self.mults = mults.value
        self.elements = elems.value

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib().stn_cache_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_branch_cache(plan: ExecutablePlan, stream=None) -> BranchCache:
    h = C.c_void_p()
    check(_lib().stn_cache_build(plan.handle, _stream_handle(stream), C.byref(h)))
    return BranchCache(h, plan)


@dataclass
class SubtaskResult:
    assignment: int = 0
    value: np.ndarray = field(default_factory=lambda: np.zeros((), np.complex128))
    step_count: int = 0
    mults: int = 0
    peak_elements: int = 0


def _result(plan: ExecutablePlan, out: np.ndarray, info: abi.SubtaskInfo) -> SubtaskResult:
    return SubtaskResult(assignment=info.assignment,
                         value=out.view(np.complex128).reshape(plan.out_dims),
                         step_count=info.step_count, mults=info.mults,
                         peak_elements=info.peak_elements)


def run_subtask(plan: ExecutablePlan, assignment: int, cache: BranchCache | None = None,
                stream=None) -> SubtaskResult:
    out = np.zeros(2 * plan.out_elements, np.float64)
    info = abi.SubtaskInfo()
    check(_lib().stn_run_subtask(plan.handle, assignment, cache.handle if cache else None,
                                 _stream_handle(stream),
                                 out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(info)))
    return _result(plan, out, info)


def run_subtask_digits(plan: ExecutablePlan, digits, cache: BranchCache | None = None,
                       stream=None) -> SubtaskResult:
    """One subtask from an explicit digit vector (plans whose uint64 subtask
    count overflows, e.g. 85 sliced edges)."""
    d = (C.c_int32 * max(1, plan.n_sliced))(*digits)
    out = np.zeros(2 * plan.out_elements, np.float64)
    info = abi.SubtaskInfo()
    check(_lib().stn_run_subtask_digits(plan.handle, d, cache.handle if cache else None,
                                        _stream_handle(stream),
                                        out.ctypes.data_as(C.POINTER(C.c_double)),
                                        C.byref(info)))
    return _result(plan, out, info)


def run_slices(plan: ExecutablePlan, cache: BranchCache, lo: int, hi: int, acc=None,
               per_slice=None, stream=None) -> None:
    """Runs slices [lo, hi) asynchronously. ``acc`` / ``per_slice`` are device
    float64 tensors (torch) or raw device pointers (int)."""

    def ptr(t):
        if t is None:
            return None
        return C.c_void_p(t if isinstance(t, int) else t.data_ptr())

    check(_lib().stn_run_slices(plan.handle, cache.handle, lo, hi, _stream_handle(stream),
                                ptr(acc), ptr(per_slice)))


def run_slices_digits(plan: ExecutablePlan, cache: BranchCache, digits: np.ndarray, acc=None,
                      per_slice=None, stream=None) -> None:
    d = np.ascontiguousarray(digits, dtype=np.int32)
    n = d.shape[0] if d.ndim == 2 else 0

    def ptr(t):
        if t is None:
            return None
        return C.c_void_p(t if isinstance(t, int) else t.data_ptr())

    check(_lib().stn_run_slices_digits(plan.handle, cache.handle,
                                       d.ctypes.data_as(C.POINTER(C.c_int32)), n,
                                       _stream_handle(stream), ptr(acc), ptr(per_slice)))


@dataclass
class RunReport:
    """RunReport (runtime.hpp:516-550); planner-side log2_tc / cw are not known
    to the executor and stay None unless the caller fills them."""
    subtasks: int = 1
    mult_count: int = 0
    branch_mults: int = 0
    wall_seconds: float = 0.0
    p50_ms: float = 0.0
    p90_ms: float = 0.0
    p99_ms: float = 0.0
    parallelism: int = 1
    precision: str = "single"
    peak_elements: int = 0
    merged_groups: int = 0
    log2_tc: float | None = None
    cw: int | None = None
    slices_per_batch: int = 1
    kernel_launches: int = 0

    def to_json(self) -> dict:
        return {"log2_tc": self.log2_tc, "cw": self.cw, "subtasks": self.subtasks,
                "mult_count": self.mult_count, "branch_mults": self.branch_mults,
                "wall_seconds": self.wall_seconds,
                "per_subtask_ms": {"p50": self.p50_ms, "p90": self.p90_ms, "p99": self.p99_ms},
                "parallelism": self.parallelism, "precision": self.precision,
                "peak_elements": self.peak_elements, "merged_groups": self.merged_groups}

    def deterministic_json(self) -> dict:
        j = self.to_json()
        for k in ("wall_seconds", "per_subtask_ms", "parallelism"):
            j.pop(k)
        return j


def run_scheme(plan: ExecutablePlan, parallelism: int = 1):
    """Every subtask, summed in ascending assignment order in double
    (bit-stable for any parallelism, runtime.hpp:552-605)."""
    out = np.zeros(2 * plan.out_elements, np.float64)
    rep = abi.RunReport()
    check(_lib().stn_run_scheme(plan.handle, parallelism,
                                out.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rep)))
    r = RunReport(subtasks=rep.subtasks, mult_count=rep.mult_count,
                  branch_mults=rep.branch_mults, wall_seconds=rep.wall_seconds,
                  p50_ms=rep.p50_ms, p90_ms=rep.p90_ms, p99_ms=rep.p99_ms,
                  parallelism=rep.parallelism,
                  precision="single" if rep.precision == abi.STN_SINGLE else "double",
                  peak_elements=rep.peak_elements, merged_groups=rep.merged_groups,
                  slices_per_batch=rep.slices_per_batch, kernel_launches=rep.kernel_launches)
    return out.view(np.complex128).reshape(plan.out_dims), r


def run_slices_host(plan: ExecutablePlan, cache: BranchCache, lo: int = 0, n: int | None = None,
                    digits: np.ndarray | None = None, per_slice: bool = True, total: bool = True,
                    stream=None):
    """A worker envelope with host buffers (queue.hpp:250-252): slices [lo, lo+n)
    or the rows of `digits`; returns (per-slice roots [n, *out_dims] or None,
    ascending-order sum or None) as complex128 host arrays. Blocking."""
    d = None
    if digits is not None:
        d = np.ascontiguousarray(digits, dtype=np.int32).reshape(-1, max(plan.n_sliced, 1))
        n = d.shape[0]
    elif n is None:
        n = plan.subtasks - lo
    rows = np.zeros((max(n, 1), 2 * plan.out_elements), np.float64) if per_slice else None
    s = np.zeros(2 * plan.out_elements, np.float64) if total else None
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None  # noqa: E731
    check(_lib().stn_run_slices_host(plan.handle, cache.handle,
                                     d.ctypes.data_as(C.POINTER(C.c_int32)) if d is not None else None,
                                     lo, n, _stream_handle(stream), dp(rows), dp(s)))
    out_rows = rows[:n].view(np.complex128).reshape((n,) + plan.out_dims) if per_slice else None
    out_sum = s.view(np.complex128).reshape(plan.out_dims) if total else None
    return out_rows, out_sum


def flush_block_cache() -> None:
    """Frees the executor's cached device blocks (arenas of destroyed plans)."""
    check(_lib().stn_flush_block_cache())


def fold_slices_ordered(per_slice, n_slices: int, out_elements: int, acc, stream=None) -> None:
    """acc = (((acc + r_0) + r_1) + ...) on the device: continues an ascending fold."""
    check(_lib().stn_fold_slices_ordered(C.c_void_p(per_slice.data_ptr()) if n_slices else None,
                                         n_slices, out_elements, C.c_void_p(acc.data_ptr()),
                                         _stream_handle(stream)))


class MultiPlan:
    """One device plan + branch cache per GPU of this box, driven from one
    process (include/stn_exec.h, "several GPUs"): the in-process replacement of
    the reference's worker processes (queue.hpp:197-336)."""

    def __init__(self, desc, devices, mode: str = "fast"):
        devs = list(devices)
        arr = (C.c_int32 * len(devs))(*devs)
        h = C.c_void_p()
        m = MODES[mode] if isinstance(mode, str) else int(mode)
        check(_lib().stn_multi_create(desc, len(devs), arr, m, C.byref(h)))
        self._h = h
        self.devices = devs
        info = abi.PlanInfo()
        check(_lib().stn_plan_get_info(_lib().stn_multi_plan(h, 0), C.byref(info)))
        self.info = info
        self.subtasks = info.subtasks
        self.n_sliced = info.n_sliced
        self.out_dims = tuple(info.out_dims[i] for i in range(info.out_rank))
        self.out_elements = info.out_elements

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib().stn_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run_scheme(self, deterministic: bool = True):
        out = np.zeros(2 * self.out_elements, np.float64)
        rep = abi.RunReport()
        check(_lib().stn_multi_run_scheme(self._h, 1 if deterministic else 0,
                                          out.ctypes.data_as(C.POINTER(C.c_double)),
                                          C.byref(rep)))
        r = RunReport(subtasks=rep.subtasks, mult_count=rep.mult_count,
                      branch_mults=rep.branch_mults, wall_seconds=rep.wall_seconds,
                      p50_ms=rep.p50_ms, p90_ms=rep.p90_ms, p99_ms=rep.p99_ms,
                      parallelism=rep.parallelism,
                      precision="single" if rep.precision == abi.STN_SINGLE else "double",
                      peak_elements=rep.peak_elements)
        return out.view(np.complex128).reshape(self.out_dims), r

    def run_slices(self, lo: int = 0, n: int | None = None, digits: np.ndarray | None = None,
                   deterministic: bool = True, per_slice: bool = False, total: bool = True):
        d = None
        if digits is not None:
            d = np.ascontiguousarray(digits, dtype=np.int32).reshape(-1, max(self.n_sliced, 1))
            n = d.shape[0]
        elif n is None:
            n = self.subtasks - lo
        rows = np.zeros((max(n, 1), 2 * self.out_elements), np.float64) if per_slice else None
        s = np.zeros(2 * self.out_elements, np.float64) if total else None
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None  # noqa: E731
        check(_lib().stn_multi_run_slices(
            self._h, d.ctypes.data_as(C.POINTER(C.c_int32)) if d is not None else None, lo, n,
            1 if deterministic else 0, dp(rows), dp(s)))
        out_rows = rows[:n].view(np.complex128).reshape((n,) + self.out_dims) if per_slice else None
        out_sum = s.view(np.complex128).reshape(self.out_dims) if total else None
        return out_rows, out_sum


def sum_slices_ordered(per_slice, n_slices: int, out_elements: int, out, stream=None) -> None:
    """Ascending-order fp64 sum of per-slice results on the device."""
    check(_lib().stn_sum_slices_ordered(C.c_void_p(per_slice.data_ptr()), n_slices,
                                        out_elements, C.c_void_p(out.data_ptr()),
                                        _stream_handle(stream)))
