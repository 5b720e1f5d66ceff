"""B200-native (sm_100a) stem executor for sliced tensor-network contraction.

Drop-in for the executor of the reference `stemtn` runtime
(/root/reference/proj/include/stemtn/runtime.hpp). The C ABI is
include/stn_exec.h; `runtime` mirrors the reference's executor API on top of
it and `distributed` shards slices over the GPUs of one box.
"""
from .abi import StnError, load_library  # noqa: F401
from .runtime import (BranchCache, ExecutablePlan, MultiPlan, RunReport,  # noqa: F401
                      SubtaskResult, build_branch_cache, flush_block_cache,
                      fold_slices_ordered, run_scheme, run_slices, run_slices_digits,
                      run_slices_host, run_subtask, run_subtask_digits, sum_slices_ordered)

__all__ = ["ExecutablePlan", "BranchCache", "SubtaskResult", "RunReport", "StnError",
           "build_branch_cache", "run_subtask", "run_subtask_digits", "run_slices",
           "run_slices_digits", "run_slices_host", "run_scheme", "sum_slices_ordered",
           "fold_slices_ordered", "flush_block_cache", "MultiPlan", "load_library"]
