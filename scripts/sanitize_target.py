"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck, one tool
per run): every kernel family of the executor on small inputs.

  * the tcgen05 split-TF32 GEMMs: fused-split (BN 64 / 128 / 256) and pre-split;
  * cfg1 (grid4x5, m=14) EXACT and FAST with fused chains everywhere (NVRTC kernels);
  * rt_grid3x4_m8_sliced over three streams with CUDA-graph replay;
  * one FAST slice of cfg2 (TMA-fed tcgen05 absorbs, lane / direct absorbs, tcgen05
    GEMMs, tile permutes, specialised chains).
Prints OK at the end; the sanitizer's own report is the result."""
import ctypes as C
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
os.environ["STN_DEBUG"] = "chain_min_bits=0"

import torch  # noqa: E402

from golden_io import plan_path  # noqa: E402
from paper_2005_06787_b200 import (ExecutablePlan, abi, build_branch_cache,  # noqa: E402
                                   run_slices, run_subtask)

lib = abi.load_library()
err, ms, msg, mss, serr = (C.c_double() for _ in range(5))
for M, N, K in ((256, 32, 256), (256, 64, 128), (256, 128, 64)):
    abi.check(lib.stn_selftest_gemm_tc(M, N, K, 2, 1, 1, 1, C.byref(err), C.byref(ms),
                                       C.byref(msg), C.byref(mss), C.byref(serr)))
    print("tcf gemm", M, N, K, err.value, flush=True)
os.environ["STN_DEBUG"] = "chain_min_bits=0,tcf=0"
abi.check(lib.stn_selftest_gemm_tc(256, 128, 64, 1, 1, 1, 1, C.byref(err), C.byref(ms),
                                   C.byref(msg), C.byref(mss), C.byref(serr)))
print("pre-split gemm", err.value, flush=True)
os.environ["STN_DEBUG"] = "chain_min_bits=0"

for mode in ("exact", "fast"):
    p = ExecutablePlan.load(plan_path("cfg1_grid4x5_m14", "single"), device=0, mode=mode)
    c = build_branch_cache(p)
    r = run_subtask(p, 3, c)
    print("cfg1", mode, p.kernel_mix(), abs(r.value).max(), flush=True)

p = ExecutablePlan.load(plan_path("rt_grid3x4_m8_sliced", "single"), device=0, mode="fast")
c = build_branch_cache(p)
p.set_streams(3)
p.set_max_batch(4)
acc = torch.zeros(2 * p.out_elements, dtype=torch.float64, device="cuda")
for _ in range(2):
    run_slices(p, c, 0, p.subtasks, acc=acc)
torch.cuda.synchronize()
print("streams + graphs", float(acc.abs().sum()), flush=True)

os.environ["STN_DEBUG"] = ""
p = ExecutablePlan.load(plan_path("cfg2_grid5x6_m16", "single"), device=0, mode="fast")
c = build_branch_cache(p)
r = run_subtask(p, 0, c)
print("cfg2", p.kernel_mix(), abs(r.value).max(), flush=True)
print("OK")
