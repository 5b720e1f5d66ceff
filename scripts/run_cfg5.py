"""BASELINE configs[4]: 53-qubit Sycamore m=20, 85 sliced edges (the uint64
subtask count overflows, so slices are addressed by digit vectors), stem
tensors of 2^33 complex64 = 64 GiB. Runs a few slices, reports per-slice time,
the plan's arena and the top steps."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2005_06787_b200 import ExecutablePlan, build_branch_cache  # noqa: E402
from paper_2005_06787_b200.runtime import run_slices_digits  # noqa: E402

path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                    "golden", "cfg5_syc53_m20", "plan_single.stnplan")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
t0 = time.time()
plan = ExecutablePlan.load(path, device=0, mode="fast")
info = plan.info
print(json.dumps({"subtasks_u64": plan.subtasks, "n_sliced": plan.n_sliced,
                  "arena_GiB_per_slice": info.arena_bytes_per_slice / 2**30,
                  "cache_MiB": info.cache_bytes / 2**20, "per_slice_steps": info.per_slice_steps,
                  "per_slice_flops": 8.0 * info.per_slice_mults,
                  "kernels": plan.kernel_mix(), "plan_s": time.time() - t0}))
cache = build_branch_cache(plan)
rng = np.random.default_rng(5)
digits = rng.integers(0, 2, size=(n, plan.n_sliced)).astype(np.int32)
acc = torch.zeros(2 * plan.out_elements, dtype=torch.float64, device="cuda")
per = torch.zeros((n, 2 * plan.out_elements), dtype=torch.float64, device="cuda")
run_slices_digits(plan, cache, digits[:1], acc=acc, per_slice=per[:1])  # warm-up
torch.cuda.synchronize()
plan.set_profiling(True)
plan.reset_profile()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run_slices_digits(plan, cache, digits, acc=acc, per_slice=per)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
vals = per.cpu().numpy().view(np.complex128)
rows = plan.get_step_profile()
tot = sum(r["ms"] for r in rows)
print(json.dumps({"slices": n, "ms_per_slice": ms, "finite": bool(np.isfinite(vals).all()),
                  "max_abs": float(np.abs(vals).max()),
                  "stem_tflops": 8.0 * info.per_slice_mults / (ms / 1e3) / 1e12,
                  "algorithmic_GBps": sum(r["bytes"] for r in rows) / (tot / 1e3) / 1e9}))
for r in sorted(rows, key=lambda r: -r["ms"])[:15]:
    print(f"{r['step']:5d} {r['kernel']:10s} M={r['M']:<11d} N={r['N']:<11d} K={r['K']:<7d} "
          f"{r['ms'] / n:8.2f} ms {r['bytes'] / (r['ms'] / 1e3) / 1e9 if r['ms'] else 0:7.0f} GB/s")
