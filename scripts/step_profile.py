"""Per-step kernel choice and device time for one config (one pass of all slices)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2005_06787_b200 import ExecutablePlan, build_branch_cache, run_slices  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
plan = ExecutablePlan.load(bench.plan_file(cfg), device=0, mode=mode)
cache = build_branch_cache(plan)
import torch  # noqa: E402
acc = torch.zeros(2 * plan.out_elements, dtype=torch.float64, device="cuda")
run_slices(plan, cache, 0, min(plan.subtasks, 4), acc=acc)
torch.cuda.synchronize()
plan.set_profiling(True)
plan.reset_profile()
n = min(plan.subtasks, 8)
run_slices(plan, cache, 0, n, acc=acc)
torch.cuda.synchronize()
rows = plan.get_step_profile()
tot = sum(r["ms"] for r in rows)
print(plan.kernel_mix())
print(f"{cfg} {mode}: {n} slices, {tot / n:.3f} ms/slice over {len(rows)} steps")
print("step kernel     M          N          K        ms/slice  share   GB/s    TFLOP/s")
for r in sorted(rows, key=lambda r: -r["ms"]):
    gbs = r["bytes"] / (r["ms"] / 1e3) / 1e9 if r["ms"] else 0
    tf = r["flops"] / (r["ms"] / 1e3) / 1e12 if r["ms"] else 0
    print(f"{r['step']:4d} {r['kernel']:9s} {r['M']:10d} {r['N']:10d} {r['K']:8d} "
          f"{r['ms'] / n:9.3f} {r['ms'] / tot:6.3f} {gbs:7.0f} {tf:8.2f}")
