"""Small driver for ncu captures: build the branch cache, run a few slices of
one config (the kernels of interest then appear in every slice)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2005_06787_b200 import ExecutablePlan, build_branch_cache, run_slices  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
plan = ExecutablePlan.load(bench.plan_file(cfg), device=0, mode="fast")
cache = build_branch_cache(plan)
acc = torch.zeros(2 * plan.out_elements, dtype=torch.float64, device="cuda")
run_slices(plan, cache, 0, n, acc=acc)
torch.cuda.synchronize()
print("ok", acc.abs().sum().item())
