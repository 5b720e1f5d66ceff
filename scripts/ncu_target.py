"""Small driver for ncu captures: build the branch cache, run a few slices of
one config (digit vectors of assignments 0..n-1, so cfg5 works too)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2005_06787_b200 import ExecutablePlan, build_branch_cache  # noqa: E402
from paper_2005_06787_b200.runtime import load_desc, run_slices_digits  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
path = bench.plan_file(cfg)
plan = ExecutablePlan.load(path, device=0, mode="fast")
d = load_desc(path).contents
dims = [d.sliced_dims[i] for i in range(d.n_sliced)]
digits = np.array([bench.digits_of(a, dims) for a in range(n)], np.int32).reshape(n, -1)
cache = build_branch_cache(plan)
acc = torch.zeros(2 * plan.out_elements, dtype=torch.float64, device="cuda")
run_slices_digits(plan, cache, digits, acc=acc)
torch.cuda.synchronize()
print("ok", acc.abs().sum().item())
