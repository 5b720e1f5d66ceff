"""Where the end-to-end time of one bench step goes: plan creation (host compile +
uploads), branch-cache build, the 64 slices, and the result copy."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2005_06787_b200 import ExecutablePlan, build_branch_cache, run_slices  # noqa: E402
from paper_2005_06787_b200.runtime import load_desc  # noqa: E402

desc = load_desc(bench.plan_file("cfg2"))
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = ExecutablePlan.from_desc(desc, device=0, mode="fast")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    c = build_branch_cache(p)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    acc = torch.zeros(2 * p.out_elements, dtype=torch.float64, device="cuda")
    run_slices(p, c, 0, p.subtasks, acc=acc)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    host = acc.cpu().numpy()
    t4 = time.perf_counter()
    print(f"iter {it}: plan {1e3*(t1-t0):.1f} ms, cache {1e3*(t2-t1):.1f} ms, "
          f"slices {1e3*(t3-t2):.1f} ms, d2h {1e3*(t4-t3):.2f} ms")
    c.close()
    p.close()
