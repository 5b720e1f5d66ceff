"""Per-step kernel choice and device time for one config.

usage: step_profile.py CFG [MODE] [N_SLICES] [OUT_JSON]
Slices are assignments 0..n-1 (digit vectors for plans whose uint64 subtask
count overflows, e.g. cfg5). Prints the steps by device time; writes all rows
to OUT_JSON when given."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2005_06787_b200 import ExecutablePlan, build_branch_cache  # noqa: E402
from paper_2005_06787_b200.runtime import load_desc, run_slices_digits  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8
out_json = sys.argv[4] if len(sys.argv) > 4 else None
path = bench.plan_file(cfg)
plan = ExecutablePlan.load(path, device=0, mode=mode)
d = load_desc(path).contents
dims = [d.sliced_dims[i] for i in range(d.n_sliced)]
total = plan.subtasks if plan.subtasks else 1 << 64
n = min(n, total)
digits = np.array([bench.digits_of(a % total, dims) for a in range(n)], np.int32).reshape(
    n, max(len(dims), 1))
cache = build_branch_cache(plan)
acc = torch.zeros(2 * plan.out_elements, dtype=torch.float64, device="cuda")
run_slices_digits(plan, cache, digits[: min(n, 2)], acc=acc)  # warm-up
torch.cuda.synchronize()
plan.set_profiling(True)
plan.reset_profile()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run_slices_digits(plan, cache, digits, acc=acc)
e1.record()
torch.cuda.synchronize()
rows = plan.get_step_profile()
tot = sum(r["ms"] for r in rows)
print(plan.kernel_mix())
print(f"{cfg} {mode} STN_DEBUG={os.environ.get('STN_DEBUG', '')}: {n} slices, "
      f"{tot / n:.3f} ms/slice over {len(rows)} steps (wall with events {e0.elapsed_time(e1) / n:.3f})")
print("step kernel     M          N          K        ms/slice  share   GB/s    TFLOP/s")
for r in sorted(rows, key=lambda r: -r["ms"])[:40]:
    gbs = r["bytes"] / (r["ms"] / 1e3) / 1e9 if r["ms"] else 0
    tf = r["flops"] / (r["ms"] / 1e3) / 1e12 if r["ms"] else 0
    print(f"{r['step']:4d} {r['kernel']:9s} {r['M']:10d} {r['N']:10d} {r['K']:8d} "
          f"{r['ms'] / n:9.3f} {r['ms'] / tot:6.3f} {gbs:7.0f} {tf:8.2f}")
if out_json:
    with open(out_json, "w") as f:
        json.dump({"cfg": cfg, "mode": mode, "slices": n, "debug": os.environ.get("STN_DEBUG"),
                   "ms_per_slice": tot / n, "rows": rows}, f)
