"""A/B timing of executor variants (STN_DEBUG strings) on one config, interleaved in
one process so clock / power-cap drift hits every variant alike.

usage: ab_compare.py CFG N_SLICES REPS VARIANT [VARIANT ...]   (VARIANT "" = default)
Prints the median ms/slice per variant and writes gpurun_out/ab_<cfg>.json."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2005_06787_b200 import ExecutablePlan, build_branch_cache  # noqa: E402
from paper_2005_06787_b200.runtime import load_desc, run_slices_digits  # noqa: E402

cfg, n, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
variants = sys.argv[4:] or [""]
path = bench.plan_file(cfg)
d = load_desc(path).contents
dims = [d.sliced_dims[i] for i in range(d.n_sliced)]
digits = np.array([bench.digits_of(a, dims) for a in range(n)], np.int32).reshape(
    n, max(len(dims), 1))
times = {v: [] for v in variants}
sums = {}
for rep in range(reps):
    for v in variants:
        os.environ["STN_DEBUG"] = v
        plan = ExecutablePlan.load(path, device=0, mode="fast")
        plan.set_streams(2)  # as bench.py
        cache = build_branch_cache(plan)
        acc = torch.zeros(2 * plan.out_elements, dtype=torch.float64, device="cuda")
        run_slices_digits(plan, cache, digits[: min(n, 2)], acc=acc)  # warm-up
        torch.cuda.synchronize()
        acc.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run_slices_digits(plan, cache, digits, acc=acc)
        e1.record()
        torch.cuda.synchronize()
        times[v].append(e0.elapsed_time(e1) / n)
        sums[v] = float(acc.abs().sum())
        print(f"rep {rep} [{v}] {times[v][-1]:.3f} ms/slice", flush=True)
        cache.close()
        plan.close()
        torch.cuda.empty_cache()
res = {v: {"median_ms_per_slice": statistics.median(t), "all": t, "abs_sum": sums[v]}
       for v, t in times.items()}
for v, r in res.items():
    print(f"{cfg} [{v}]: median {r['median_ms_per_slice']:.3f} ms/slice  sum {r['abs_sum']:.6e}")
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/ab_{cfg}.json", "w") as f:
    json.dump({"cfg": cfg, "slices": n, "reps": reps, "variants": res}, f, indent=1)
