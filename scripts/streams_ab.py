"""Slices/s of one config for several stream counts, with and without CUDA graphs.
usage: streams_ab.py CFG N_SLICES [streams ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2005_06787_b200 import ExecutablePlan, build_branch_cache  # noqa: E402
from paper_2005_06787_b200.runtime import load_desc, run_slices_digits  # noqa: E402

cfg, n = sys.argv[1], int(sys.argv[2])
streams = [int(x) for x in sys.argv[3:]] or [1, 2, 3]
path = bench.plan_file(cfg)
d = load_desc(path).contents
dims = [d.sliced_dims[i] for i in range(d.n_sliced)]
out = []
for graphs in ("1", "0"):
    os.environ["STN_DEBUG"] = f"graphs={graphs}"
    plan = ExecutablePlan.load(path, device=0, mode="fast")
    cache = build_branch_cache(plan)
    total = plan.subtasks if plan.subtasks else 1 << 64
    digits = np.array([bench.digits_of(a % total, dims) for a in range(n)], np.int32).reshape(n, -1)
    acc = torch.zeros(2 * plan.out_elements, dtype=torch.float64, device="cuda")
    for s in streams:
        plan.set_streams(s)
        for _ in range(2):
            run_slices_digits(plan, cache, digits, acc=acc)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            run_slices_digits(plan, cache, digits, acc=acc)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        r = {"cfg": cfg, "graphs": graphs, "streams": s, "slices": n, "ms": ms,
             "slices_per_s": n / ms * 1e3}
        print(json.dumps(r), flush=True)
        out.append(r)
    cache.close()
    plan.close()
