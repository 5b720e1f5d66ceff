"""Per-step device times of bench.py's timed loop (cfg5 by default), with and without
the nvidia-smi clock sampler running, to see what the sampler or the loop costs.
usage: bench_diag.py [CFG] [STEPS]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2005_06787_b200 import ExecutablePlan, build_branch_cache  # noqa: E402
from paper_2005_06787_b200.distributed import distributed_sum  # noqa: E402
from paper_2005_06787_b200.runtime import fold_slices_ordered, load_desc, run_slices_digits  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
S = bench.SLICES_PER_GPU[cfg]
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
desc = load_desc(bench.plan_file(cfg))
plan = ExecutablePlan.from_desc(desc, device=0, mode="fast")
plan.set_streams(2)
cache = build_branch_cache(plan, stream)
oe = plan.out_elements
dims = [desc.contents.sliced_dims[i] for i in range(plan.n_sliced)]


def digits(k):
    return np.array([bench.digits_of(k * S + i, dims) for i in range(S)], np.int32).reshape(
        S, max(len(dims), 1))


def step(k, mode):
    dg = digits(k)
    if mode == "acc":
        acc = torch.zeros(2 * oe, dtype=torch.float64, device=dev)
        run_slices_digits(plan, cache, dg, acc=acc, stream=stream)
        return acc

    def compute(lo, hi, per_slice, acc):
        run_slices_digits(plan, cache, dg[lo:hi], acc=acc, per_slice=per_slice, stream=stream)

    return distributed_sum(S, oe, compute, lambda r, n, a: fold_slices_ordered(r, n, oe, a, stream=stream),
                           dev, True, None)


for k in range(3):
    step(k, "rows")
torch.cuda.synchronize()
for mode, sampler in (("rows", False), ("rows", True), ("acc", False), ("rows", False)):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ctx = bench.ClockSampler(0) if sampler else None
    if ctx:
        ctx.__enter__()
    ev[0].record(stream)
    for k in range(steps):
        step(3 + k, mode)
        ev[k + 1].record(stream)
    torch.cuda.synchronize()
    if ctx:
        ctx.__exit__()
    t = [ev[i].elapsed_time(ev[i + 1]) / S for i in range(steps)]
    print(f"{cfg} mode={mode} sampler={sampler}: ms/slice per step {[round(x, 2) for x in t]} "
          f"mean {statistics.mean(t):.2f}", flush=True)
