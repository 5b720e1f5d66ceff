"""Slices/s of the in-process multi-GPU C ABI (stn_multi_*) on every visible GPU:
cfg2 run_scheme (all 64 slices, deterministic chained fold and one NCCL all-reduce)
and cfg5 digit-vector envelopes, against 1 GPU."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2005_06787_b200 import MultiPlan  # noqa: E402
from paper_2005_06787_b200.runtime import load_desc  # noqa: E402

ngpu = torch.cuda.device_count()
for cfg, per_gpu in (("cfg2", None), ("cfg5", 2)):
    desc = load_desc(bench.plan_file(cfg))
    dims = [desc.contents.sliced_dims[i] for i in range(desc.contents.n_sliced)]
    for n in sorted({1, ngpu}):
        mp = MultiPlan(desc, list(range(n)))
        for det in (True, False):
            if per_gpu is None:
                mp.run_scheme(det)
                t0 = time.perf_counter()
                out, rep = mp.run_scheme(det)
                dt = time.perf_counter() - t0
                slices = mp.subtasks
            else:
                slices = per_gpu * n
                digits = np.array([bench.digits_of(a, dims) for a in range(slices)], np.int32)
                mp.run_slices(digits=digits, deterministic=det)
                t0 = time.perf_counter()
                _, out = mp.run_slices(digits=digits, deterministic=det)
                dt = time.perf_counter() - t0
            print(json.dumps({"cfg": cfg, "gpus": n, "deterministic": det, "slices": slices,
                              "seconds": dt, "slices_per_s": slices / dt,
                              "checksum": float(np.abs(out).sum())}), flush=True)
        mp.close()
