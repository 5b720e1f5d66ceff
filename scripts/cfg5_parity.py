"""cfg5 (BASELINE configs[4], 2^33-element stems) parity on a GPU box.

Phase 1 (GPU): slices given by the digit vectors of assignments 0 and 1
(mixed radix, first sliced edge most significant, runtime.hpp:371-378) in FAST
and -- if its arena fits -- EXACT mode; values saved.
Phase 2 (host): the same slices through the lean oracle (bitwise the
reference's arithmetic; the reference's own Engine::gemm needs 256 GiB of host
RAM at this stem size, the lean restatement 128 GiB) on all host threads, with
per-step times (the CPU-baseline calibration, profiles/cpu_calib_cfg5.json).
Writes gpurun_out/cfg5_parity.json."""
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402

PLAN = os.path.join(REPO, "tests", "golden", "cfg5_syc53_m20", "plan_single.stnplan")
OUT = os.path.join(REPO, "gpurun_out")
SLICES = [int(x) for x in os.environ.get("CFG5_SLICES", "0,1").split(",")]


def digits_of(a, dims):
    out = [0] * len(dims)
    for i in range(len(dims) - 1, -1, -1):
        a, out[i] = divmod(a, dims[i])
    return out


def gpu_phase():
    import torch
    from paper_2005_06787_b200 import ExecutablePlan, build_branch_cache, run_subtask_digits
    res = {}
    for mode in ("fast", "exact"):
        try:
            t0 = time.time()
            plan = ExecutablePlan.load(PLAN, device=0, mode=mode)
            cache = build_branch_cache(plan)
            dims = None
            from paper_2005_06787_b200.runtime import load_desc
            d = load_desc(PLAN).contents
            dims = [d.sliced_dims[i] for i in range(d.n_sliced)]
            vals = []
            for a in SLICES:
                r = run_subtask_digits(plan, digits_of(a, dims), cache)
                vals.append(r.value.ravel().copy())
                res.setdefault(mode + "_bookkeeping", []).append(
                    [r.step_count, r.mults, r.peak_elements])
            np.save(os.path.join(OUT, f"cfg5_gpu_{mode}.npy"), np.array(vals))
            res[mode] = {"ok": True, "seconds": time.time() - t0,
                         "arena_GiB": plan.info.arena_bytes_per_slice / 2**30}
            cache.close()
            plan.close()
        except Exception as e:  # EXACT's arena may not fit next to the 2^33 stems
            res[mode] = {"ok": False, "error": str(e)[:300]}
        torch.cuda.empty_cache()
        from paper_2005_06787_b200 import flush_block_cache
        flush_block_cache()
    return res


def host_phase(res):
    from oracle.oracle import OraclePlan
    p = OraclePlan(PLAN)
    cache = p.build_cache()
    threads = os.cpu_count()
    out = {}
    for i, a in enumerate(SLICES):
        t0 = time.time()
        ms, complete, val = p.time_slice_lean(digits_of(a, p.sliced_dims),
                                              cache, threads, 0.0, with_value=True)
        wall = time.time() - t0
        entry = {"assignment": a, "oracle_seconds": wall, "complete": complete,
                 "max_abs": float(np.abs(val).max())}
        scale = max(float(np.abs(val).max()), 1e-300)
        for mode in ("fast", "exact"):
            f = os.path.join(OUT, f"cfg5_gpu_{mode}.npy")
            if res.get(mode, {}).get("ok") and os.path.exists(f):
                g = np.load(f)[i]
                entry[mode + "_rel_err"] = float(np.abs(g - val).max() / scale)
                entry[mode + "_bitwise"] = bool(np.array_equal(g.view(np.uint64),
                                                               val.view(np.uint64)))
        out[str(a)] = entry
        if i == 0:
            calib = {"step_ms": ms, "threads": threads,
                     "source": (f"of one full slice of the port on a GPU box host "
                                f"({threads} threads, {sum(ms) / 1e3:.1f} s, "
                                f"scripts/cfg5_parity.py)")}
            with open(os.path.join(OUT, "cpu_calib_cfg5.json"), "w") as f:
                json.dump(calib, f)
        np.save(os.path.join(OUT, f"cfg5_oracle_{a}.npy"), val)
        print(json.dumps(entry), flush=True)
    return out


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    r = {}
    if os.environ.get("CFG5_SKIP_GPU") != "1":
        r["gpu"] = gpu_phase()
        print(json.dumps(r["gpu"]), flush=True)
    else:
        r["gpu"] = {m: {"ok": True} for m in ("fast", "exact")}
    r["slices"] = host_phase(r["gpu"])
    with open(os.path.join(OUT, "cfg5_parity.json"), "w") as f:
        json.dump(r, f, indent=1)
