#!/usr/bin/env python3
"""Benchmark of the B200 stem executor on BASELINE.json's headline workload.

Workload (BASELINE.json configs[1]): 30-qubit 5x6-grid
Sycamore-style random circuit, 16 cycles, batch of 64 amplitudes (6 open
qubits), 2^6 sliced edges, planned by the REFERENCE planner (PlannerParams
defaults, seed 1, target width 28) and lowered by the reference compile();
the plan file is tests/golden/cfg2_grid5x6_m16/plan_single.stnplan.

A "step" is the whole sliced contraction: all 64 slices through the per-slice
stem program with the branch cache resident in HBM, their roots combined in
fp64 in ascending slice order. With N GPUs the 64 slices are sharded (strong
scaling) and combined with one NCCL all-reduce.

  value  slices/s over the whole job, inputs already resident (device time,
         max over ranks)
  e2e    the same through the C ABI from HOST buffers: plan upload (vertex
         tensors H2D), branch-cache build, all slices, result D2H
Every stem tensor of this workload is 2^27 complex64 (1 GiB) > L2 (126 MB),
so no L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "slices/sec and achieved stem FLOP/s vs roofline at 1/2/4/8 B200 vs CPU ref"
CONFIGS = {
    "cfg1": "cfg1_grid4x5_m14",
    "cfg2": "cfg2_grid5x6_m16",
    "cfg3": "cfg3_syc53_m12",
    "cfg4": "cfg4_syc53_m14",
}
WORKLOAD_TEXT = {
    "cfg1": "grid4x5 m=14 single amplitude, 16 slices (BASELINE configs[0])",
    "cfg2": "grid5x6 m=16, batch of 64 amplitudes, 2^6 sliced edges (BASELINE configs[1])",
    "cfg3": "sycamore53 m=12, batch of 64 amplitudes, 2^14 slices (BASELINE configs[2])",
    "cfg4": "sycamore53 m=14, batch of 64 amplitudes, 2^19 slices (BASELINE configs[3])",
}


def plan_file(cfg: str) -> str:
    return os.path.join(REPO, "tests", "golden", CONFIGS[cfg], "plan_single.stnplan")


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for n, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def cpu_baseline(cfg: str, threads: int, budget_s: float):
    """The reference CPU executor (oracle/_ref/ref_tool: the reference headers
    compiled as they lie; its Engine<float>::load_leaf/gemm in Engine::run's
    order, runtime.hpp:420-453) on this host's cores, as a bounded sample:
    every thread runs the per-slice steps of its own slice for `budget_s`
    seconds. A thread's slice time is its prefix time scaled by the full-slice /
    prefix time ratio of the same steps recorded on the build host
    (tests/golden/<cfg>/ref_step_ms.json, one full reference slice, 1 thread)."""
    tool = os.path.join(REPO, "oracle", "_ref", "ref_tool")
    d = os.path.join(REPO, "tests", "golden", CONFIGS[cfg])
    calib_path = os.path.join(d, "ref_step_ms.json")
    if not os.path.exists(tool):
        return None
    calib = None
    if os.path.exists(calib_path):
        with open(calib_path) as f:
            calib = json.load(f)["step_ms"]
    out = subprocess.run([tool, "bench-prefix", d, "--threads", str(threads), "--budget",
                          str(budget_s)], capture_output=True, text=True, check=True).stdout
    j = json.loads(out.strip().splitlines()[-1])
    rates, fracs = [], []
    for t in j["per_thread"]:
        ms = t["step_ms"]
        k = len(ms)
        if t["complete"]:
            slice_s = sum(ms) / 1e3
            fracs.append(1.0)
        elif calib is None:
            return None
        else:
            slice_s = sum(ms) / 1e3 * sum(calib) / max(sum(calib[:k]), 1e-9)
            fracs.append(sum(calib[:k]) / sum(calib))
        rates.append(1.0 / slice_s)
    value = sum(rates)
    return {"value": value, "unit": "slices/s", "cores": threads, "kind": "reference",
            "sample": (f"{threads} thread(s), each running the per-slice steps of its own slice "
                       f"through the reference executor for {budget_s:.0f} s "
                       f"({100 * statistics.mean(fracs):.1f}% of a slice's reference time on "
                       f"average), scaled to a full slice by the per-step times of one full "
                       f"reference slice recorded on the build host; wall {j['wall_s']:.1f} s")}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = args.cpu_threads or os.cpu_count() or 1
    vals = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(args.config, threads, args.ref_budget)
        if cb is None:
            print(json.dumps({"impl": "reference",
                              "unavailable": "oracle/_ref/ref_tool or calibration not built"}))
            return
        if i >= args.warmup:
            vals.append(cb["value"])
    v = statistics.median(vals)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "slices/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * args.ref_budget, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c64", "data": "synthetic",
        "config": {"workload": WORKLOAD_TEXT[args.config], "plan": CONFIGS[args.config]},
        "cpu_baseline": dict(cb, value=v),
        "e2e": {"value": v, "unit": "slices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="fast", choices=["fast", "exact"])
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-budget", type=float, default=12.0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2005_06787_b200 import ExecutablePlan, build_branch_cache
    from paper_2005_06787_b200.distributed import distributed_sum
    from paper_2005_06787_b200.runtime import (desc_leaf_bytes, free_desc, load_desc,
                                               run_slices, sum_slices_ordered)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)

    path = plan_file(args.config)
    desc = load_desc(path)
    plan = ExecutablePlan.from_desc(desc, device=local, mode=args.mode)
    cache = build_branch_cache(plan, stream)
    n, oe = plan.subtasks, plan.out_elements

    def step(p, c):
        def compute(lo, hi, per_slice, acc):
            run_slices(p, c, lo, hi, acc=acc, per_slice=per_slice, stream=stream)

        def ordered(buf, nn, out):
            sum_slices_ordered(buf, nn, oe, out, stream=stream)

        return distributed_sum(n, oe, compute, ordered, dev, True, None)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident throughput (no per-launch events in this region) ----
    for _ in range(args.warmup):
        step(plan, cache)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            result = step(plan, cache)
        e1.record(stream)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    # ---- per-kernel roofline: the same steps again with CUDA events around
    # every launch on the launch stream ----
    plan.set_profiling(True)
    plan.reset_profile()
    for _ in range(args.steps):
        step(plan, cache)
    barrier()
    prof = plan.get_profile()
    plan.set_profiling(False)
    slices_per_sec = n / (ms / 1e3)
    flops_per_slice = 8.0 * plan.info.per_slice_mults
    stem_tflops = flops_per_slice * slices_per_sec / 1e12

    # ---- end to end through the C ABI from host buffers ----
    h2d = desc_leaf_bytes(desc)
    d2h = 16 * oe
    e2e_ms = []
    for i in range(args.e2e_steps + 1 if args.e2e_steps > 0 else 0):
        barrier()
        t0 = time.perf_counter()
        p2 = ExecutablePlan.from_desc(desc, device=local, mode=args.mode)
        c2 = build_branch_cache(p2, stream)
        out = step(p2, c2)
        host = out.cpu().numpy()
        barrier()
        dt = max_over_ranks(time.perf_counter() - t0)
        if i > 0:  # first call pays one-time CUDA module/attribute setup
            e2e_ms.append(1e3 * dt)
        c2.close()
        p2.close()
    e2e_value = n / (statistics.median(e2e_ms) / 1e3) if e2e_ms else None

    # ---- roofline of the dominant kernel ----
    hbm_peak, tc_peak, peak_src = peaks()
    dom = max((k for k in prof if k not in ("leaf", "root")), key=lambda k: prof[k]["ms"])
    d = prof[dom]
    step_ms_total = sum(v["ms"] for v in prof.values())
    if dom in ("gemm_tc",):
        achieved = d["flops"] / (d["ms"] / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tc_peak / 2, "unit": "TFLOP/s"}
    else:
        achieved = d["bytes"] / (d["ms"] / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    # DRAM bytes per launch of the dominant class from the committed ncu launch list
    # (dram__bytes_read.sum + dram__bytes_write.sum, scripts/traffic_from_ncu.py), next
    # to the algorithmic bytes per launch that `achieved` is computed from
    roof["traffic"] = None
    roof["algorithmic_bytes_per_launch"] = d["bytes"] / d["launches"] if d["launches"] else None
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                         "r01_dram_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tcls = json.load(f).get("classes", {}).get(dom)
        if tcls:
            roof["traffic"] = tcls["bytes_per_launch"]
            roof["traffic_source"] = "profiles/r01_dram_traffic.json (ncu, cfg2, 1 slice + cache build)"
    roof["kernel"] = dom
    roof["share_of_step"] = d["ms"] / step_ms_total if step_ms_total else None
    roof["launches_per_step"] = d["launches"] / args.steps
    roof["peak_source"] = peak_src
    roof["per_kernel_class"] = {k: {"ms_per_step": v["ms"] / args.steps,
                                    "launches_per_step": v["launches"] / args.steps,
                                    "GBps": v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] else None,
                                    "TFLOPs": v["flops"] / (v["ms"] / 1e3) / 1e12 if v["ms"] else None}
                                for k, v in prof.items() if v["launches"]}
    launches = sum(v["launches"] for v in prof.values()) // args.steps + 1  # + ordered sum

    line = {
        "metric": METRIC, "value": slices_per_sec * 1.0, "unit": "slices/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c64",
        "data": "synthetic (reference-planned random circuit, seed 1)",
        "config": {"workload": WORKLOAD_TEXT[args.config], "plan": CONFIGS[args.config],
                   "slices": n, "amplitudes": oe, "mode": args.mode,
                   "parallelism": f"slices sharded over {world} GPU(s), 1 NCCL all-reduce",
                   "l2": "stem tensors 1 GiB > L2; no flush needed",
                   "roofline_timing": "separate pass of the same steps with per-launch events"},
        "stem_tflops": stem_tflops,
        "flops_per_slice": flops_per_slice,
        "clocks": clocks.summary(),
        "e2e": {"value": e2e_value, "unit": "slices/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "ms_per_step": statistics.median(e2e_ms) if e2e_ms else None},
        "gpu_launches": int(launches) * args.steps,
        "roofline": roof,
        "checksum": float(np.abs(result.cpu().numpy()).sum()),
    }
    if rank == 0 and world == 1 and args.cpu_baseline:
        threads = args.cpu_threads or os.cpu_count() or 1
        line["cpu_baseline"] = cpu_baseline(args.config, threads, args.cpu_budget)
    if rank == 0:
        print(json.dumps(line))
    free_desc(desc)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
