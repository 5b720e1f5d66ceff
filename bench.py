#!/usr/bin/env python3
"""Benchmark of the B200 stem executor on BASELINE.json's headline workload.

Workload (default, BASELINE.json configs[4], SURVEY cfg5): the 53-qubit
Sycamore layout, m=20 cycles, a batch of 64 amplitudes (6 open qubits), planned
by the REFERENCE planner (PlannerParams defaults, seed 1, target width 33) and
lowered by the reference compile(): 85 sliced edges (2^85 slices: the
reference's uint64 subtasks() overflows, scheme.hpp:33-37, so slices are
addressed by digit vectors -- assignment a's mixed-radix digits, first sliced
edge most significant, runtime.hpp:371-378), 677 per-slice steps, stem tensors
of 2^33 complex64 = 64 GiB: the per-slice stem benchmark at the largest stem
that fits 180 GB of HBM. Plan file: tests/golden/cfg5_syc53_m20/plan_single.stnplan.
`--config cfg2|cfg3|cfg4|cfg1` runs the other BASELINE configs (companion lines).

A "step" is one pass of the per-slice stem program over S slices per GPU
(--slices-per-gpu; 2 for cfg5), branch cache resident in HBM, followed by the
cross-GPU combination of the per-slice amplitudes (the chained ascending fold
of distributed.py: bitwise the reference's run_scheme order). Every rank runs
its own slices (weak scaling); the only cross-GPU traffic is the 1 KiB fp64
accumulator.

  value  slices/s over the whole job, device-resident (CUDA events on the
         launch stream, max over ranks)
  e2e    the same through the C ABI with HOST buffers (stn_run_slices_host:
         pinned digit vectors H2D, per-slice amplitudes + sum D2H, every step),
         plus the cross-rank all-reduce; plan upload + branch-cache build are
         one-time setup, reported beside it
Stem tensors (cfg5: 64 GiB; cfg2: 1 GiB) are far larger than L2 (126 MB), so no
L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import ctypes as C
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
    "cfg5": "cfg5_syc53_m20",
}
WORKLOAD_TEXT = {
    "cfg1": "grid4x5 m=14 single amplitude, 16 slices (BASELINE configs[0])",
    "cfg2": "grid5x6 m=16, batch of 64 amplitudes, 2^6 sliced edges (BASELINE configs[1])",
    "cfg3": "sycamore53 m=12, batch of 64 amplitudes, 2^14 slices (BASELINE configs[2])",
    "cfg4": "sycamore53 m=14, batch of 64 amplitudes, 2^19 slices (BASELINE configs[3])",
    "cfg5": ("sycamore53 m=20, batch of 64 amplitudes, 2^85 slices addressed by digit vectors, "
             "per-slice stem benchmark at the largest stem fitting 180 GB HBM "
             "(2^33 complex64) (BASELINE configs[4])"),
}
SLICES_PER_GPU = {"cfg1": 16, "cfg2": 64, "cfg3": 16, "cfg4": 16, "cfg5": 8}


def plan_file(cfg: str) -> str:
    return os.path.join(REPO, "tests", "golden", CONFIGS[cfg], "plan_single.stnplan")


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return (float(j["hbm_gbs"]), float(j["bf16_tflops"]),
                float(j.get("bf16_tflops_sustained", j["bf16_tflops"])), "measured")
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def digits_of(a: int, dims: list[int]) -> list[int]:
    """Mixed-radix digits of assignment a, first sliced edge most significant
    (runtime.hpp:371-378); python ints, so 85 sliced edges are fine."""
    out = [0] * len(dims)
    for i in range(len(dims) - 1, -1, -1):
        a, out[i] = divmod(a, dims[i])
    return out


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


# ---------------------------------------------------------------------------
# CPU baselines (test infrastructure: the reference executor or the oracle port)
# ---------------------------------------------------------------------------
def _calib_path(cfg: str) -> str:
    return os.path.join(REPO, "profiles", f"cpu_calib_{cfg}.json")


def port_slice_profile(cfg: str, threads: int, budget_s: float, slice_index: int = 0):
    """The oracle port of the reference executor (oracle/stn_oracle.c, bitwise the
    reference's arithmetic; its strided gemm_lean holds a step's operands and
    output only, so a 2^33 stem needs 128 GiB of host RAM where the reference's
    Engine::gemm needs 256 GiB) on one slice, `threads` host threads splitting
    every large step. Returns (per-step ms, complete)."""
    from oracle.oracle import OraclePlan
    p = OraclePlan(plan_file(cfg))
    cache = p.build_cache()
    return p.time_slice_lean(digits_of(slice_index, p.sliced_dims), cache, threads, budget_s)


def scale_prefix(ms: list[float], complete: bool, calib: list[float]):
    """Slice seconds from a timed prefix, scaled by the full-slice per-step times
    of the same code on the same host (calib)."""
    k = len(ms)
    if complete:
        return sum(ms) / 1e3, 1.0
    done = sum(calib[:k])
    return sum(ms) / 1e3 * sum(calib) / max(done, 1e-9), done / sum(calib)


def cpu_port_baseline(cfg: str, threads: int, budget_s: float, calib: dict | None):
    ms, complete = port_slice_profile(cfg, threads, budget_s)
    if not complete and calib is None:
        return None
    slice_s, frac = scale_prefix(ms, complete, calib["step_ms"] if calib else ms)
    return {"value": 1.0 / slice_s, "unit": "slices/s", "cores": threads, "kind": "port",
            "sample": (f"one slice through the oracle port of the reference executor "
                       f"(oracle/stn_oracle.c gemm_lean; the reference's own Engine::gemm "
                       f"needs 4 stem tensors = 256 GiB > this host's RAM), {threads} threads "
                       f"splitting each step, timed for {budget_s:.0f} s = "
                       f"{100 * frac:.1f}% of the slice, scaled by the full-slice per-step "
                       f"times {calib.get('source', '') if calib else ''}"),
            "slice_seconds": slice_s}


def cpu_reference_baseline(cfg: str, threads: int, budget_s: float, calib: dict | None):
    """The reference CPU executor itself (oracle/_ref/ref_tool: the reference
    headers compiled as they lie; Engine<float>::load_leaf/gemm in Engine::run's
    order, runtime.hpp:420-453) on `threads` host threads, each running the
    per-slice steps of its own slice for budget_s; scaled to full slices by the
    per-step times of full reference slices recorded on a GPU box host."""
    tool = os.path.join(REPO, "oracle", "_ref", "ref_tool")
    d = os.path.join(REPO, "tests", "golden", CONFIGS[cfg])
    if not os.path.exists(tool):
        return None
    threads = min(threads, ref_threads_for_memory(d))
    if calib is None:
        cpath = os.path.join(d, "ref_step_ms.json")
        if os.path.exists(cpath):
            with open(cpath) as f:
                calib = {"step_ms": json.load(f)["step_ms"],
                         "source": "of one reference slice on the 8-core build host"}
    out = subprocess.run([tool, "bench-prefix", d, "--threads", str(threads), "--budget",
                          str(budget_s)], capture_output=True, text=True, check=True).stdout
    j = json.loads(out.strip().splitlines()[-1])
    rates, fracs = [], []
    for t in j["per_thread"]:
        if not t["complete"] and calib is None:
            return None
        s, fr = scale_prefix(t["step_ms"], t["complete"], calib["step_ms"] if calib else [])
        rates.append(1.0 / s)
        fracs.append(fr)
    return {"value": sum(rates), "unit": "slices/s", "cores": threads, "kind": "reference",
            "sample": (f"{threads} thread(s), each running the per-slice steps of its own slice "
                       f"through the reference executor for {budget_s:.0f} s "
                       f"({100 * statistics.mean(fracs):.1f}% of a slice on average), scaled "
                       f"to a full slice by the per-step times "
                       f"{calib.get('source', '') if calib else ''}; wall {j['wall_s']:.1f} s")}


def ref_threads_for_memory(golden_dir: str) -> int:
    """Threads of the reference executor that fit this host's free RAM: each holds
    up to four stem-sized tensors of 2^exec_cw complex64 (Engine::gemm's operands,
    output and a permute buffer, runtime.hpp:341-453)."""
    try:
        with open(os.path.join(golden_dir, "meta.json")) as f:
            cw = int(json.load(f)["plan"]["exec_cw"])
        with open("/proc/meminfo") as f:
            avail = next(int(line.split()[1]) * 1024 for line in f
                         if line.startswith("MemAvailable:"))
    except (OSError, KeyError, ValueError, StopIteration):
        return 1
    return max(1, int(0.6 * avail) // (4 * 8 << cw))


def load_calib(cfg: str):
    try:
        with open(_calib_path(cfg)) as f:
            return json.load(f)
    except FileNotFoundError:
        return None


def run_reference_arm(args):
    """The reference's CPU path on this box's host cores, same config/metric."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = args.cpu_threads or os.cpu_count() or 1
    cfg = args.config
    vals, walls, cb = [], [], None
    calib = None
    if cfg == "cfg5":
        # same-box calibration: one full slice of the port in the first warm-up step
        t0 = time.perf_counter()
        ms, complete = port_slice_profile(cfg, threads, 0.0)
        calib = {"step_ms": ms, "source": f"of a full slice on this host in this run "
                                          f"({sum(ms) / 1e3:.1f} s)"}
        walls.append(time.perf_counter() - t0)
        # the calibration slice is the first warm-up step, or the first timed one
        if args.warmup == 0:
            vals.append(1e3 / sum(ms))
        cb = {"value": 1e3 / sum(ms), "unit": "slices/s", "cores": threads, "kind": "port",
              "sample": (f"one full slice through the oracle port of the reference executor "
                         f"(oracle/stn_oracle.c gemm_lean), {threads} threads splitting each "
                         f"step, {sum(ms) / 1e3:.1f} s"),
              "slice_seconds": sum(ms) / 1e3}
    for i in range(args.warmup + args.steps - (1 if cfg == "cfg5" else 0)):
        t0 = time.perf_counter()
        if cfg == "cfg5":
            cb = cpu_port_baseline(cfg, threads, args.ref_budget, calib)
        else:
            cb = cpu_reference_baseline(cfg, threads, args.ref_budget, load_calib(cfg))
        walls.append(time.perf_counter() - t0)
        if cb is None:
            print(json.dumps({"impl": "reference",
                              "unavailable": "reference tool or calibration not built"}))
            return
        if i >= args.warmup - (1 if cfg == "cfg5" else 0):
            vals.append(cb["value"])
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "slices/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(walls[-args.steps:]),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c64",
        "data": "synthetic (reference-planned random circuit, seed 1)",
        "config": config_keys(args, args.slices_per_gpu or SLICES_PER_GPU[cfg]),
        "cpu_baseline": dict(cb, value=v),
        "e2e": {"value": v, "unit": "slices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def config_keys(args, slices_per_step: int) -> dict:
    return {"workload": WORKLOAD_TEXT[args.config], "plan": CONFIGS[args.config],
            "slices_per_gpu_per_step": slices_per_step, "mode": args.mode,
            "streams": args.streams,
            "parallelism": "slices sharded over the GPUs (one process each), chained "
                           "1 KiB fp64 fold across ranks",
            "l2": "stem tensors >> L2 (126 MB); no flush needed"}


# ---------------------------------------------------------------------------
# the B200 executor
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5", choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="fast", choices=["fast", "exact"])
    ap.add_argument("--slices-per-gpu", type=int, default=0)
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-budget", type=float, default=15.0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--streams", type=int, default=2)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2005_06787_b200 import ExecutablePlan, abi, build_branch_cache
    from paper_2005_06787_b200.distributed import distributed_sum
    from paper_2005_06787_b200.runtime import (_stream_handle, fold_slices_ordered, free_desc,
                                               load_desc, run_slices_digits)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # rank 0's stdout carries exactly one JSON line: no NCCL version / info banner
    # (NCCL prints its version banner to stdout at any NCCL_DEBUG level: leave it unset
    # unless STN_NCCL_DEBUG asks for one)
    if "STN_NCCL_DEBUG" in os.environ:
        os.environ["NCCL_DEBUG"] = os.environ["STN_NCCL_DEBUG"]
    else:
        os.environ.pop("NCCL_DEBUG", None)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    S = args.slices_per_gpu or SLICES_PER_GPU[args.config]

    t_setup = time.perf_counter()
    desc = load_desc(plan_file(args.config))
    plan = ExecutablePlan.from_desc(desc, device=local, mode=args.mode)
    # batches of slices rotate over this many streams, each with its own arena (the
    # library caps it by free HBM: cfg5's 96 GiB arena runs one lane)
    plan.set_streams(args.streams)
    cache = build_branch_cache(plan, stream)
    torch.cuda.synchronize(dev)
    setup_s = time.perf_counter() - t_setup
    oe = plan.out_elements
    dims = [desc.contents.sliced_dims[i] for i in range(plan.n_sliced)]
    n_total = plan.subtasks if plan.subtasks else 1 << 64  # cfg5: assignments < 2^64

    def step_digits(step: int, r: int = rank, n_ranks: int = world) -> np.ndarray:
        base = step * n_ranks * S + r * S
        d = [digits_of((base + i) % n_total, dims) for i in range(S)]
        return np.array(d, np.int32).reshape(S, max(len(dims), 1))

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

    def fold(rows, n, acc):
        fold_slices_ordered(rows, n, oe, acc, stream=stream)

    def step(p, c, k: int):
        # this rank's S slices of step k, then the chained ascending fold across ranks
        dg = step_digits(k)

        def compute(lo, hi, per_slice, acc):
            run_slices_digits(p, c, dg[lo - rank * S: hi - rank * S], acc=acc,
                              per_slice=per_slice, stream=stream)

        return distributed_sum(S * world, oe, compute, fold, dev, True, None)

    # ---- device-resident throughput (no per-launch events in this region) ----
    for k in range(args.warmup):
        step(plan, cache, k)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for k in range(args.steps):
            result = step(plan, cache, args.warmup + k)
        e1.record(stream)
        barrier()
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    slices_per_sec = S * world / (ms / 1e3)
    flops_per_slice = 8.0 * plan.info.per_slice_mults
    stem_tflops = flops_per_slice * slices_per_sec / 1e12

    # ---- per-kernel roofline: the same steps again with CUDA events around every
    # launch on the launch stream ----
    # one lane here: with several, kernels of different lanes overlap and their event
    # durations would add up to more than the wall time
    plan.set_streams(1)
    plan.set_profiling(True)
    plan.reset_profile()
    for k in range(args.steps):
        step(plan, cache, args.warmup + k)
    barrier()
    prof = plan.get_profile()
    steps_prof = plan.get_step_profile()
    plan.set_profiling(False)
    plan.set_streams(args.streams)

    # ---- end to end through the C ABI from HOST buffers ----
    lib = abi.load_library()
    rows_h = torch.empty((S, 2 * oe), dtype=torch.float64).pin_memory()
    sum_h = torch.empty(2 * oe, dtype=torch.float64).pin_memory()
    dig_h = torch.empty((S, max(len(dims), 1)), dtype=torch.int32).pin_memory()
    acc_d = torch.zeros(2 * oe, dtype=torch.float64, device=dev)
    e2e_ms = []
    base_k = args.warmup + args.steps
    for k in range(args.e2e_steps + 1 if args.e2e_steps > 0 else 0):
        barrier()
        t0 = time.perf_counter()
        dig_h.numpy()[:] = step_digits(base_k + k)
        abi.check(lib.stn_run_slices_host(
            plan.handle, cache.handle, C.cast(C.c_void_p(dig_h.data_ptr()), C.POINTER(C.c_int32)),
            0, S, _stream_handle(stream),
            C.cast(C.c_void_p(rows_h.data_ptr()), C.POINTER(C.c_double)),
            C.cast(C.c_void_p(sum_h.data_ptr()), C.POINTER(C.c_double))))
        if world > 1:  # combine the per-GPU partial amplitudes (1 KiB)
            acc_d.copy_(sum_h, non_blocking=True)
            dist.all_reduce(acc_d)
            sum_h.copy_(acc_d)
        torch.cuda.synchronize(dev)
        dt = max_over_ranks(time.perf_counter() - t0)
        if k > 0:  # first call pays one-time host-side setup of the pinned path
            e2e_ms.append(1e3 * dt)
    e2e_value = S * world / (statistics.median(e2e_ms) / 1e3) if e2e_ms else None
    h2d = S * max(len(dims), 1) * 4
    d2h = S * 2 * oe * 8 + 2 * oe * 8

    # ---- roofline of the dominant kernel class ----
    hbm_peak, tc_peak, tc_sust, peak_src = peaks()
    dom = max((k for k in prof if k not in ("leaf", "root")), key=lambda k: prof[k]["ms"])
    d = prof[dom]
    step_ms_total = sum(v["ms"] for v in prof.values())
    if dom == "gemm_tc":
        # split-TF32: 3 TF32 products per algorithmic product; TF32 = half the bf16 rate
        achieved = d["flops"] / (d["ms"] / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tc_peak / 2 / 3,
                "unit": "TFLOP/s", "peak_note": "3xTF32 split: measured bf16 burst / 2 / 3"}
    else:
        achieved = d["bytes"] / (d["ms"] / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = None
    roof["algorithmic_bytes_per_launch"] = d["bytes"] / d["launches"] if d["launches"] else None
    # (traffic below: ncu dram__bytes_read.sum + dram__bytes_write.sum per launch of the same
    # class over one slice, committed under profiles/; per-launch averages of one slice)
    tpath = os.path.join(REPO, "profiles", f"dram_traffic_{args.config}.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        tcls = tj.get("classes", {}).get(dom)
        if tcls:
            roof["traffic"] = tcls["dram_bytes_per_launch"]
            roof["traffic_source"] = tj.get("source")
    roof["kernel"] = dom
    roof["share_of_step"] = d["ms"] / step_ms_total if step_ms_total else None
    roof["launches_per_step"] = d["launches"] / args.steps
    roof["peak_source"] = peak_src
    roof["per_kernel_class"] = {k: {"ms_per_step": v["ms"] / args.steps,
                                    "launches_per_step": v["launches"] / args.steps,
                                    "GBps": v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] else None,
                                    "TFLOPs": v["flops"] / (v["ms"] / 1e3) / 1e12 if v["ms"] else None}
                                for k, v in prof.items() if v["launches"]}
    top = sorted(steps_prof, key=lambda r: -r["ms"])[:8]
    roof["top_steps"] = [{"step": r["step"], "kernel": r["kernel"], "M": r["M"], "N": r["N"],
                          "K": r["K"], "ms_per_slice": r["ms"] / (args.steps * S),
                          "GBps": r["bytes"] / (r["ms"] / 1e3) / 1e9 if r["ms"] else None,
                          "TFLOPs": r["flops"] / (r["ms"] / 1e3) / 1e12 if r["ms"] else None}
                         for r in top]
    slice_bytes = sum(v["bytes"] for v in prof.values()) / (args.steps * S)
    launches = sum(v["launches"] for v in prof.values()) / args.steps + 1  # + fold

    line = {
        "metric": METRIC, "value": slices_per_sec, "unit": "slices/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c64",
        "data": "synthetic (reference-planned random circuit, seed 1)",
        "config": config_keys(args, S),
        "stem_tflops": stem_tflops,
        "flops_per_slice": flops_per_slice,
        "algorithmic_bytes_per_slice": slice_bytes,
        "slice_roofline_ms": slice_bytes / (hbm_peak * 1e9) * 1e3,
        "clocks": clocks.summary(),
        "e2e": {"value": e2e_value, "unit": "slices/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "ms_per_step": statistics.median(e2e_ms) if e2e_ms else None,
                "api": "stn_run_slices_host (C ABI, pinned host digits in, amplitudes out)",
                "one_time_setup_s": setup_s,
                "allocation": "the plan's lane arenas and workspaces are allocated by its first "
                              "batches (warm-up) and reused; the timed region allocates "
                              "nothing (the executor's block cache only serves plans that are "
                              "destroyed and created again)",
                "setup": "plan upload (vertex tensors H2D) + branch-cache build, once per "
                         "process like the reference worker's ensure_plan (queue.hpp:204-219)"},
        "gpu_launches": int(launches * args.steps),
        "arena_bytes_per_slice": int(plan.info.arena_bytes_per_slice),
        "roofline": roof,
        "checksum": float(np.abs(result.cpu().numpy()).sum()),
    }
    if rank == 0 and world == 1 and args.cpu_baseline:
        threads = args.cpu_threads or os.cpu_count() or 1
        if args.config == "cfg5":
            line["cpu_baseline"] = cpu_port_baseline(args.config, threads, args.cpu_budget,
                                                     load_calib(args.config))
        else:
            line["cpu_baseline"] = cpu_reference_baseline(args.config, threads, args.cpu_budget,
                                                          load_calib(args.config))
    if rank == 0:
        print(json.dumps(line))
    cache.close()
    plan.close()
    free_desc(desc)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
