#!/usr/bin/env bash
# Regenerates the golden fixtures under tests/golden/ from the REFERENCE itself.
#
# Needs /root/reference (only present in the build container) and the oracle
# tool built from it:  make -C oracle ref
# For every case it writes, through the reference pipeline (oracle/ref_tool.cpp):
#   network.json, order.json        reference file formats (network.hpp:361, scheme.hpp:52)
#   plan_single.stnplan, plan_double.stnplan
#                                   compile() output flattened by include/stemtn_b200/flatten.hpp
#   meta.json                       generation parameters and plan summary
#   ref_<precision>.bin / .json     reference run_subtask values per slice (+ run_scheme sum)
# Large files are gzipped afterwards (the tests read both forms).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
TOOL="$HERE/../../oracle/_ref/ref_tool"
[ -x "$TOOL" ] || { echo "build the reference tool first: make -C oracle ref"; exit 1; }
T=${THREADS:-8}

circuit() {  # name layout cycles open target_cw golden-slices scheme-sum precisions...
  local name=$1 layout=$2 m=$3 open=$4 tcw=$5 slices=$6 sum=$7; shift 7
  local d="$HERE/$name"; mkdir -p "$d"
  "$TOOL" gen-circuit "$d" --layout "$layout" --cycles "$m" --open "$open" --target-cw "$tcw" > /dev/null
  for p in "$@"; do
    "$TOOL" golden "$d" --precision "$p" --slices "$slices" --scheme "$sum" --threads "$T" > /dev/null
  done
}

slice0() {  # name precision: the reference's run_subtask on slice 0 only (15-90 CPU-minutes
            # per 53-qubit slice), no uncached rerun
  "$TOOL" golden "$HERE/$1" --precision "$2" --slices 0 --scheme 0 --uncached 0 --threads 1 > /dev/null
}

random_net() {  # name seed vertices extra open hyper mixed target_cw merge
  local name=$1; local d="$HERE/$name"; mkdir -p "$d"
  "$TOOL" gen-random "$d" --seed "$2" --vertices "$3" --extra "$4" --open "$5" --hyper "$6" \
    --mixed "$7" --target-cw "$8" --merge-min-dim "$9" --light 1 --width-budget 30 > /dev/null
  for p in single double; do
    "$TOOL" golden "$d" --precision "$p" --slices all --scheme 1 --merge-min-dim "$9" \
      --width-budget 30 > /dev/null
  done
}

# Small cases mirroring proj/tests/test_runtime.cpp (hyperedges -> D>1 batches,
# mixed bond dimensions, sliced plans, merged and unmerged branches).
random_net rt_hyper_unmerged 1400 9 6 2 0.3 0 29 1
random_net rt_hyper_sliced   1401 9 7 2 0.3 0 3 32
random_net rt_cache_sliced   77   10 8 1 0.2 0 3 32
random_net rt_mixed_dims     21   8 6 1 0.2 1 4 32
random_net rt_unsliced       8    6 3 1 0.2 0 29 32
# 12-qubit batch-amplitude circuit (test_runtime.cpp:279-306 shape)
circuit rt_grid3x4_m4 grid3x4 4 6 10 all 1 single double
# sliced 12-qubit batch-amplitude circuit: 32 slices, 64 per-slice steps
circuit rt_grid3x4_m8_sliced grid3x4 8 6 6 all 1 single double

# BASELINE.json configs (cfg1..cfg5). Planner: PlannerParams defaults, seed 1.
circuit cfg1_grid4x5_m14 grid4x5 14 0 16 all 1 single double
# cfg2: three sampled slices plus the run_scheme sum over all 64 (~1 CPU-hour per precision)
circuit cfg2_grid5x6_m16 grid5x6 16 6 28 sample:3 1 single double
circuit cfg3_syc53_m12   sycamore53 12 6 29 none 0
circuit cfg4_syc53_m14   sycamore53 14 6 29 none 0
circuit cfg5_syc53_m20   sycamore53 20 6 33 none 0
# 53-qubit slices: slice 0 through the reference executor itself
# cfg3 single: slices 0 and 16383 (the last: every sliced digit at its maximum)
"$TOOL" golden "$HERE/cfg3_syc53_m12" --precision single --slices 0,16383 --scheme 0 --uncached 0 --threads 2 > /dev/null
slice0 cfg3_syc53_m12 double
# cfg4 single: slices 0 and 524287 (the last)
"$TOOL" golden "$HERE/cfg4_syc53_m14" --precision single --slices 0,524287 --scheme 0 --uncached 0 --threads 2 > /dev/null
slice0 cfg4_syc53_m14 double
# cfg5: the reference cannot hold its 2^33 stems (Engine::gemm keeps 4 of them, 256 GiB)
# and refuses every assignment (subtasks() overflows, scheme.hpp:33-37); its slices 0, 1
# and 11400714819323198485 (digits across 64 of its 85 sliced edges) come from the oracle
# port on a GPU box host: CFG5_SLICES=... scripts/cfg5_parity.py, then
# scripts/port_golden.py -> port_single.bin
# (tests/test_gpu_parity.py::test_cfg5_2pow33_stems_against_the_oracle_port)
