set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
STN_LANES=all timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "exact or fast_mode" 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
for L in 0 1 all; do STN_LANES=$L timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_lanes_$L.json > gpurun_out/steps_cfg5_lanes_$L.txt 2>&1; head -4 gpurun_out/steps_cfg5_lanes_$L.txt; done
for L in 0 all; do STN_LANES=$L timeout 600 python scripts/step_profile.py cfg2 fast 64 gpurun_out/steps_cfg2_lanes_$L.json > gpurun_out/steps_cfg2_lanes_$L.txt 2>&1; head -3 gpurun_out/steps_cfg2_lanes_$L.txt; done
timeout 600 python bench.py --config cfg5 --steps 3 --warmup 2 --cpu-baseline 0 > gpurun_out/bench_cfg5_a.json 2> gpurun_out/bench_cfg5_a.err; tail -3 gpurun_out/bench_cfg5_a.err; cat gpurun_out/bench_cfg5_a.json
timeout 2400 python scripts/cfg5_parity.py > gpurun_out/cfg5_parity.log 2>&1; tail -8 gpurun_out/cfg5_parity.log
