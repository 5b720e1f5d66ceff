set -x
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_o.json > gpurun_out/steps_cfg5_o.txt 2>&1; grep -E "slices|Error|error|jit" gpurun_out/steps_cfg5_o.txt | head -5; grep -E "^ *[0-9]+ " gpurun_out/steps_cfg5_o.txt | head -14
STN_DEBUG=chain_min_bits=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "exact or cfg5" 2>&1 | tail -2
timeout 900 python bench.py --config cfg5 > gpurun_out/bench_cfg5_o.json 2> gpurun_out/bench_cfg5_o.err; tail -2 gpurun_out/bench_cfg5_o.err; cut -c1-300 gpurun_out/bench_cfg5_o.json
