set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s -k "fast_mode or streams" 2>&1 | grep -E "err|passed|failed|assert|Error" | head -30
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python scripts/streams_ab.py cfg2 64 1 2 3 2>&1 | tail -6
timeout 600 python scripts/streams_ab.py cfg1 16 1 2 4 2>&1 | tail -6
timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_d.json > gpurun_out/steps_cfg5_d.txt 2>&1; head -8 gpurun_out/steps_cfg5_d.txt
timeout 600 python scripts/step_profile.py cfg4 fast 4 gpurun_out/steps_cfg4_d.json > gpurun_out/steps_cfg4_d.txt 2>&1; head -5 gpurun_out/steps_cfg4_d.txt
timeout 600 python scripts/step_profile.py cfg3 fast 4 gpurun_out/steps_cfg3_d.json > gpurun_out/steps_cfg3_d.txt 2>&1; head -5 gpurun_out/steps_cfg3_d.txt
for B in 10 12; do STN_DEBUG=sweep_bits=$B,sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_sweep$B.json > gpurun_out/steps_cfg5_sweep$B.txt 2>&1; grep -v "^ *stage" gpurun_out/steps_cfg5_sweep$B.txt | grep -E "sweep [0-9]+:|slices" | head -30; done
