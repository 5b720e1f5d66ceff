set -x
timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_v.json > gpurun_out/steps_cfg5_v.txt 2>&1; grep -E "slices|Error|error" gpurun_out/steps_cfg5_v.txt | head -3; grep -E " sweep " gpurun_out/steps_cfg5_v.txt | head -8
timeout 600 python scripts/step_profile.py cfg2 fast 16 gpurun_out/steps_cfg2_v.json > gpurun_out/steps_cfg2_v.txt 2>&1; grep -E "slices|Error|error" gpurun_out/steps_cfg2_v.txt | head -3; grep -E " sweep " gpurun_out/steps_cfg2_v.txt | head -4
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "fast or cfg5 or 53" 2>&1 | tail -2
