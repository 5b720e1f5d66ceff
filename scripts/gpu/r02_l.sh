set -x
timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_l.json > gpurun_out/steps_cfg5_l.txt 2>&1; grep -E "slices|Error|error" gpurun_out/steps_cfg5_l.txt | head; grep -E " sweep " gpurun_out/steps_cfg5_l.txt | head -8
STN_DEBUG=chain_min_bits=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "exact or cfg5" 2>&1 | tail -2
