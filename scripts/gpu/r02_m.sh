set -x
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_m.json > gpurun_out/steps_cfg5_m.txt 2>&1; grep -E "slices|Error|error|jit" gpurun_out/steps_cfg5_m.txt | head; grep -E " sweep " gpurun_out/steps_cfg5_m.txt | head -8
STN_DEBUG=chain_min_bits=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "exact or fast or cfg5" 2>&1 | tail -2
