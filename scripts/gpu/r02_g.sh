set -x
STN_DEBUG=chain_min_bits=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "exact or fast_mode" 2>&1 | tail -4
timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_g.json > gpurun_out/steps_cfg5_g.txt 2>&1; grep -E "slices|Error|error" gpurun_out/steps_cfg5_g.txt | head; grep -E " sweep " gpurun_out/steps_cfg5_g.txt | head -12
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
