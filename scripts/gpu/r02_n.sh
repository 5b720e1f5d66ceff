set -x
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_n.json > gpurun_out/steps_cfg5_n.txt 2>&1; grep -E "^chain|slices|Error|error|jit" gpurun_out/steps_cfg5_n.txt | head -40; grep -E " sweep " gpurun_out/steps_cfg5_n.txt | head -8
STN_DEBUG=chain_min_bits=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "exact or fast or cfg5" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for C in cfg2 cfg3 cfg4; do timeout 600 python scripts/step_profile.py $C fast 4 gpurun_out/steps_${C}_n.json > gpurun_out/steps_${C}_n.txt 2>&1; grep -E "slices" gpurun_out/steps_${C}_n.txt; done
