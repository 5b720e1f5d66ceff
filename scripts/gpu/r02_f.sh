set -x
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_f.json > gpurun_out/steps_cfg5_f.txt 2>&1; grep -E "^chain|slices|Error|error" gpurun_out/steps_cfg5_f.txt | head -30; grep -E " sweep " gpurun_out/steps_cfg5_f.txt | head -12
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
STN_DEBUG=chain_min_bits=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "exact or fast_mode or streams" 2>&1 | tail -4
STN_DEBUG=chain=0 timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_f0.json > gpurun_out/steps_cfg5_f0.txt 2>&1; grep -E "slices" gpurun_out/steps_cfg5_f0.txt
for C in cfg2 cfg4 cfg3; do timeout 600 python scripts/step_profile.py $C fast 4 gpurun_out/steps_${C}_f.json > gpurun_out/steps_${C}_f.txt 2>&1; grep -E "slices" gpurun_out/steps_${C}_f.txt; done
