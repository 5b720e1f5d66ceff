set -x
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_i.json > gpurun_out/steps_cfg5_i.txt 2>&1; grep -E "^chain 2[0-9]|slices|Error|error" gpurun_out/steps_cfg5_i.txt | head; grep -E " sweep " gpurun_out/steps_cfg5_i.txt | head -12
STN_DEBUG=chain_min_bits=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "exact or fast_mode or cfg5" 2>&1 | tail -3
timeout 600 python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_plain_i.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:k_chain -c 1 -o gpurun_out/chain_i python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_i.log 2>&1; tail -2 gpurun_out/ncu_i.log
