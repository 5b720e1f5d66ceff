set -x
timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_j.json > gpurun_out/steps_cfg5_j.txt 2>&1; grep -E "slices|Error|error" gpurun_out/steps_cfg5_j.txt | head; grep -E " sweep " gpurun_out/steps_cfg5_j.txt | head -12
STN_DEBUG=chain_min_bits=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "exact or cfg5" 2>&1 | tail -2
timeout 600 python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_plain_j.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:k_chain -s 22 -c 1 -o gpurun_out/chain_j python scripts/ncu_target.py cfg5 1 > gpurun_out/ncu_j.log 2>&1; tail -1 gpurun_out/ncu_j.log
