set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_chains or cfg5 or 53" 2>&1 | tail -2
timeout 1200 python scripts/ab_compare.py cfg5 4 3 "" "chain_exp_pen=0" "chain_multi_log=6" "chain_multi_log=6,chain_exp_pen=0" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 2 "" "chain_exp_pen=0" "chain_multi_log=6" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg4 8 2 "" "chain_multi_log=6" 2>&1 | grep -E "median|rror"
STN_DEBUG=sweep_debug,chain_exp_pen=0 timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_as.json > gpurun_out/steps_cfg5_as.txt 2>&1; grep -E "slices|rror" gpurun_out/steps_cfg5_as.txt; sed -n '/step kernel/,+12p' gpurun_out/steps_cfg5_as.txt
