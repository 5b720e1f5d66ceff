set -x
timeout 900 python scripts/ab_compare.py cfg5 4 3 "" "chain_swap=0" "chain_vec=1" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg4 8 3 "" "chain_swap=0" "chain_vec=1" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 3 "" "chain_swap=0" "chain_vec=1" 2>&1 | grep -E "median|rror"
STN_DEBUG=sweep_debug,chain_swap=0 timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_ah.json > gpurun_out/steps_cfg5_ah.txt 2>&1; grep -E "slices" gpurun_out/steps_cfg5_ah.txt
