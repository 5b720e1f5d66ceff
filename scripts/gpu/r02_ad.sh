set -x
timeout 900 python scripts/ab_compare.py cfg5 4 3 "" "chain_single=1" "chain_single=1,chain_vec=0" "chain_vec=0" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg4 8 3 "" "chain_single=1" "chain_single=1,chain_vec=0" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 3 "" "chain_single=1" "chain_single=1,chain_vec=0" 2>&1 | grep -E "median|rror"
STN_DEBUG=sweep_debug,chain_single=1 timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_ad.json > gpurun_out/steps_cfg5_ad.txt 2>&1; grep -E "slices" gpurun_out/steps_cfg5_ad.txt
