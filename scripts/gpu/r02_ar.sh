set -x
STN_DEBUG=sweep_debug,chain_multi_log=6 timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_ar.json > gpurun_out/steps_cfg5_ar.txt 2>&1; grep -E "li 6|slices|rror" gpurun_out/steps_cfg5_ar.txt | head -60; sed -n '/step kernel/,+14p' gpurun_out/steps_cfg5_ar.txt
timeout 900 python scripts/ab_compare.py cfg5 4 3 "" "chain_multi_log=6" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 2 "" "chain_multi_log=6" 2>&1 | grep -E "median|rror"
