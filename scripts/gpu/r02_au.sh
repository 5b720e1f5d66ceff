set -x
timeout 1200 python scripts/ab_compare.py cfg5 4 3 "chain_multi_log=5" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 3 "chain_multi_log=5" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg4 8 2 "chain_multi_log=5" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg3 8 2 "chain_multi_log=5" "" 2>&1 | grep -E "median|rror"
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg2 fast 16 gpurun_out/steps_cfg2_au.json > gpurun_out/steps_cfg2_au.txt 2>&1; grep -E "chain kernel|slices|rror" gpurun_out/steps_cfg2_au.txt | head -30
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
