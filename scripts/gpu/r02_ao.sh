set -x
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_ao.json > gpurun_out/steps_cfg5_ao.txt 2>&1; grep -E "^chain [0-9]|slices|rror" gpurun_out/steps_cfg5_ao.txt | head -60; sed -n '/step kernel/,+14p' gpurun_out/steps_cfg5_ao.txt
timeout 900 python scripts/ab_compare.py cfg5 4 3 "chain_exp=0" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg4 8 2 "chain_exp=0" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 2 "chain_exp=0" "" 2>&1 | grep -E "median|rror"
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
