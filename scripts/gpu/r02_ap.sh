set -x
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_ap.json > gpurun_out/steps_cfg5_ap.txt 2>&1; grep -E "^chain [0-9]|slices|rror" gpurun_out/steps_cfg5_ap.txt | head -60; sed -n '/step kernel/,+20p' gpurun_out/steps_cfg5_ap.txt
timeout 900 python scripts/ab_compare.py cfg5 4 3 "chain_exp=0" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 2 "chain_exp=0" "" 2>&1 | grep -E "median|rror"
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
