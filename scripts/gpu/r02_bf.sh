set -x
timeout 1500 python scripts/ab_compare.py cfg5 8 3 "chain_alt=0" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 3 "chain_alt=0" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg4 16 2 "chain_alt=0" "" 2>&1 | grep -E "median|rror"
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_bf.json > gpurun_out/steps_cfg5_bf.txt 2>&1; grep -E "slices|rror|-> " gpurun_out/steps_cfg5_bf.txt | head -60
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
