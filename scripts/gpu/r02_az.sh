set -x
timeout 1200 python scripts/ab_compare.py cfg5 4 3 "chain_ffma2=0" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 3 "chain_ffma2=0" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg4 8 2 "chain_ffma2=0" "" 2>&1 | grep -E "median|rror"
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_az.json > gpurun_out/steps_cfg5_az.txt 2>&1; grep -E "slices|rror" gpurun_out/steps_cfg5_az.txt; sed -n '/step kernel/,+16p' gpurun_out/steps_cfg5_az.txt
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python scripts/fast_errors.py gpurun_out/fast_errors_az.json 2>&1 | grep -E "cfg(2|3|4|5)" | cut -c1-220
