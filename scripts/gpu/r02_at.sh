set -x
STN_DEBUG=sweep_debug,chain_multi_log=6 timeout 600 python scripts/step_profile.py cfg2 fast 16 gpurun_out/steps_cfg2_at.json > gpurun_out/steps_cfg2_at.txt 2>&1; grep -E "^chain|slices|rror" gpurun_out/steps_cfg2_at.txt | head -60; sed -n '/step kernel/,+12p' gpurun_out/steps_cfg2_at.txt
STN_DEBUG=sweep_debug,chain_multi_log=6 timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_at.json > gpurun_out/steps_cfg5_at.txt 2>&1; grep -E "^chain|slices|rror" gpurun_out/steps_cfg5_at.txt | head -100; sed -n '/step kernel/,+25p' gpurun_out/steps_cfg5_at.txt
