set -x
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_w.json > gpurun_out/steps_cfg5_w.txt 2>&1; grep -E "chain kernel|slices" gpurun_out/steps_cfg5_w.txt | head -40
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg2 fast 16 gpurun_out/steps_cfg2_w.json > gpurun_out/steps_cfg2_w.txt 2>&1; grep -E "chain kernel|^chain|slices" gpurun_out/steps_cfg2_w.txt | head -30
