set -x
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_ay.json > gpurun_out/steps_cfg5_ay.txt 2>&1; grep -E "^chain [0-9]|chain kernel|slices|rror" gpurun_out/steps_cfg5_ay.txt | sort -u | head -120; sed -n '/step kernel/,+40p' gpurun_out/steps_cfg5_ay.txt
