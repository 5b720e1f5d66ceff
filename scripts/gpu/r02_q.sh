set -x
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_q.json > gpurun_out/steps_cfg5_q.txt 2>&1; grep -E "^chain (1[0-9]|2[0-9]):|slices|Error|error" gpurun_out/steps_cfg5_q.txt | head -20; grep -E "^ *[0-9]+ " gpurun_out/steps_cfg5_q.txt | head -12
date; timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -4; date
