set -x
STN_DEBUG=sweep_debug,chain_why=1605 timeout 600 python scripts/step_profile.py cfg5 fast 1 > gpurun_out/why_1605.txt 2>&1; grep -E "no fit|^chain [0-9]+: steps 16" gpurun_out/why_1605.txt | head
STN_DEBUG=chain_why=1155 timeout 600 python scripts/step_profile.py cfg5 fast 1 > gpurun_out/why_1155.txt 2>&1; grep -E "no fit" gpurun_out/why_1155.txt | head
