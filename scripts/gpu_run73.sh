mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r73_prof.txt 2>&1; echo prof=$?; sed -n 2p gpurun_out/r73_prof.txt; grep " 750 " gpurun_out/r73_prof.txt
STN_PLAN_TIMING=1 timeout 300 python scripts/e2e_breakdown.py 2>&1 | tail -9
