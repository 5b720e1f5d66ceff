rm -rf gpurun_out; mkdir -p gpurun_out
timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r58_prof.txt 2>&1; head -2 gpurun_out/r58_prof.txt | tail -1; grep absorb_tc gpurun_out/r58_prof.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
