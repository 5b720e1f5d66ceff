rm -rf gpurun_out; mkdir -p gpurun_out
export STN_ABSORB_LOADER=tma
timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r42_prof.txt 2>&1; head -40 gpurun_out/r42_prof.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
