mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r71_prof.txt 2>&1; echo prof=$?; head -12 gpurun_out/r71_prof.txt; grep -E "^ *(475|546|568|583|501|588|513) " gpurun_out/r71_prof.txt
