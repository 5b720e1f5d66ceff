mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r76_prof.txt 2>&1; echo prof=$?; sed -n 2p gpurun_out/r76_prof.txt; grep -E "^ *(485|488|475|546|568|583) " gpurun_out/r76_prof.txt
