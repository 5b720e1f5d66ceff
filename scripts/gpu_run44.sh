rm -rf gpurun_out; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -s -k bitperm 2>&1 | grep -E "bitperm|passed|failed"
STN_BITPERM_LEGACY=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -s -k bitperm 2>&1 | grep -E "bitperm|passed|failed"
timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r44_prof.txt 2>&1; head -16 gpurun_out/r44_prof.txt; grep -E "^ (736|737|738|637) " gpurun_out/r44_prof.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
