set -x
python -m pytest tests/test_gpu_kernels.py -q -s --timeout 300 -p no:cacheprovider > gpurun_out/kern.log 2>&1; echo kern=$?
timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/step_profile_cfg2.txt 2>&1; echo prof=$?
timeout 1800 python -m pytest tests -m gpu -q -s --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_cfg2.log 2>&1; echo bench=$?
grep -E "tc gemm" gpurun_out/kern.log; tail -3 gpurun_out/kern.log; head -45 gpurun_out/step_profile_cfg2.txt; grep -E "cfg3|cfg4|FAIL|passed|failed" gpurun_out/pytest_gpu.log | tail -12; tail -c 300 gpurun_out/bench_cfg2.log
