set -x
timeout 1800 python -m pytest tests -m gpu -q -s --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/step_profile_cfg2_default.txt 2>&1; echo prof=$?
timeout 900 python scripts/run_cfg5.py 2 > gpurun_out/cfg5.log 2>&1; echo cfg5=$?
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_cfg2.log 2>&1; echo bench=$?
grep -E "FAIL|passed|failed" gpurun_out/pytest_gpu.log | tail -5; head -30 gpurun_out/step_profile_cfg2_default.txt; cat gpurun_out/cfg5.log | tail -20; tail -c 300 gpurun_out/bench_cfg2.log
