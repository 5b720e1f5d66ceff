mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "large_config" -s 2>&1 | grep -E "err|passed|failed"
timeout 600 python scripts/step_profile.py cfg4 > gpurun_out/r81_prof_cfg4.txt 2>&1; echo cfg4=$?; sed -n 2,8p gpurun_out/r81_prof_cfg4.txt; grep " 1081 " gpurun_out/r81_prof_cfg4.txt
