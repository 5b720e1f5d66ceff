rm -rf gpurun_out; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r27_pytest.log 2>&1; echo pytest=$?
timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r27_prof.txt 2>&1; echo prof=$?
timeout 1200 python bench.py > gpurun_out/r27_bench.log 2>&1; echo bench=$?
tail -3 gpurun_out/r27_pytest.log; head -14 gpurun_out/r27_prof.txt; tail -c 1200 gpurun_out/r27_bench.log
