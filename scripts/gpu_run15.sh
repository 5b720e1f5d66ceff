set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r15_pytest.log 2>&1; echo pytest=$?
timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r15_prof_sweep.txt 2>&1; echo prof=$?
STN_SWEEP_BITS=0 timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r15_prof_nosweep.txt 2>&1; echo prof0=$?
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-baseline 0 > gpurun_out/r15_bench.log 2>&1; echo bench=$?
tail -25 gpurun_out/r15_pytest.log; head -30 gpurun_out/r15_prof_sweep.txt; head -8 gpurun_out/r15_prof_nosweep.txt; head -c 700 gpurun_out/r15_bench.log
