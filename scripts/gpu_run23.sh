rm -rf gpurun_out; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r23_pytest.log 2>&1; echo pytest=$?
STN_SWEEP_DEBUG=1 timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r23_prof.txt 2>&1; echo prof=$?
STN_SWEEP_BITS=0 timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r23_prof_nosweep.txt 2>&1; echo prof=$?
tail -30 gpurun_out/r23_pytest.log | grep -v "^$" | tail -25; grep -A22 "ms/slice" gpurun_out/r23_prof.txt; grep -A22 "ms/slice" gpurun_out/r23_prof_nosweep.txt
