timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r16_pytest.log 2>&1; echo pytest=$?
timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r16_prof_sweep.txt 2>&1; echo prof=$?
STN_SWEEP_BITS=11 timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r16_prof_sweep11.txt 2>&1; echo prof=$?
tail -5 gpurun_out/r16_pytest.log; head -40 gpurun_out/r16_prof_sweep.txt; head -12 gpurun_out/r16_prof_sweep11.txt
