rm -rf gpurun_out; mkdir -p gpurun_out
STN_PLAN_DUMP=1 timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r32_prof.txt 2> gpurun_out/r32_dump.txt; echo prof=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r32_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r32_pytest.log; head -30 gpurun_out/r32_prof.txt; grep -c tma gpurun_out/r32_dump.txt; tail -5 gpurun_out/r32_dump.txt
