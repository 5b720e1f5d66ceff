rm -rf gpurun_out; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r20_pytest.log 2>&1; echo pytest=$?
STN_SWEEP_DEBUG=1 timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r20_prof_0.txt 2>&1; echo prof0=$?
STN_SWEEP_DBG=2 timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r20_prof_2.txt 2>&1; echo prof2=$?
tail -3 gpurun_out/r20_pytest.log
for d in 0 2; do echo "== dbg $d"; grep -A14 "ms/slice" gpurun_out/r20_prof_$d.txt; done
