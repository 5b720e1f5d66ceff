rm -rf gpurun_out; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r43_pytest.log 2>&1; echo pytest=$?
timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r43_prof.txt 2>&1; echo prof=$?
timeout 1200 python bench.py > gpurun_out/r43_bench.log 2>&1; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r43_launches.csv python scripts/ncu_target.py cfg2 1 > gpurun_out/r43_l.log 2>&1; echo ncu=$?
tail -3 gpurun_out/r43_pytest.log; head -3 gpurun_out/r43_prof.txt; tail -c 1500 gpurun_out/r43_bench.log
