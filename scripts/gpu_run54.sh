rm -rf gpurun_out; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r54_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r54_smoke.log 2>&1; echo smoke=$?
timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r54_prof.txt 2>&1; echo prof=$?
timeout 1200 python bench.py > gpurun_out/r54_bench.log 2>&1; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r54_launches.csv python scripts/ncu_target.py cfg2 1 > gpurun_out/r54_l.log 2>&1; echo ncu=$?
tail -2 gpurun_out/r54_pytest.log; tail -2 gpurun_out/r54_smoke.log; head -3 gpurun_out/r54_prof.txt; grep "^{" gpurun_out/r54_bench.log | cut -c1-300
