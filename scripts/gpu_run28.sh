rm -rf gpurun_out; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r28_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r28_pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r28_smoke.log 2>&1; echo smoke=$?
timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r28_prof.txt 2>&1; echo prof=$?
timeout 1200 python bench.py > gpurun_out/r28_bench.log 2>&1; echo bench=$?
tail -3 gpurun_out/r28_pytest.log; tail -3 gpurun_out/r28_smoke.log; head -14 gpurun_out/r28_prof.txt; tail -c 1500 gpurun_out/r28_bench.log
