set -x
nproc; free -g | head -2; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --config cfg1 --steps 3 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_cfg1.log 2>&1; echo b1=$?
timeout 900 python bench.py --config cfg2 --steps 3 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_cfg2.log 2>&1; echo b2=$?
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -5; tail -c 3000 gpurun_out/bench_cfg2.log
