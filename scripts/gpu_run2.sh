set -x
python -m pytest tests/test_gpu_kernels.py -q -s --timeout 300 -p no:cacheprovider > gpurun_out/kern.log 2>&1; echo kern=$?
timeout 1500 python -m pytest tests -m gpu -q -s --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
CMD="python bench.py --config cfg2 --steps 2 --warmup 1 --cpu-baseline 0 --e2e-steps 0"
if timeout 900 $CMD > gpurun_out/bench_cfg2_plain.log 2>&1; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_absorb|k_gemm" -s 20 -c 4 -o gpurun_out/prof_cfg2 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
fi
tail -3 gpurun_out/kern.log; grep -E "tc gemm" gpurun_out/kern.log; tail -8 gpurun_out/pytest_gpu.log; tail -c 2500 gpurun_out/bench_cfg2_plain.log
