set -x
nproc
python -m pytest tests/test_gpu_kernels.py -q -s --timeout 300 -p no:cacheprovider > gpurun_out/kern.log 2>&1; echo kern=$?
timeout 1800 python -m pytest tests -m gpu -q -s --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
CMD="python bench.py --config cfg2 --steps 2 --warmup 1 --cpu-baseline 0 --e2e-steps 0"
if timeout 900 $CMD > gpurun_out/bench_cfg2_plain.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_absorb2|k_gemm_tc|k_gemm_simt|k_generic|k_splitk" -s 40 -c 8 -o gpurun_out/prof_cfg2_r3 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
fi
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --cpu-budget 20 > gpurun_out/bench_cfg2_full.log 2>&1; echo bench=$?
python scripts/step_profile.py cfg2 > gpurun_out/step_profile_cfg2.txt 2>&1
tail -3 gpurun_out/kern.log; grep -E "tc gemm" gpurun_out/kern.log; tail -8 gpurun_out/pytest_gpu.log; tail -c 3000 gpurun_out/bench_cfg2_full.log
