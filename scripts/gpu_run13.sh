set -x
for L in 4 2 3; do
  STN_DIRECT_MIN_L=$L timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/step_profile_cfg2_L$L.txt 2>&1; echo prof_$L=$?
done
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --cpu-baseline 0 > gpurun_out/bench_cfg2_n1.log 2>&1; echo bench1=$?
for L in 4 2 3; do head -12 gpurun_out/step_profile_cfg2_L$L.txt; done; tail -c 300 gpurun_out/bench_cfg2_n1.log
