set -x
rm -f gpurun_out/*.ncu-rep gpurun_out/*_source.csv gpurun_out/*_details.csv
CMD="python bench.py --steps 2 --warmup 1 --cpu-baseline 0 --e2e-steps 1"
if timeout 900 $CMD > gpurun_out/r14_plain.log 2>&1; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 700 -c 300 --csv --log-file gpurun_out/r14_launches.csv $CMD > gpurun_out/r14_ncu_launch.log 2>&1; echo ncu1=$?
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_absorb_direct" -s 5 -c 2 -o gpurun_out/r14_direct $CMD > gpurun_out/r14_ncu_direct.log 2>&1; echo ncu2=$?
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:k_gemm_tc" -s 4 -c 1 -o gpurun_out/r14_gemm_tc $CMD > gpurun_out/r14_ncu_gemm.log 2>&1; echo ncu3=$?
  python scripts/ncu_summary.py gpurun_out/r14_summary.md gpurun_out/r14_direct.ncu-rep gpurun_out/r14_gemm_tc.ncu-rep gpurun_out/r14_launches.csv > /dev/null 2>&1
  for f in gpurun_out/r14_direct.ncu-rep; do ncu -i $f --page details --csv > ${f%.ncu-rep}_details.csv 2>/dev/null; done
  find gpurun_out -name "*.ncu-rep" -size +30M -delete
fi
timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/step_profile_cfg2.txt 2>&1; echo prof=$?
timeout 1200 python bench.py > gpurun_out/r14_bench_default.log 2>&1; echo bench=$?
cat gpurun_out/r14_summary.md | head -60; head -30 gpurun_out/step_profile_cfg2.txt; tail -c 1500 gpurun_out/r14_bench_default.log
