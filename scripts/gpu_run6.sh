set -x
timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/step_profile_cfg2.txt 2>&1; echo prof=$?
CMD="python scripts/ncu_target.py cfg2 2"
if timeout 300 $CMD > gpurun_out/ncu_target_plain.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 700 -c 400 --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
  for K in "k_absorb_tc<16, 16>" "k_absorb_tc<16, 8>" "k_absorb2<false, false, 4, 4, false>" "k_absorb2<false, false, 4, 4, true>" "k_gemm_tc" "k_splitk_partial"; do
    tag=$(echo "$K" | tr -cd 'a-z0-9_')
    timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" -c 1 -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_$tag.log 2>&1; echo ncu_$tag=$?
  done
fi
head -30 gpurun_out/step_profile_cfg2.txt
