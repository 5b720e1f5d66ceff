set -x
for POL in default simt tc; do
  if [ $POL = default ]; then unset STN_ABSORB_POLICY; else export STN_ABSORB_POLICY=$POL; fi
  timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/step_profile_cfg2_$POL.txt 2>&1; echo prof_$POL=$?
done
unset STN_ABSORB_POLICY
CMD="python scripts/ncu_target.py cfg2 2"
if timeout 300 $CMD > gpurun_out/ncu_target_plain.log 2>&1; then
  for K in "k_absorb_tc<16. 16>" "k_absorb2<0. 0. 4. 4. 0>" "k_absorb2<0. 0. 4. 4. 1>" "k_splitk_partial"; do
    tag=$(echo "$K" | tr -cd 'a-z0-9_')
    timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" -c 1 -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_$tag.log 2>&1; echo ncu_$tag=$?
  done
fi
head -12 gpurun_out/step_profile_cfg2_default.txt; head -3 gpurun_out/step_profile_cfg2_simt.txt; head -3 gpurun_out/step_profile_cfg2_tc.txt
