set -x
timeout 1800 python -m pytest tests -m gpu -q -s --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/step_profile_cfg2_default.txt 2>&1; echo prof=$?
STN_NO_BULK=1 timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/step_profile_cfg2_nobulk.txt 2>&1; echo prof2=$?
CMD="python scripts/ncu_target.py cfg2 2"
if timeout 300 $CMD > gpurun_out/ncu_target_plain.log 2>&1; then
  for K in "k_absorb3ILb0ELb0ELi4ELi4ELb0E" "k_absorb3ILb0ELb0ELi4ELi4ELb1E" "k_absorb_tcILi32ELi32E"; do
    timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:$K" -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_$K.log 2>&1; echo ncu_$K=$?
  done
fi
grep -E "FAIL|passed|failed" gpurun_out/pytest_gpu.log | tail -5; head -25 gpurun_out/step_profile_cfg2_default.txt; head -12 gpurun_out/step_profile_cfg2_nobulk.txt
