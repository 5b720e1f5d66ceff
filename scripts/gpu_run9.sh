set -x
rm -rf gpurun_out/*.ncu-rep
python -m pytest tests/test_gpu_kernels.py -q -s -k bitperm --timeout 300 -p no:cacheprovider > gpurun_out/bitperm.log 2>&1; echo bitperm=$?
CMD="python scripts/ncu_target.py cfg2 2"
if timeout 300 $CMD > gpurun_out/ncu_target_plain.log 2>&1; then
  for K in "k_absorb3ILb0ELb0ELi4ELi4ELb0E" "k_absorb3ILb0ELb0ELi4ELi4ELb1E" "k_absorb_tcILi32ELi32E" "k_absorb3ILb0ELb1E"; do
    timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k "regex:$K" -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_$K.log 2>&1; echo ncu_$K=$?
  done
  python scripts/ncu_summary.py gpurun_out/ncu_r9_summary.md gpurun_out/prof_*.ncu-rep > /dev/null 2>&1
  for f in gpurun_out/prof_*.ncu-rep; do ncu -i $f --page details --csv > ${f%.ncu-rep}_details.csv 2>/dev/null; ncu -i $f --page source --csv > ${f%.ncu-rep}_source.csv 2>/dev/null; done
  ls -la gpurun_out/
  find gpurun_out -name "*.ncu-rep" -size +20M -delete
fi
grep -E "bitperm" gpurun_out/bitperm.log; cat gpurun_out/ncu_r9_summary.md
