rm -rf gpurun_out; mkdir -p gpurun_out
for cfg in "STN_MMA_MIN_BITS=8" "STN_MMA_MIN_BITS=10" "STN_MMA_MIN_BITS=8 STN_SWEEP_BITS=0" "STN_MMA_MIN_BITS=10 STN_SWEEP_BITS=0" "STN_MMA_MIN_BITS=99 STN_SWEEP_BITS=0"; do
  echo "== $cfg"; env $cfg timeout 300 python scripts/step_profile.py cfg2 2>&1 | grep -E "ms/slice over|^ (485|488|489|494|546|476|592|536) "
done
