rm -rf gpurun_out; mkdir -p gpurun_out
for d in 0 1 2 4 3 6 5 7; do echo "== dbg $d"; STN_SWEEP_BITS=0 STN_MMA_DBG=$d timeout 300 python scripts/step_profile.py cfg2 2>&1 | grep -E "^ (485|488|489|494|546) "; done
