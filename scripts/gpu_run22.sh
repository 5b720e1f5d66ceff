rm -rf gpurun_out; mkdir -p gpurun_out
for d in 0 2; do STN_SWEEP_DBG=$d timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r22_prof_$d.txt 2>&1; echo prof$d=$?; done
for d in 0 2; do echo "== dbg $d"; grep -A12 "ms/slice" gpurun_out/r22_prof_$d.txt; done
