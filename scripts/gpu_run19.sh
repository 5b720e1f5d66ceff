rm -rf gpurun_out; mkdir -p gpurun_out
for d in 0 1 2 3; do STN_SWEEP_DBG=$d timeout 600 python scripts/step_profile.py cfg2 > gpurun_out/r19_prof_$d.txt 2>&1; echo prof$d=$?; done
for d in 0 1 2 3; do echo "== dbg $d"; grep sweep gpurun_out/r19_prof_$d.txt | head -12; done
