rm -rf gpurun_out; mkdir -p gpurun_out
for d in 0 1 2 4 7; do echo "== dbg $d"; STN_TMA_DBG=$d timeout 300 python scripts/step_profile.py cfg2 2>&1 | grep -E "^ (477|485|536|508) "; done
timeout 600 ncu --set full --clock-control none -k regex:absorb_tma -s 2 -c 2 -o gpurun_out/r34_tma python scripts/ncu_target.py cfg2 1 > gpurun_out/r34_ncu.log 2>&1; echo ncu=$?
