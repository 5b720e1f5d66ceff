rm -rf gpurun_out; mkdir -p gpurun_out
for d in 7 15; do echo "== dbg $d"; STN_TMA_DBG=$d timeout 300 python scripts/step_profile.py cfg2 2>&1 | grep -E "^ (477|485|536|508) "; done
