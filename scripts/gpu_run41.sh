rm -rf gpurun_out; mkdir -p gpurun_out
export STN_TMA_MIN_BITS=6 STN_ABSORB_LOADER=tma
for d in 0 1 2 4 3 5 6; do echo "== dbg $d"; STN_TMA_DBG=$d timeout 300 python scripts/step_profile.py cfg2 2>&1 | grep -E "^ (477|485|536|508) "; done
