rm -rf gpurun_out; mkdir -p gpurun_out
export STN_TMA_MIN_BITS=6
for d in 0 7; do echo "== dbg $d"; STN_TMA_DBG=$d timeout 300 python scripts/step_profile.py cfg2 2>&1 | grep -E "ms/slice over|^ (477|485|489|494|536|559|592|508|588) "; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
