rm -rf gpurun_out; mkdir -p gpurun_out
for v in gather tma; do echo "== loader $v"; STN_ABSORB_LOADER=$v timeout 300 python scripts/step_profile.py cfg2 > gpurun_out/r36_prof_$v.txt 2>&1; grep -E "ms/slice over" gpurun_out/r36_prof_$v.txt; grep -E "^ (477|485|488|489|494|536|559|592|508|588) " gpurun_out/r36_prof_$v.txt; done
STN_TMA_DBG=7 timeout 300 python scripts/step_profile.py cfg2 2>&1 | grep -E "^ (477|485|536|508) "
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
