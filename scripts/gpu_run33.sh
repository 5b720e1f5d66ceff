rm -rf gpurun_out; mkdir -p gpurun_out
for nsr in 4 6 10; do echo "== nsr $nsr"; STN_TMA_NSR=$nsr timeout 300 python scripts/step_profile.py cfg2 2>&1 | grep -E "ms/slice over|^ (477|485|488|536|592|559|508|588) "; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
