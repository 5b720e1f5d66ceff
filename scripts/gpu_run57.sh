rm -rf gpurun_out; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -s -k tc_gemm 2>&1 | grep -E "err|passed|failed|Error" | head -20
for bn in 128 256; do echo "== bn $bn"; for c in cfg2 cfg4; do STN_GEMM_BN=$bn timeout 600 python scripts/step_profile.py $c 2>&1 | grep -E "ms/slice over|gemm_tc" | head -4; done; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
