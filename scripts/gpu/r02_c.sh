set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -s 2>&1 | grep -E "gemm|passed|failed|Error" | head -40
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for T in 0 1; do STN_DEBUG=tcf=$T timeout 600 python scripts/step_profile.py cfg4 fast 4 gpurun_out/steps_cfg4_c_tcf$T.json > gpurun_out/steps_cfg4_c_tcf$T.txt 2>&1; head -6 gpurun_out/steps_cfg4_c_tcf$T.txt; done
for T in 0 1; do STN_DEBUG=tcf=$T timeout 600 python scripts/step_profile.py cfg5 fast 2 gpurun_out/steps_cfg5_c_tcf$T.json > gpurun_out/steps_cfg5_c_tcf$T.txt 2>&1; head -8 gpurun_out/steps_cfg5_c_tcf$T.txt; done
for T in 0 1; do STN_DEBUG=tcf=$T timeout 600 python scripts/step_profile.py cfg3 fast 4 gpurun_out/steps_cfg3_c_tcf$T.json > gpurun_out/steps_cfg3_c_tcf$T.txt 2>&1; head -6 gpurun_out/steps_cfg3_c_tcf$T.txt; done
timeout 600 python scripts/step_profile.py cfg2 fast 64 gpurun_out/steps_cfg2_c.json > gpurun_out/steps_cfg2_c.txt 2>&1; head -3 gpurun_out/steps_cfg2_c.txt
