set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -2
STN_DEBUG=sweep_debug timeout 600 python scripts/step_profile.py cfg4 fast 4 gpurun_out/steps_cfg4_bi.json > gpurun_out/steps_cfg4_bi.txt 2>&1; grep -E "slices|rror" gpurun_out/steps_cfg4_bi.txt; sed -n '/step kernel/,+8p' gpurun_out/steps_cfg4_bi.txt
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
