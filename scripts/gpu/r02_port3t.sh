set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg5" -s 2>&1 | grep -E "cfg5 slice|passed|failed|Error" | head
timeout 900 python scripts/fast_errors.py gpurun_out/fast_errors_p3.json 2>&1 | grep cfg5 | cut -c1-200
