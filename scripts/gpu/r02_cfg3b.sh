set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "53" 2>&1 | tail -2
