set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "fused_chains" 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -30
