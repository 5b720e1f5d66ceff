set -x
timeout 1500 python scripts/ab_compare.py cfg5 8 3 "chain_wreg=0" "" "chain_wreg=48" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 3 "chain_wreg=0" "" "chain_wreg=48" 2>&1 | grep -E "median|rror"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_chains or cfg5" 2>&1 | tail -2
