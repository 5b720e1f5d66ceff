set -x
timeout 900 python scripts/ab_compare.py cfg5 4 3 "" "chain_swap=0" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg4 8 3 "" "chain_swap=0" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 3 "" "chain_swap=0" 2>&1 | grep -E "median|rror"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_chains or cfg2 or cfg1 or cfg5" 2>&1 | tail -2
