set -x
timeout 900 python scripts/ab_compare.py cfg5 4 3 "chain_single=0" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg4 8 3 "chain_single=0" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 3 "chain_single=0" "" 2>&1 | grep -E "median|rror"
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
