set -x
timeout 600 python scripts/bench_diag.py cfg5 6 2>&1 | grep -E "ms/slice|rror"
timeout 900 python scripts/ab_compare.py cfg5 4 3 "side=0" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg4 8 3 "side=0" "" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 3 "side=0" "" 2>&1 | grep -E "median|rror"
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
