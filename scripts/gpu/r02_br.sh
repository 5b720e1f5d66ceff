set -x
timeout 1500 python scripts/ab_compare.py cfg5 8 3 "" "chain_min_bits=22" "chain_min_bits=20" 2>&1 | grep -E "median|rror"
timeout 1200 python scripts/ab_compare.py cfg4 16 2 "" "gemm_gm=8" "gemm_gm=24" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg2 32 3 "" "chain_min_bits=22" "chain_min_bits=20" 2>&1 | grep -E "median|rror"
