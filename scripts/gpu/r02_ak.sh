set -x
timeout 1200 python scripts/ab_compare.py cfg4 8 3 "gemm_mc=2,gemm_gm=2" "gemm_mc=2" "gemm_mc=2,gemm_gm=32" "gemm_mc=4,gemm_gm=4" "gemm_mc=4" "gemm_mc=4,gemm_gm=32" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg3 8 3 "gemm_mc=2,gemm_gm=2" "gemm_mc=2" "gemm_mc=4" 2>&1 | grep -E "median|rror"
for v in "tcf=0,gemm_mc=2,gemm_gm=2" "tcf=0,gemm_mc=2" "tcf=0,gemm_mc=4"; do STN_DEBUG=$v timeout 300 python scripts/gemm_ab.py 2>&1 | tail -4; done
