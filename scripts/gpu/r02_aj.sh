set -x
for v in "tcf=0,gemm_mc=1" "tcf=0,gemm_mc=2" "tcf=0,gemm_mc=4"; do STN_DEBUG=$v timeout 300 python scripts/gemm_ab.py 2>&1 | tail -4; done
timeout 900 python scripts/ab_compare.py cfg4 8 3 "gemm_mc=1" "" "gemm_mc=4" 2>&1 | grep -E "median|rror"
timeout 900 python scripts/ab_compare.py cfg3 8 2 "gemm_mc=1" "" "gemm_mc=4" 2>&1 | grep -E "median|rror"
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -k "gemm or 53" 2>&1 | tail -2
