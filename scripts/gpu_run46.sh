for tb in 9 10 11 12; do echo "== tb $tb"; STN_PERM_TB=$tb timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -s -k bitperm 2>&1 | grep -E "bitperm (id|rev|swap)"; done
