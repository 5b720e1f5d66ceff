"""A/B of the tcgen05 GEMM variants on the selftest (error vs fp64 and TFLOP/s).
usage: STN_DEBUG=... gemm_ab.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_06787_b200 import abi  # noqa: E402

lib = abi.load_library()
for M, N, K in ((4096, 1024, 1024), (8192, 2048, 4096), (4096, 4096, 8192), (256, 128, 16384)):
    err, ms, msg, mss, serr = (C.c_double() for _ in range(5))
    st = lib.stn_selftest_gemm_tc(M, N, K, 1, 1, 1, 5, C.byref(err), C.byref(ms), C.byref(msg),
                                  C.byref(mss), C.byref(serr))
    fl = 8.0 * M * N * K
    print(f"{os.environ.get('STN_DEBUG','')} {M}x{N}x{K}: status {st} err {err.value:.2e} "
          f"total {fl / ms.value / 1e9:.1f} TFLOP/s gemm {fl / msg.value / 1e9:.1f} TFLOP/s", flush=True)
