"""Kernel-level GPU checks: the tcgen05 split-TF32 complex GEMM against an
fp64 SIMT GEMM on seeded random operands (tolerance 1e-5 of max|C|, the
fp32-level accuracy the split-TF32 scheme is designed to hold)."""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _needs_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("kernel", ["tcf", "presplit"])
@pytest.mark.parametrize("M,N,K,batches,ab,bb", [
    (128, 128, 32, 1, 1, 1),
    (256, 128, 64, 3, 1, 0),
    (128, 256, 96, 2, 0, 1),
    (1024, 512, 1024, 1, 1, 1),
    (4096, 1024, 1024, 1, 1, 1),
    (256, 128, 16384, 1, 1, 1),  # long K: chunked TMEM accumulation keeps fp32 accuracy
    (4096, 32, 8192, 1, 1, 1),   # cfg5's skinny steps (2N = 64: the 128 x 64 fused tile)
    (512, 96, 512, 2, 1, 1),     # 2N = 192: 128 x 64 tiles
    (65536, 8, 512, 1, 1, 1),    # narrow N (cfg4's 2^20 x 8 x 512): zero-padded B'' tile
    (65536, 16, 256, 2, 1, 0),
])
def test_tc_gemm_matches_fp64(M, N, K, batches, ab, bb, kernel, monkeypatch):
    """Both tcgen05 GEMMs: the fused-split one (gemm_tcf.cu, raw fp32 TMA tiles, lo
    formed in shared memory) and the pre-split one (gemm_tc.cu, hi / lo planes)."""
    from paper_2005_06787_b200 import abi
    if kernel == "presplit":
        if (2 * N) % 128:
            pytest.skip("the pre-split kernel needs 2N % 128 == 0")
        monkeypatch.setenv("STN_DEBUG", "tcf=0")
    lib = abi.load_library()
    err, ms, msg, mss, serr = (C.c_double() for _ in range(5))
    abi.check(lib.stn_selftest_gemm_tc(M, N, K, batches, ab, bb, 3, C.byref(err), C.byref(ms),
                                       C.byref(msg), C.byref(mss), C.byref(serr)))
    fl = 8.0 * M * N * K * batches
    print(f"{kernel} gemm {M}x{N}x{K}x{batches}: rel err {err.value:.2e}, "
          f"{ms.value:.3f} ms total ({fl / ms.value / 1e9:.1f} TFLOP/s), {msg.value:.3f} ms gemm "
          f"({fl / msg.value / 1e9:.1f} TFLOP/s); simt fp32 {mss.value:.3f} ms "
          f"({fl / mss.value / 1e9:.1f} TFLOP/s), simt fp32 rel err {serr.value:.2e}")
    # fp32-level: within 1e-5 of max|C| or 4x the plain fp32 GEMM's own error
    assert err.value <= max(1e-5, 4 * serr.value)


@pytest.mark.parametrize("name,perm", [
    ("identity", None),
    ("reverse-low-8", list(range(7, -1, -1)) + list(range(8, 27))),
    ("swap-low-high", list(range(20, 27)) + list(range(7, 20)) + list(range(0, 7))),
])
def test_tiled_bitperm_correct_and_fast(name, perm):
    """The tiled bit-permute (absorb machinery, bulk async copies) on a 2^27
    complex64 tensor (1 GiB): exact result, bandwidth next to cudaMemcpy."""
    from paper_2005_06787_b200 import abi
    lib = abi.load_library()
    arr = (C.c_int32 * 27)(*perm) if perm else None
    gk, gm, ok = C.c_double(), C.c_double(), C.c_int32()
    abi.check(lib.stn_selftest_bitperm(27, arr, 5, C.byref(gk), C.byref(gm), C.byref(ok)))
    print(f"bitperm {name}: kernel {gk.value:.0f} GB/s, cudaMemcpy {gm.value:.0f} GB/s")
    assert ok.value == 1
