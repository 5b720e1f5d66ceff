"""The reference's own runtime TEST_CASEs (proj/tests/test_runtime.cpp) re-run
with the B200 executor swapped in through include/stemtn_b200/runtime_gpu.hpp:
oracle/_ref/ref_gpu_dropin is compiled against the reference headers in the
build container and executed here on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "oracle", "_ref", "ref_gpu_dropin")


def test_reference_runtime_cases_with_gpu_executor():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/ref_gpu_dropin not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
