"""CPU-side checks of the C-ABI boundary: the library loads, exports exactly
what include/stn_exec.h declares, plan files round-trip, errors follow the
reference's ErrorKind convention, and nothing silently falls back to the CPU."""
import ctypes as C
import os
import re
import tempfile

import numpy as np
import pytest

from golden_io import plan_path
from paper_2005_06787_b200 import abi

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "stn_exec.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(stn_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = abi.load_library()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in stn_exec.h but not exported"
    # and the ctypes mirror covers all of them with a signature
    assert sorted(abi.SIGNATURES) == names


def test_version_and_status_names():
    lib = abi.load_library()
    assert lib.stn_abi_version() == 1
    assert b"sm_100a" in lib.stn_version()
    # ErrorKind order (errors.hpp:8-30) -> status = index + 1
    for i, kind in enumerate(abi.ERROR_KINDS):
        assert lib.stn_status_name(i + 1).decode() == kind
    assert lib.stn_status_name(0) == b"Ok"


def load_desc(path):
    lib = abi.load_library()
    d = C.POINTER(abi.PlanDesc)()
    abi.check(lib.stn_plan_load(path.encode(), C.byref(d)))
    return d


def test_plan_file_roundtrip_is_byte_identical():
    lib = abi.load_library()
    for name in ("cfg1_grid4x5_m14", "rt_mixed_dims", "rt_hyper_sliced", "cfg5_syc53_m20"):
        src = plan_path(name, "single")
        d = load_desc(src)
        with tempfile.TemporaryDirectory() as t:
            out = os.path.join(t, "p.stnplan")
            abi.check(lib.stn_plan_save(d, out.encode()))
            assert open(out, "rb").read() == open(src, "rb").read()
        lib.stn_plan_desc_free(d)


def test_plan_descriptor_contents():
    d = load_desc(plan_path("cfg1_grid4x5_m14", "single")).contents
    assert d.precision == abi.STN_SINGLE
    assert d.subtasks == 16 and d.n_sliced == 4
    assert d.n_nodes == 2 * d.n_leaves - 1 and d.n_steps == d.n_leaves - 1
    # D*M*N*K bookkeeping of every step (runtime.hpp:330)
    for i in range(d.n_steps):
        s = d.steps[i]
        assert s.mults == s.D * s.M * s.N * s.K
        assert s.lrank == s.nd + s.nm + s.nk and s.rrank == s.nd + s.nk + s.nn


def test_truncated_plan_file_is_a_schema_error():
    lib = abi.load_library()
    src = open(plan_path("rt_mixed_dims", "single"), "rb").read()
    with tempfile.TemporaryDirectory() as t:
        bad = os.path.join(t, "bad.stnplan")
        open(bad, "wb").write(src[: len(src) // 2])
        d = C.POINTER(abi.PlanDesc)()
        st = lib.stn_plan_load(bad.encode(), C.byref(d))
        assert abi.status_name(st) == "SchemaError"
        open(bad, "wb").write(b"NOTAPLAN" + src[8:])
        assert abi.status_name(lib.stn_plan_load(bad.encode(), C.byref(d))) == "SchemaError"
        st = lib.stn_plan_load(os.path.join(t, "missing").encode(), C.byref(d))
        assert abi.status_name(st) == "IOError"


def test_no_silent_cpu_fallback_without_gpu():
    """Without a CUDA device the executor refuses loudly (NoDevice)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2005_06787_b200 import ExecutablePlan, StnError
    with pytest.raises(StnError) as e:
        ExecutablePlan.load(plan_path("cfg1_grid4x5_m14", "single"))
    assert e.value.kind == "NoDevice"


def test_missing_library_fails_loudly(tmp_path):
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        abi.load_library.__wrapped__(str(tmp_path / "nope.so")) if hasattr(
            abi.load_library, "__wrapped__") else _load_missing(tmp_path)


def _load_missing(tmp_path):
    saved = abi._lib
    abi._lib = None
    try:
        abi.load_library(str(tmp_path / "nope.so"))
    finally:
        abi._lib = saved


@pytest.mark.parametrize("exact", [0, 1])
def test_chain_jit_codegen_compiles_for_sm100a(exact):
    """The plan-specialised fused-chain kernels (chain_jit.cpp) are generated CUDA
    compiled by NVRTC at plan creation; the generator's output must build for
    sm_100a in both arithmetic modes (no GPU needed to compile)."""
    import ctypes as C
    from paper_2005_06787_b200 import abi
    lib = abi.load_library()
    buf = C.create_string_buffer(4096)
    st = lib.stn_selftest_chain_jit(exact, buf, 4096)
    assert st == 0, buf.value.decode()[:2000]
