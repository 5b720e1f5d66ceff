"""Several GPUs of one box through the C ABI (stn_multi_*, runtime.MultiPlan) and
the host-buffer envelope call (stn_run_slices_host).

The multi-device executor must reproduce the reference's run_scheme bit for bit
(EXACT mode, deterministic chained fold: runtime.hpp:601-605) whatever the
number of device plans; with one GPU on the box, several device plans share it
(the sharding and the accumulator hand-over are the same code). With two or
more GPUs the NCCL all-reduce path is checked too."""
import numpy as np
import pytest

from golden_io import bits, plan_path, read_ref

pytestmark = pytest.mark.gpu

CASE = "rt_grid3x4_m8_sliced"  # 32 slices, 64 amplitudes


def _gpus():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.cuda.device_count()


def _desc(name, precision):
    from paper_2005_06787_b200.runtime import load_desc
    return load_desc(plan_path(name, precision))


@pytest.mark.parametrize("precision", ["single", "double"])
@pytest.mark.parametrize("n_plans", [1, 2, 3, 5])
def test_multi_run_scheme_bitwise_reference(precision, n_plans):
    from paper_2005_06787_b200 import MultiPlan
    g = _gpus()
    devices = list(range(n_plans)) if g >= n_plans else [0] * n_plans
    _, _, want, _, _ = read_ref(CASE, precision)
    mp = MultiPlan(_desc(CASE, precision), devices, mode="exact")
    got, rep = mp.run_scheme(deterministic=True)
    assert np.array_equal(bits(got.ravel()), bits(want))
    assert rep.subtasks == mp.subtasks == 32
    # one NCCL all-reduce over distinct GPUs (partials added on one GPU otherwise)
    fast, _ = mp.run_scheme(deterministic=False)
    assert np.abs(fast.ravel() - want).max() <= 1e-12 * np.abs(want).max()
    mp.close()


def test_multi_run_slices_rows_and_digits():
    from paper_2005_06787_b200 import MultiPlan
    from oracle.oracle import OraclePlan
    g = _gpus()
    devices = [0, 1] if g >= 2 else [0, 0]
    asg, vals, _, _, _ = read_ref("cfg1_grid4x5_m14", "single")
    mp = MultiPlan(_desc("cfg1_grid4x5_m14", "single"), devices, mode="exact")
    rows, total = mp.run_slices(0, mp.subtasks, per_slice=True)
    for a, want in zip(asg, vals):
        assert np.array_equal(bits(rows[int(a)].ravel()), bits(want))
    # the same slices addressed by digit vectors (the cfg5 entry point)
    o = OraclePlan(plan_path("cfg1_grid4x5_m14", "single"))
    digits = np.array([o.digits(a) for a in range(mp.subtasks)], np.int32)
    rows2, total2 = mp.run_slices(digits=digits, per_slice=True)
    assert np.array_equal(bits(rows2), bits(rows))
    assert np.array_equal(bits(total2), bits(total))
    mp.close()


def test_run_slices_host_envelope():
    from paper_2005_06787_b200 import ExecutablePlan, build_branch_cache, run_slices_host
    _gpus()
    asg, vals, want_sum, _, _ = read_ref(CASE, "single")
    plan = ExecutablePlan.load(plan_path(CASE, "single"), device=0, mode="exact")
    cache = build_branch_cache(plan)
    rows, total = run_slices_host(plan, cache, 0, plan.subtasks)
    for a, want in zip(asg, vals):
        assert np.array_equal(bits(rows[int(a)].ravel()), bits(want))
    assert np.array_equal(bits(total.ravel()), bits(want_sum))
    # a sub-envelope [5, 12)
    r2, _ = run_slices_host(plan, cache, 5, 7, total=False)
    assert np.array_equal(bits(r2), bits(rows[5:12]))


def test_multi_cfg2_on_distinct_gpus_bitwise():
    """cfg2 (64 slices, every kernel family incl. the tensor-core ones) over the
    distinct GPUs of the box: EXACT chained fold == the reference's run_scheme sum."""
    from paper_2005_06787_b200 import MultiPlan
    g = _gpus()
    if g < 2:
        pytest.skip("needs two GPUs")
    try:
        _, _, want, _, _ = read_ref("cfg2_grid5x6_m16", "single")
    except FileNotFoundError:
        pytest.skip("no reference values")
    if want is None:
        pytest.skip("no reference run_scheme sum recorded")
    mp = MultiPlan(_desc("cfg2_grid5x6_m16", "single"), list(range(min(g, 4))), mode="exact")
    got, _ = mp.run_scheme(deterministic=True)
    assert np.array_equal(bits(got.ravel()), bits(want))
    fast = MultiPlan(_desc("cfg2_grid5x6_m16", "single"), list(range(min(g, 4))), mode="fast")
    f1, _ = fast.run_scheme(deterministic=True)
    f2, _ = fast.run_scheme(deterministic=False)
    assert np.abs(f1.ravel() - want).max() <= 1e-4 * np.abs(want).max()
    assert np.abs(f2.ravel() - f1.ravel()).max() <= 1e-12 * np.abs(f1).max()
