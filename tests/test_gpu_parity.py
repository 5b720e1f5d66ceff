"""GPU parity of the B200 executor against the reference (through the C ABI).

EXACT mode reproduces the reference loop order and rounding, so it must be
bitwise identical to the reference CPU executor's own outputs (tests/golden,
written by the reference via oracle/_ref/ref_tool). FAST mode (tcgen05
split-TF32 GEMMs, FMA SIMT kernels) must agree within the stated tolerance:

    |gpu - ref| <= RTOL * max|ref|,  RTOL = 1e-5      (single precision)

the north star's amplitude tolerance; the reference's own single-precision
path is ~2e-6 from exact at these sizes."""
import numpy as np
import pytest

from golden_io import bits, cases, meta, plan_path, read_ref

pytestmark = pytest.mark.gpu
RTOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _needs_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def load(name, precision, mode):
    from paper_2005_06787_b200 import ExecutablePlan
    return ExecutablePlan.load(plan_path(name, precision), device=0, mode=mode)


def rel_err(got, want):
    scale = max(np.abs(want).max(), 1e-300)
    return float(np.abs(np.asarray(got).ravel() - np.asarray(want).ravel()).max() / scale)


SMALL = [c for c in cases() if not c.startswith(("cfg3", "cfg4", "cfg5"))]


@pytest.mark.parametrize("precision", ["single", "double"])
@pytest.mark.parametrize("name", SMALL)
def test_exact_mode_is_bitwise_reference(name, precision):
    from paper_2005_06787_b200 import build_branch_cache, run_scheme, run_subtask
    try:
        asg, vals, s, bk, info = read_ref(name, precision)
    except FileNotFoundError:
        pytest.skip("no reference values for this case/precision")
    plan = load(name, precision, "exact")
    cache = build_branch_cache(plan)
    assert cache.plan_identity == plan.identity
    assert (cache.mults, cache.elements) == (info["cache"]["mults"], info["cache"]["elements"])
    for a, want in zip(asg, vals):
        r = run_subtask(plan, int(a), cache)
        assert np.array_equal(bits(r.value.ravel()), bits(want)), (name, precision, int(a))
    assert (r.step_count, r.mults, r.peak_elements) == bk
    # without a cache every step runs for the assignment; bitwise the same value
    nc = run_subtask(plan, int(asg[0]), None)
    assert np.array_equal(bits(nc.value.ravel()), bits(vals[0]))
    u = info["uncached"]
    assert (nc.step_count, nc.mults, nc.peak_elements) == (
        u["step_count"], u["mults"], u["peak_elements"])
    if s is not None:
        total, rep = run_scheme(plan, 1)
        assert np.array_equal(bits(total.ravel()), bits(s))
        assert rep.subtasks == plan.subtasks
        assert rep.kernel_launches > 0


E_REF_MAX = 5e-5  # bound on the reference single path's own error before it may widen tol


def truth_and_tolerance(name, a, ref_single):
    """fp64 truth for slice `a` and the amplitude tolerance. The truth is the
    reference's own double-precision value of the slice (tests/golden, written by
    the reference executor); the tolerance is RTOL of max|truth|, or twice the
    reference single-precision path's own error on that slice if larger -- and
    that error must itself be small (<= E_REF_MAX), so a broken fixture cannot
    widen the bound."""
    try:
        asg, dvals, _, _, _ = read_ref(name, "double")
        truth = dvals[list(asg).index(a)]
    except (FileNotFoundError, ValueError):
        pytest.skip(f"no reference double value recorded for {name} slice {a}")
    tol = RTOL
    if ref_single is not None:
        e_ref = rel_err(ref_single, truth)
        assert e_ref <= E_REF_MAX, (name, a, e_ref)
        tol = max(RTOL, 2 * e_ref)
    return truth, tol


@pytest.mark.parametrize("name", SMALL)
def test_fast_mode_within_tolerance(name):
    from paper_2005_06787_b200 import build_branch_cache, run_scheme, run_subtask
    try:
        asg, vals, s, _, _ = read_ref(name, "single")
    except FileNotFoundError:
        pytest.skip("no reference values")
    plan = load(name, "single", "fast")
    cache = build_branch_cache(plan)
    for a, want in zip(asg, vals):
        got = run_subtask(plan, int(a), cache).value
        truth, tol = truth_and_tolerance(name, int(a), want)
        err = rel_err(got, truth)
        print(f"{name} slice {int(a)}: fast err {err:.2e}, reference single err "
              f"{rel_err(want, truth):.2e}, tol {tol:.2e}")
        assert err <= tol, (name, int(a))
    if s is not None:
        total, _ = run_scheme(plan, 1)
        _, _, ds, _, _ = read_ref(name, "double")
        if ds is not None:  # the reference double run_scheme sum, when recorded
            assert rel_err(total, ds) <= max(RTOL, 2 * rel_err(s, ds))
        assert rel_err(total, s) <= 2 * E_REF_MAX  # and the reference single sum


@pytest.mark.parametrize("name", ["rt_grid3x4_m8_sliced", "cfg1_grid4x5_m14"])
def test_fast_single_vs_reference_double(name):
    """Accuracy against the reference's double path (the truth)."""
    from paper_2005_06787_b200 import run_scheme
    _, dv, ds, _, _ = read_ref(name, "double")
    _, sv, ss, _, _ = read_ref(name, "single")
    total, _ = run_scheme(load(name, "single", "fast"), 1)
    ref_single_err = rel_err(ss, ds)
    assert rel_err(total, ds) <= max(RTOL, 2 * ref_single_err)


def test_results_bit_stable_across_parallelism_and_batching():
    """runtime.hpp:552-554 / test_runtime.cpp:258-277: same bits for any
    parallelism; here also for any slice batch size."""
    from paper_2005_06787_b200 import run_scheme
    plan = load("rt_grid3x4_m8_sliced", "single", "fast")
    v1, r1 = run_scheme(plan, 1)
    v8, r8 = run_scheme(plan, 8)
    assert np.array_equal(bits(v1.ravel()), bits(v8.ravel()))
    assert r1.deterministic_json() == r8.deterministic_json()
    for nb in (1, 3, 32):
        plan.set_max_batch(nb)
        vb, _ = run_scheme(plan, 1)
        assert np.array_equal(bits(vb.ravel()), bits(v1.ravel())), nb


@pytest.mark.parametrize("graphs", ["1", "0"])
def test_streams_and_graphs_keep_the_bits(graphs, monkeypatch):
    """Batches rotating over several streams (own arenas; roots folded in ascending
    slice order through an event chain) and CUDA-graph replays of full batches give
    the same bits as one stream launching kernel by kernel -- and the reference's."""
    import torch
    from paper_2005_06787_b200 import build_branch_cache, run_slices
    monkeypatch.setenv("STN_DEBUG", f"graphs={graphs}")
    name = "rt_grid3x4_m8_sliced"
    _, _, want, _, _ = read_ref(name, "single")
    plan = load(name, "single", "exact")
    cache = build_branch_cache(plan)
    n, oe = plan.subtasks, plan.out_elements
    for nb in (1, 3):
        plan.set_max_batch(nb)
        for streams in (1, 2, 3):
            plan.set_streams(streams)
            for _ in range(2):  # second pass replays the captured graphs
                acc = torch.zeros(2 * oe, dtype=torch.float64, device="cuda")
                per = torch.zeros((n, 2 * oe), dtype=torch.float64, device="cuda")
                run_slices(plan, cache, 0, n, acc=acc, per_slice=per)
                torch.cuda.synchronize()
                got = acc.cpu().numpy()
                assert np.array_equal(got.view(np.uint64), want.view(np.float64).view(np.uint64)), (
                    nb, streams)
                rows = per.cpu().numpy().view(np.complex128)
                assert np.array_equal(bits(rows.sum(axis=0) * 0 + rows[0]), bits(rows[0]))


def test_run_slices_device_accumulation_matches_scheme():
    import torch
    from paper_2005_06787_b200 import build_branch_cache, run_scheme, run_slices, sum_slices_ordered
    plan = load("rt_grid3x4_m8_sliced", "single", "fast")
    cache = build_branch_cache(plan)
    n, oe = plan.subtasks, plan.out_elements
    acc = torch.zeros(2 * oe, dtype=torch.float64, device="cuda")
    per = torch.zeros((n, 2 * oe), dtype=torch.float64, device="cuda")
    run_slices(plan, cache, 0, n // 2, acc=acc, per_slice=per[: n // 2])
    run_slices(plan, cache, n // 2, n, acc=acc, per_slice=per[n // 2:])
    out = torch.zeros(2 * oe, dtype=torch.float64, device="cuda")
    sum_slices_ordered(per, n, oe, out)
    torch.cuda.synchronize()
    total, _ = run_scheme(plan, 1)
    want = total.ravel().view(np.float64)
    assert np.array_equal(acc.cpu().numpy().view(np.uint64), want.view(np.uint64))
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want.view(np.uint64))


def test_digit_vector_entry_point_matches_assignment():
    from paper_2005_06787_b200 import build_branch_cache, run_subtask, run_subtask_digits
    from oracle.oracle import OraclePlan
    plan = load("cfg1_grid4x5_m14", "single", "exact")
    ref = OraclePlan(plan_path("cfg1_grid4x5_m14", "single"))
    cache = build_branch_cache(plan)
    for a in (0, 5, 15):
        r1 = run_subtask(plan, a, cache)
        r2 = run_subtask_digits(plan, ref.digits(a), cache)
        assert np.array_equal(bits(r1.value.ravel()), bits(r2.value.ravel()))


def test_errors_mirror_the_reference():
    from paper_2005_06787_b200 import StnError, build_branch_cache, run_subtask
    plan = load("rt_cache_sliced", "single", "fast")
    other = load("rt_hyper_sliced", "single", "fast")
    cache = build_branch_cache(plan)
    with pytest.raises(StnError) as e:  # runtime.hpp:504
        run_subtask(plan, plan.subtasks, cache)
    assert e.value.kind == "SubtaskFailure"
    with pytest.raises(StnError) as e:  # runtime.hpp:505-507
        run_subtask(plan, 0, build_branch_cache(other))
    assert e.value.kind == "SubtaskFailure"


def test_leaf_update_invalidates_cache_and_changes_values():
    """The sampler pokes projector tensors between batches (sampler.hpp:206-213)."""
    from paper_2005_06787_b200 import StnError, build_branch_cache, run_subtask
    from oracle.oracle import OraclePlan
    name = "rt_grid3x4_m8_sliced"
    plan = load(name, "single", "exact")
    cache = build_branch_cache(plan)
    ref = OraclePlan(plan_path(name, "single"))
    d = ref.desc.contents
    branch_inputs = set()
    for i in range(d.n_steps):
        st = d.steps[i]
        if st.is_branch:
            branch_inputs.update((st.lhs, st.rhs))
    # flip the output projectors (rank-1 [1,0] leaves after the 12 input kets)
    flipped, stale = 0, False
    for i in range(d.n_leaves):
        L = d.leaves[i]
        if L.rank == 1 and L.n_sliced == 0 and L.vertex >= 12 and L.values[0] == 1.0:
            plan.set_leaf_values(L.vertex, np.array([0, 1], np.complex128))
            L.values[0], L.values[2] = 0.0, 1.0
            flipped += 1
            stale |= L.node in branch_inputs
    assert flipped > 0
    if stale:
        with pytest.raises(StnError) as e:
            run_subtask(plan, 0, cache)
        assert e.value.kind == "SubtaskFailure"
    fresh = build_branch_cache(plan)
    got = run_subtask(plan, 0, fresh).value.ravel()
    want, _ = ref.run_subtask(0, ref.build_cache())
    assert np.array_equal(bits(got), bits(want))


BIG = ["cfg3_syc53_m12", "cfg4_syc53_m14"]


@pytest.mark.parametrize("name", BIG)
def test_53_qubit_exact_is_bitwise_reference(name):
    """53-qubit slices against the reference executor's own outputs (recorded by
    oracle/_ref/ref_tool, 15-70 CPU-minutes per slice): EXACT mode bit for bit,
    with the SubtaskResult bookkeeping and the branch-cache counts."""
    from paper_2005_06787_b200 import build_branch_cache, run_subtask
    try:
        asg, vals, _, bk, info = read_ref(name, "single")
    except FileNotFoundError:
        pytest.skip("no reference values recorded")
    plan = load(name, "single", "exact")
    cache = build_branch_cache(plan)
    assert (cache.mults, cache.elements) == (info["cache"]["mults"], info["cache"]["elements"])
    for a, want in zip(asg, vals):
        r = run_subtask(plan, int(a), cache)
        assert np.array_equal(bits(r.value.ravel()), bits(want)), (name, int(a))
        assert (r.step_count, r.mults, r.peak_elements) == bk


@pytest.mark.parametrize("name", BIG)
def test_53_qubit_fast_vs_reference_double(name):
    """FAST mode (tcgen05 split-TF32 GEMMs, FMA kernels) against the reference's
    double-precision value of the same slice, within max(RTOL, 2 e_ref)."""
    from paper_2005_06787_b200 import build_branch_cache, run_subtask
    try:
        asg, vals, _, _, _ = read_ref(name, "single")
    except FileNotFoundError:
        pytest.skip("no reference values recorded")
    try:
        dasg = set(int(x) for x in read_ref(name, "double")[0])
    except FileNotFoundError:
        pytest.skip("no reference double values recorded")
    plan = load(name, "single", "fast")
    cache = build_branch_cache(plan)
    checked = 0
    for a, want in zip(asg, vals):
        if int(a) not in dasg:  # slices recorded in single precision only
            continue
        truth, tol = truth_and_tolerance(name, int(a), want)
        err = rel_err(run_subtask(plan, int(a), cache).value, truth)
        print(f"{name} slice {int(a)}: fast err {err:.2e}, reference single err "
              f"{rel_err(want, truth):.2e}, tol {tol:.2e}")
        assert err <= tol, (name, int(a), err, tol)
        checked += 1
    assert checked > 0


@pytest.mark.parametrize("name", ["cfg1_grid4x5_m14", "cfg2_grid5x6_m16"])
def test_stem_sweeps_are_bitwise_the_unfused_steps(name, monkeypatch):
    """Fused stem sweeps (STN_SWEEP_BITS) keep every output's operation order:
    EXACT mode stays bitwise equal to the reference, FAST mode within tolerance."""
    from paper_2005_06787_b200 import build_branch_cache, run_subtask
    monkeypatch.setenv("STN_DEBUG", "sweep_bits=12")
    asg, vals, _, _, _ = read_ref(name, "single")
    plan = load(name, "single", "exact")
    assert plan.kernel_mix()["sweeps"] > 0
    cache = build_branch_cache(plan)
    for a, want in list(zip(asg, vals))[:2]:
        r = run_subtask(plan, int(a), cache)
        assert np.array_equal(bits(r.value.ravel()), bits(want)), (name, int(a))
    fast = load(name, "single", "fast")
    cache = build_branch_cache(fast)
    a, want = int(asg[0]), vals[0]
    truth, tol = truth_and_tolerance(name, a, want)
    assert rel_err(run_subtask(fast, a, cache).value, truth) <= tol


@pytest.mark.parametrize("name", ["cfg1_grid4x5_m14", "cfg2_grid5x6_m16"])
@pytest.mark.parametrize("opts", ["chain_min_bits=0,chain_single=1",
                                  "chain_min_bits=0,chain_single=1,chain_pf_log=3",
                                  "chain_min_bits=0,chain_jit=0"])
def test_fused_chains_everywhere_are_bitwise_the_reference(name, opts, monkeypatch):
    """Fused stem chains on every run of stem absorbs that fits, including one-stage
    chains (the specialised kernel in place of a single absorb, up to 64-value tiles),
    without software pipelining, and on the table-driven kernel (chain_jit=0): EXACT
    mode stays bitwise the reference's values, FAST mode within tolerance."""
    from paper_2005_06787_b200 import build_branch_cache, run_subtask
    monkeypatch.setenv("STN_DEBUG", opts)
    asg, vals, _, _, _ = read_ref(name, "single")
    plan = load(name, "single", "exact")
    # the table-driven kernel's stage limits (K, N <= 8, K x N <= 16) fit no cfg1 run
    assert plan.kernel_mix()["sweeps"] > 0 or (opts.endswith("chain_jit=0") and "cfg1" in name)
    cache = build_branch_cache(plan)
    for a, want in list(zip(asg, vals))[:2]:
        r = run_subtask(plan, int(a), cache)
        assert np.array_equal(bits(r.value.ravel()), bits(want)), (name, opts, int(a))
    fast = load(name, "single", "fast")
    cache = build_branch_cache(fast)
    a, want = int(asg[0]), vals[0]
    truth, tol = truth_and_tolerance(name, a, want)
    assert rel_err(run_subtask(fast, a, cache).value, truth) <= tol


def test_tensor_core_absorbs_run_and_meet_tolerance():
    """cfg2's K=N=64 and K=64,N=16 stem absorbs run on the tcgen05 direct
    absorb (absorb_mma.cu) in FAST mode; the slice stays within tolerance."""
    from paper_2005_06787_b200 import build_branch_cache, run_subtask
    name = "cfg2_grid5x6_m16"
    asg, vals, _, _, _ = read_ref(name, "single")
    plan = load(name, "single", "fast")
    plan.set_profiling(True)
    cache = build_branch_cache(plan)
    plan.reset_profile()
    got = run_subtask(plan, int(asg[0]), cache).value
    rows = plan.get_step_profile()
    tc = [r for r in rows if r["kernel"] == "absorb_tc" and r["K"] == 64]
    assert len(tc) >= 2, rows
    truth, tol = truth_and_tolerance(name, int(asg[0]), vals[0])
    assert rel_err(got, truth) <= tol


@pytest.mark.parametrize("loader", ["tma", "gather"])
def test_tma_gather_absorb_every_eligible_step(loader, monkeypatch):
    """Forces the gather/TMA-fed tcgen05 absorb (absorb_tma.cu) onto every cfg2 stem step
    it can take (K x N >= 64), with either loader; the slice stays within tolerance of
    the fp64 truth and the kernel really ran (absorb_tc-class steps with K <= 32)."""
    from paper_2005_06787_b200 import build_branch_cache, run_subtask
    monkeypatch.setenv("STN_DEBUG", f"tma_min_bits=6,absorb_loader={loader},lanes=0")
    name = "cfg2_grid5x6_m16"
    asg, vals, _, _, _ = read_ref(name, "single")
    plan = load(name, "single", "fast")
    plan.set_profiling(True)
    cache = build_branch_cache(plan)
    plan.reset_profile()
    got = run_subtask(plan, int(asg[0]), cache).value
    rows = plan.get_step_profile()
    tc = [r for r in rows if r["kernel"] == "absorb_tc"]
    assert len(tc) >= 10, rows
    truth, tol = truth_and_tolerance(name, int(asg[0]), vals[0])
    assert rel_err(got, truth) <= tol


def _read_port(name):
    """tests/golden/<name>/port_single.bin: same layout as ref_*.bin."""
    import os
    import struct
    from golden_io import GOLDEN
    b = open(os.path.join(GOLDEN, name, "port_single.bin"), "rb").read()
    n, oe = struct.unpack_from("<QQ", b, 0)
    asg = [int(x) for x in np.frombuffer(b, np.uint64, n, 16)]  # up to 2^64 - 1
    vals = np.frombuffer(b, np.complex128, n * oe, 16 + 8 * n).reshape(n, oe)
    return asg, vals


def _expected_bookkeeping(name):
    """SubtaskResult fields of a cached run, from the plan itself as Engine::run
    counts them (runtime.hpp:440-446): per-slice steps, their mults, largest output."""
    from paper_2005_06787_b200.runtime import load_desc
    d = load_desc(plan_path(name, "single")).contents
    steps = mults = peak = 0
    for i in range(d.n_steps):
        s = d.steps[i]
        if s.is_branch:
            continue
        n = 1
        for k in range(s.orank):
            n *= s.out_dims[k]
        steps, mults, peak = steps + 1, mults + s.mults, max(peak, n)
    return steps, mults, peak


CFG5_FAST_TOL = 5e-5  # FAST vs the reference SINGLE path: both are ~2e-5 from exact (cfg1-4)


def test_cfg5_2pow33_stems_against_the_oracle_port():
    """BASELINE configs[4]: 85 sliced edges (digit-vector slices; the reference's
    uint64 subtasks() overflows, scheme.hpp:33-37), 2^33-element stems. The
    reference executor cannot hold this plan on any host here (Engine::gemm keeps
    4 stem tensors = 256 GiB), so the values come from the oracle port
    (oracle/stn_oracle.c gemm_lean: the reference's arithmetic, bitwise equal to
    the reference on every recorded case) run on a GPU box host
    (scripts/cfg5_parity.py). EXACT must match bit for bit; FAST within
    CFG5_FAST_TOL of max|amp| (no fp64 truth fits: a double stem is 128 GiB)."""
    import torch
    from paper_2005_06787_b200 import build_branch_cache, flush_block_cache, run_subtask_digits
    from oracle.oracle import OraclePlan
    name = "cfg5_syc53_m20"
    asg, vals = _read_port(name)
    ref = OraclePlan(plan_path(name, "single"))
    want_bk = _expected_bookkeeping(name)
    for mode in ("exact", "fast"):
        plan = load(name, "single", mode)
        cache = build_branch_cache(plan)
        for a, want in zip(asg, vals):
            digits = ref.digits(int(a))
            r = run_subtask_digits(plan, digits, cache)
            assert (r.step_count, r.mults, r.peak_elements) == want_bk
            if mode == "exact":
                assert np.array_equal(bits(r.value.ravel()), bits(want)), int(a)
            else:
                err = rel_err(r.value, want)
                print(f"cfg5 slice {int(a)}: fast vs reference-single arithmetic {err:.2e}")
                assert err <= CFG5_FAST_TOL, (int(a), err)
        cache.close()
        plan.close()
        flush_block_cache()
        torch.cuda.empty_cache()
