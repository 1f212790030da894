"""CPU checks of the reference-side binding (integration/conegrad_cuda.py):
it imports against the unmodified reference, ``install()`` rebinds every
name the reference bound by value, and ``uninstall()`` restores them.  No
compute (the GPU suite is tests/test_gpu_reference_suite.py)."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "conegrad")),
                                reason="reference not installed (baseline/install_ref.sh)")


def test_install_rebinds_reference_entry_points():
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import conegrad
    import conegrad.cli
    import conegrad.solution_map as sm

    import conegrad_cuda as cc

    orig = (sm.jvp, sm.vjp, sm.check_solution)
    cc.install()
    try:
        for mod in (conegrad, sm, conegrad.cli):
            assert mod.jvp is cc.jvp and mod.vjp is cc.vjp
        assert sm.check_solution is cc.check_solution
    finally:
        cc.uninstall()
    assert (sm.jvp, sm.vjp, sm.check_solution) == orig


def test_error_translation_keeps_reference_classes():
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    from conegrad import errors as ref_errors

    import conegrad_cuda as cc
    from paper_2508_17522_b200 import errors as qg_errors

    with pytest.raises(ref_errors.ValidationError, match="bad shape"):
        with cc._reference_errors():
            raise qg_errors.ValidationError("bad shape")
    with pytest.raises(ref_errors.NumericalError) as ei:
        with cc._reference_errors():
            raise qg_errors.NumericalError("broke", iteration=7)
    assert ei.value.iteration == 7


def test_golden_relaxation_is_per_kind_and_measured():
    """The plugin relaxes each golden to the reference's own measured
    spread under ulp noise (tests/golden/golden_noise.json), never below
    1e-6 / +-3 iterations, and maps it onto the suite's 1e-9 threshold."""
    sys.path.insert(0, os.path.join(REF, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import copy

    import conegrad_plugin as cp
    import helpers

    for kind in cp.NOISE:
        for op in ("jvp", "vjp"):
            want = helpers.load_golden(f"{kind}_{op}.json")
            tol, slack, _ = cp.kind_tolerance(want)
            assert tol >= 1e-6 and slack >= 3
            assert tol == max(1e-6, 10 * cp.NOISE[kind][f"{op}_gap"])
            assert cp.relaxed_golden_result_gap(copy.deepcopy(want), want) == 0.0
            got = copy.deepcopy(want)
            key = "dx" if op == "jvp" else "dq"
            got[key] = [v + 2.0 * tol * (1.0 + max(abs(x) for x in want[key])) for v in want[key]]
            assert cp.relaxed_golden_result_gap(got, want) > cp.SUITE_TOL
    assert cp.kind_tolerance(helpers.load_golden("soc_jvp.json"))[0] == 1e-6
    assert cp.kind_tolerance(helpers.load_golden("soc_jvp.json"))[2] is None       # flags exact
    assert cp.kind_tolerance(helpers.load_golden("nonneg_jvp.json"))[0] > 1e-3
    assert cp.kind_tolerance(helpers.load_golden("zero_vjp.json"))[2] == {(True, False), (True, True)}
