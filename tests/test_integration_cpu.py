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
