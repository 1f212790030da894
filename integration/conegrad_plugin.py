"""pytest plugin: run the reference's OWN test modules against the GPU path.

    PYTHONPATH=baseline/_ref:integration:. python -m pytest -p conegrad_plugin \\
        baseline/_ref/tests/test_solution_map.py baseline/_ref/tests/test_golden.py ...

At start-up (before any test module binds ``jvp``/``vjp`` by name) it
installs ``conegrad_cuda``: every ``conegrad.jvp`` / ``vjp`` /
``check_solution`` call of the suite -- direct, through the CLI, or through
the acceptance criteria -- runs on the B200 through libqcpgrad's C ABI.

The golden files were frozen from the reference's own CPU run with a 1e-9
gap and exact LSMR iteration counts (tests/test_golden.py:18,
tests/helpers.py:46-71).  A GPU path sums in a different order, so -- as
SURVEY §8(c) prescribes -- golden comparisons are relaxed to a 1e-6 relative
gap and +-3 iterations (converged / unreliable flags stay exact).  Nothing
else in the suite is changed.
"""

import numpy as np

import conegrad_cuda

GOLDEN_TOL = 1e-6
ITER_SLACK = 3


def _array_gap(got, want):
    got, want = np.asarray(got, dtype=float), np.asarray(want, dtype=float)
    if got.shape != want.shape:
        raise AssertionError(f"shape {got.shape} != golden {want.shape}")
    gap = float(np.max(np.abs(got - want))) if got.size else 0.0
    return gap / (1.0 + (float(np.max(np.abs(want))) if want.size else 0.0))


def relaxed_golden_result_gap(payload, committed):
    """helpers.golden_result_gap with iteration counts compared to +-3."""
    if set(payload) != set(committed):
        raise AssertionError(f"keys {set(payload)} != golden {set(committed)}")
    worst = 0.0
    for key, want in committed.items():
        got = payload[key]
        if key == "diagnostics":
            for field in ("converged", "derivative_unreliable"):
                if got[field] != want[field]:
                    raise AssertionError(f"diagnostics.{field}: {got[field]!r} != golden {want[field]!r}")
            if abs(got["lsmr_iterations"] - want["lsmr_iterations"]) > ITER_SLACK:
                raise AssertionError(f"diagnostics.lsmr_iterations: {got['lsmr_iterations']} vs golden "
                                     f"{want['lsmr_iterations']} (more than {ITER_SLACK} apart)")
        elif isinstance(want, dict):
            for field in ("shape", "col_ptr", "row_idx"):
                if got[field] != want[field]:
                    raise AssertionError(f"{key}.{field} differs from golden")
            worst = max(worst, _array_gap(got["values"], want["values"]))
        else:
            worst = max(worst, _array_gap(got, want))
    return worst


def pytest_configure(config):
    conegrad_cuda.install()


def pytest_collection_modifyitems(session, config, items):
    seen = set()
    for item in items:
        mod = getattr(item, "module", None)
        if mod is None or mod in seen:
            continue
        seen.add(mod)
        if hasattr(mod, "golden_result_gap"):
            mod.golden_result_gap = relaxed_golden_result_gap
        if mod.__name__.endswith("test_golden") and hasattr(mod, "TOL"):
            mod.TOL = GOLDEN_TOL


def pytest_report_header(config):
    import paper_2508_17522_b200._native as N
    return f"conegrad jvp/vjp/check_solution -> libqcpgrad ({N.LIB_PATH}) via integration/conegrad_cuda.py"
