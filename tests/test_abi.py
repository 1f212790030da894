"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every entry point include/qcpgrad.h declares; the Python surface
matches the reference's name set; compute fails loudly without a GPU."""

import ctypes

import numpy as np
import pytest

import paper_2508_17522_b200 as qg
from paper_2508_17522_b200 import _native


def test_library_exports_header_symbols():
    lib = _native.load_library()
    names = _native.header_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert lib.qg_version().decode().startswith("qcpgrad")


def test_library_built_for_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_public_names_match_reference():
    # reference tests/test_package.py:11-25
    expected = {
        "ProblemData", "DataPerturbation", "Solution", "SolutionDelta",
        "ConeBlock", "ConeSpec", "CscMatrix", "Diagnostics", "KktReport",
        "jvp", "vjp", "check_solution", "embed", "phi",
        "project", "project_dual", "dproject", "dproject_dual",
        "dprojection", "dprojection_dual",
        "ConegradError", "ValidationError", "DomainError",
        "NumericalError", "NotDifferentiableError",
    }
    assert expected == set(qg.__all__)
    for name in qg.__all__:
        assert hasattr(qg, name)


def test_struct_layouts_match_header():
    # sizes of the by-value structs the C side reads
    assert ctypes.sizeof(_native.ConeBlockC) == 24
    assert ctypes.sizeof(_native.LsmrOpts) == 24
    assert ctypes.sizeof(_native.DiagC) == 40


def test_host_validation_mirrors_reference():
    with pytest.raises(qg.ValidationError):
        qg.CscMatrix(2, 2, [0, 1, 2], [1, 0, 0], [1.0, 2.0])  # malformed col_ptr end
    with pytest.raises(qg.ValidationError):
        qg.ConeSpec([qg.ConeBlock.soc(3), qg.ConeBlock.nonneg(2)])  # out of order
    with pytest.raises(qg.ValidationError):
        qg.ConeBlock.power(1.5)
    P = qg.CscMatrix.from_dense(np.array([[1.0, 2.0], [0.0, 1.0]]))
    A = qg.CscMatrix.from_dense(np.eye(2))
    with pytest.raises(qg.ValidationError):
        qg.ProblemData(P, A, np.zeros(2), np.zeros(2), qg.ConeSpec([qg.ConeBlock.zero(2)]))


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    spec = qg.ConeSpec([qg.ConeBlock.soc(3)])
    with pytest.raises(qg.DeviceError):
        qg.project(spec, np.array([0.0, 3.0, 4.0]))
