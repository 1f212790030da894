"""The deferred finalize of single-problem graph loops (kFeatDF): each step
launch's CTA 0 runs the finalize the previous step owes while the unit CTAs
stage their row sums, so the loop runs 2 launches per LSMR iteration instead
of 4.  Checked against the round-1 loop (QG_DEFER_FIN=0, separate k_fin_cta
launches) and the oracle: same iteration counts and flags, outputs equal to
summation-order level at caps where the reference itself is stable
(DESIGN.md §5), bit-identical repeats, and the launch count it claims.
"""

import numpy as np
import pytest

from fixtures import gap
from oracle import cpu_bench
from oracle_runs import OracleRuns

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2508_17522_b200 import QCPBatch, _native, synth  # noqa: E402

KEYS = ("P_colptr", "P_rowidx", "P_vals", "A_colptr", "A_rowidx", "A_vals", "q", "b", "x", "y", "s")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _batch(bt):
    return QCPBatch.from_device(bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks, {k: _dev(getattr(bt, k)) for k in KEYS})


def _run(b, dirs, **kw):
    j = b.jvp_device(_dev(dirs.dP), _dev(dirs.dA), _dev(dirs.dq), _dev(dirs.db), **kw)
    v = b.vjp_device(_dev(dirs.dx), _dev(dirs.dy), _dev(dirs.ds), **kw)
    return [t.cpu().numpy() for t in j[:3]], [t.cpu().numpy() for t in v[:4]], j[3], v[4]


@pytest.fixture(scope="module")
def c2():
    # c2's cone mix and density at a quarter of its size (SOC(8) blocks) with
    # the fast-converging diagonal P of the parity recipe
    bt = synth.custom([("soc", 8, 0, 0)] * 125, n=500, nnzA=25_000, seed=21, diag_P=True)
    return bt, synth.directions(bt, seed=22)


def test_defer_fin_matches_finalize_kernels(monkeypatch, c2):
    bt, dirs = c2
    monkeypatch.setenv("QG_ENGINE", "0")
    monkeypatch.setenv("QG_TARGET_NNZ", "1024")  # the same work units for both loops
    monkeypatch.setenv("QG_DEFER_FIN", "1")
    b1 = _batch(bt)
    monkeypatch.setenv("QG_DEFER_FIN", "0")
    b0 = _batch(bt)
    # (K = 20 is past this operator's stable caps: 1e-16 noise moves the
    # reference's own iterate by ~1e-6 there; the oracle test
    # below covers the stable caps)
    for K in (2, 5):
        kw = dict(atol=0.0, btol=0.0, max_iter=K)
        r1, r0 = _run(b1, dirs, **kw), _run(b0, dirs, **kw)
        assert [d.iterations for d in r1[2] + r1[3]] == [K, K]
        assert [d.iterations for d in r0[2] + r0[3]] == [K, K]
        for a, c in zip(r1[0] + r1[1], r0[0] + r0[1]):
            assert gap(a, c) <= 1e-9, K
    # converged at the default tolerance: the stopping iteration within the
    # spread summation order alone produces on this ill-conditioned operator
    # (the stopping iterate itself moves ~1e-6 under ulp noise),
    # same convergence flags
    r1, r0 = _run(b1, dirs), _run(b0, dirs)
    for d1, d0 in zip(r1[2] + r1[3], r0[2] + r0[3]):
        assert abs(d1.iterations - d0.iterations) <= max(3, d0.iterations // 50)
        assert d1.converged == d0.converged


def test_defer_fin_vs_oracle_and_repeat(monkeypatch, c2):
    bt, dirs = c2
    monkeypatch.setenv("QG_ENGINE", "0")
    monkeypatch.setenv("QG_DEFER_FIN", "1")
    b = _batch(bt)
    th, sol, pert, de = cpu_bench.problem(bt, dirs, 0)
    runs = OracleRuns(th, sol, pert, de).stable_caps((2, 5, 20))
    assert runs, "no stable cap"
    for K, (j0, v0) in runs.items():
        jv = _run(b, dirs, atol=0.0, btol=0.0, max_iter=K)
        assert gap(np.concatenate(jv[0]), j0) <= 1e-6 and gap(np.concatenate(jv[1]), v0) <= 1e-6, K
    a1 = _run(b, dirs, atol=0.0, btol=0.0, max_iter=20)
    a2 = _run(b, dirs, atol=0.0, btol=0.0, max_iter=20)
    for x, y in zip(a1[0] + a1[1], a2[0] + a2[1]):
        assert np.array_equal(x, y)


def test_defer_fin_launch_count(monkeypatch, c2):
    """2 launches per LSMR iteration (step kernels with the finalize in CTA 0)
    instead of 4 (steps + finalize kernels)."""
    bt, dirs = c2
    monkeypatch.setenv("QG_ENGINE", "0")
    counts = {}
    for f in ("1", "0"):
        monkeypatch.setenv("QG_DEFER_FIN", f)
        b = _batch(bt)
        _run(b, dirs, atol=0.0, btol=0.0, max_iter=4)  # graphs captured, warm
        n0 = _native.kernel_launches()
        _run(b, dirs, atol=0.0, btol=0.0, max_iter=40)
        n1 = _native.kernel_launches()
        _run(b, dirs, atol=0.0, btol=0.0, max_iter=80)
        counts[f] = (_native.kernel_launches() - n1) - (n1 - n0)   # launches of 2 x 40 extra iterations
    assert counts["1"] == 2 * 2 * 40 + 2 * 40 // 4 and counts["0"] == 2 * 4 * 40 + 2 * 40 // 4, counts


@pytest.fixture(scope="module")
def c4s():
    # c4's cone mix at 1/8 of its PSD blocks (nonneg + 64 x PSD(32)), diagonal P
    cones = [("nonneg", 1250, 0, 0)] + [("psd", 528, 32, 0)] * 64
    bt = synth.custom(cones, n=2500, nnzA=250_000, seed=31, diag_P=True)
    return bt, synth.directions(bt, seed=32)


def test_mixed_defer_fin_psd(monkeypatch, c4s):
    """PSD blocks (the F' step split into k_step + k_step_psd): only the F step
    defers -- its CTA 0 runs the F' step's finalize, a k_fin_cta the F step's
    own (3 launches + the PSD branch per iteration).  Against the finalize-
    kernel loop on the same work units at stable caps, the oracle, repeats."""
    bt, dirs = c4s
    monkeypatch.setenv("QG_TARGET_NNZ", "2048")
    monkeypatch.setenv("QG_DEFER_FIN", "1")
    b1 = _batch(bt)
    monkeypatch.setenv("QG_DEFER_FIN", "0")
    b0 = _batch(bt)
    for K in (2, 5):
        kw = dict(atol=0.0, btol=0.0, max_iter=K)
        r1, r0 = _run(b1, dirs, **kw), _run(b0, dirs, **kw)
        assert [d.iterations for d in r1[2] + r1[3]] == [K, K]
        for a, c in zip(r1[0] + r1[1], r0[0] + r0[1]):
            assert gap(a, c) <= 1e-9, K
    th, sol, pert, de = cpu_bench.problem(bt, dirs, 0)
    runs = OracleRuns(th, sol, pert, de).stable_caps((2, 5, 10))
    assert runs, "no stable cap"
    for K, (j0, v0) in runs.items():
        jv = _run(b1, dirs, atol=0.0, btol=0.0, max_iter=K)
        assert gap(np.concatenate(jv[0]), j0) <= 1e-6 and gap(np.concatenate(jv[1]), v0) <= 1e-6, K
    a1 = _run(b1, dirs, atol=0.0, btol=0.0, max_iter=12)
    a2 = _run(b1, dirs, atol=0.0, btol=0.0, max_iter=12)
    for x, y in zip(a1[0] + a1[1], a2[0] + a2[1]):
        assert np.array_equal(x, y)
    # converged runs agree with the finalize-kernel loop on iterations and flags
    c1, c0 = _run(b1, dirs), _run(b0, dirs)
    for d1, d0 in zip(c1[2] + c1[3], c0[2] + c0[3]):
        assert abs(d1.iterations - d0.iterations) <= max(3, d0.iterations // 50)
        assert d1.converged == d0.converged
    # launches: F (+ CTA 0), k_fin_cta, F' main + k_step_psd per iteration
    n0 = _native.kernel_launches()
    _run(b1, dirs, atol=0.0, btol=0.0, max_iter=40)
    n1 = _native.kernel_launches()
    _run(b1, dirs, atol=0.0, btol=0.0, max_iter=80)
    assert (_native.kernel_launches() - n1) - (n1 - n0) == 2 * 4 * 40 + 2 * 40 // 4
