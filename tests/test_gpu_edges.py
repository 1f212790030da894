"""Edge cases of the CUDA path against the oracle on the same inputs:
empty cone (m = 0), empty P, perturbations on patterns different from P/A
(the general transpose path), PSD orders 1 and 64 (the build limit), SOC
blocks of dim 1 and > 32 (generic epilogue), heterogeneous batches, and the
error taxonomy (reference errors.py / cones.py:916-922)."""

import numpy as np
import pytest

from fixtures import gap
from oracle import cones as C
from oracle import qcp as Q

pytestmark = pytest.mark.gpu
qg = pytest.importorskip("paper_2508_17522_b200")


def to_oracle(theta, sol, pert=None, delta=None):
    m = lambda M: Q.Csc(M.nrows, M.ncols, M.col_ptr, M.row_idx, M.values)
    blocks = [C.Block(b.kind, b.dim, b.order, b.alpha) for b in theta.cone.blocks]
    th = Q.Problem(m(theta.P), m(theta.A), theta.q, theta.b, blocks)
    so = Q.Sol(sol.x, sol.y, sol.s)
    pe = None if pert is None else Q.Pert(m(pert.dP), m(pert.dA), pert.dq, pert.db)
    de = None if delta is None else Q.Delta(delta.dx, delta.dy, delta.ds)
    return th, so, pe, de


def kkt_instance(rng, cone_blocks, n, density=0.5, diag_p=False):
    """Well-posed KKT-reverse instance (reference tests/helpers.py:169-209 style)."""
    spec = qg.ConeSpec(cone_blocks)
    m = spec.dim
    w = rng.standard_normal(m)
    s = qg.project(spec, w) if m else np.zeros(0)
    y = s - w
    x = rng.standard_normal(n)
    if diag_p:
        P = qg.CscMatrix.from_dense(np.diag(1.0 + np.abs(rng.standard_normal(n))))
    else:
        M = rng.standard_normal((n, n)) / np.sqrt(n)
        P = qg.CscMatrix.from_dense(M.T @ M + 0.5 * np.eye(n))
    Ad = rng.standard_normal((m, n)) / np.sqrt(n)
    Ad[rng.random((m, n)) > density] = 0.0
    A = qg.CscMatrix.from_dense(Ad) if m else qg.CscMatrix.zeros(0, n)
    b = (A.to_dense() @ x if m else np.zeros(0)) + s
    q = -(P.to_dense() @ x + (A.to_dense().T @ y if m else 0.0))
    return qg.ProblemData(P, A, q, b, spec), qg.Solution(x, y, s)


def random_directions(rng, theta, same_pattern=True):
    n, m = theta.n, theta.m
    if same_pattern:
        sym = rng.standard_normal((n, n))
        sym = sym + sym.T
        dP = theta.P.with_values(sym[theta.P.row_idx, theta.P.entry_cols()])
        dA = theta.A.with_values(rng.standard_normal(theta.A.nnz))
    else:  # different sparsity patterns than P and A
        sym = rng.standard_normal((n, n))
        sym[rng.random((n, n)) > 0.3] = 0.0
        sym = sym + sym.T
        dP = qg.CscMatrix.from_dense(sym)
        da = rng.standard_normal((m, n))
        da[rng.random((m, n)) > 0.4] = 0.0
        dA = qg.CscMatrix.from_dense(da) if m else qg.CscMatrix.zeros(0, n)
    pert = qg.DataPerturbation(dP, dA, rng.standard_normal(n), rng.standard_normal(m))
    delta = qg.SolutionDelta(rng.standard_normal(n), rng.standard_normal(m), rng.standard_normal(m))
    return pert, delta


def check_vs_oracle(theta, sol, pert, delta, tol=1e-14, bound=1e-6):
    th, so, pe, de = to_oracle(theta, sol, pert, delta)
    dl, dg = qg.jvp(theta, sol, pert, atol=tol, btol=tol)
    ol, og, _ = Q.jvp(th, so, pe, atol=tol, btol=tol)
    assert max(gap(dl.dx, ol.dx), gap(dl.dy, ol.dy), gap(dl.ds, ol.ds)) <= bound
    assert abs(dg.iterations - og.iterations) <= max(3, og.iterations // 20)
    g, vg = qg.vjp(theta, sol, delta, atol=tol, btol=tol)
    ov, vog, _ = Q.vjp(th, so, de, atol=tol, btol=tol)
    assert max(gap(g.dP.values, ov.dP.values), gap(g.dA.values, ov.dA.values), gap(g.dq, ov.dq),
               gap(g.db, ov.db)) <= bound
    D = g.dP.to_dense()
    assert np.array_equal(D, D.T)


def test_empty_cone():
    rng = np.random.default_rng(1)
    theta, sol = kkt_instance(rng, [], 4)
    pert, delta = random_directions(rng, theta)
    check_vs_oracle(theta, sol, pert, delta)


def test_empty_P():
    rng = np.random.default_rng(2)
    theta, sol = kkt_instance(rng, [qg.ConeBlock.zero(4), qg.ConeBlock.nonneg(6)], 8)
    P0 = qg.CscMatrix.zeros(8, 8)
    x, y = sol.x, sol.y
    q = -(theta.A.to_dense().T @ y)
    theta = qg.ProblemData(P0, theta.A, q, theta.b, theta.cone)
    pert, delta = random_directions(rng, theta)
    check_vs_oracle(theta, sol, pert, delta)


@pytest.mark.parametrize("seed", [3, 4])
def test_perturbation_on_other_patterns(seed):
    rng = np.random.default_rng(seed)
    cone = [qg.ConeBlock.zero(3), qg.ConeBlock.nonneg(5), qg.ConeBlock.soc(4), qg.ConeBlock.psd(3),
            qg.ConeBlock.exp(), qg.ConeBlock.power(0.4)]
    theta, sol = kkt_instance(rng, cone, 30, density=0.6)
    pert, delta = random_directions(rng, theta, same_pattern=False)
    check_vs_oracle(theta, sol, pert, delta)


@pytest.mark.parametrize("order", [1, 2, 7, 64])
def test_psd_orders(order):
    rng = np.random.default_rng(order)
    cone = [qg.ConeBlock.nonneg(3), qg.ConeBlock.psd(order)]
    m = 3 + order * (order + 1) // 2
    theta, sol = kkt_instance(rng, cone, m + 2, density=0.3, diag_p=True)
    th, so, _, _ = to_oracle(theta, sol)
    q = qg.QCP(theta, sol)
    z = Q.embed(so)
    F = Q.make_F(th, z)
    w = rng.standard_normal(z.size)
    assert gap(q.apply_F(w), F.matvec(w)) <= 1e-12
    assert gap(q.apply_F(w, transpose=True), F.rmatvec(w)) <= 1e-12


def test_psd_order_above_limit_is_rejected():
    spec = qg.ConeSpec([qg.ConeBlock.psd(65)])
    with pytest.raises(qg.ConegradError):
        qg.project(spec, np.zeros(spec.dim))


@pytest.mark.parametrize("dim", [1, 2, 40, 200])
def test_soc_dims(dim):
    rng = np.random.default_rng(dim)
    cone = [qg.ConeBlock.soc(dim), qg.ConeBlock.soc(dim)]
    theta, sol = kkt_instance(rng, cone, 2 * dim + 3, density=0.4, diag_p=True)
    th, so, _, _ = to_oracle(theta, sol)
    q = qg.QCP(theta, sol)
    z = Q.embed(so)
    F = Q.make_F(th, z)
    for _ in range(2):
        w = rng.standard_normal(z.size)
        assert gap(q.apply_F(w), F.matvec(w)) <= 1e-12
        assert gap(q.apply_F(w, transpose=True), F.rmatvec(w)) <= 1e-12


def test_heterogeneous_batch_matches_singles():
    rng = np.random.default_rng(11)
    cones = [[qg.ConeBlock.nonneg(7)], [qg.ConeBlock.zero(2), qg.ConeBlock.soc(5)],
             [qg.ConeBlock.psd(3), qg.ConeBlock.dual_exp()], [qg.ConeBlock.dual_power(0.3)], []]
    items = []
    for i, c in enumerate(cones):
        theta, sol = kkt_instance(rng, c, 10 + i, density=0.6)
        pert, delta = random_directions(rng, theta)
        items.append((theta, sol, pert, delta))
    batch = qg.QCPBatch([t for t, _, _, _ in items], [s for _, s, _, _ in items])
    outs = batch.jvp_all([p for _, _, p, _ in items], atol=1e-14, btol=1e-14)
    vouts = batch.vjp_all([d for _, _, _, d in items], atol=1e-14, btol=1e-14)
    for (theta, sol, pert, delta), (dl, dg), (g, vg) in zip(items, outs, vouts):
        th, so, pe, de = to_oracle(theta, sol, pert, delta)
        ol, og, _ = Q.jvp(th, so, pe, atol=1e-14, btol=1e-14)
        assert max(gap(dl.dx, ol.dx), gap(dl.dy, ol.dy)) <= 1e-6
        ov, vog, _ = Q.vjp(th, so, de, atol=1e-14, btol=1e-14)
        assert max(gap(g.dA.values, ov.dA.values), gap(g.dq, ov.dq)) <= 1e-6


def test_not_differentiable_pow_apex_propagates():
    # dual power block at z = (x, y, 0) with y = 0: apex stratum (cones.py:676-678)
    P = qg.CscMatrix.from_dense(np.eye(2))
    A = qg.CscMatrix.from_dense(np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0]]))
    spec = qg.ConeSpec([qg.ConeBlock.dual_power(0.5)])
    y = np.array([0.0, 0.0, 0.0])
    s = np.array([1.0, 0.0, 0.0])     # z = y - s = (-1, 0, 0): x != 0, y = 0, z = 0
    x = np.zeros(2)
    theta = qg.ProblemData(P, A, -(A.to_dense().T @ y), A.to_dense() @ x + s, spec)
    sol = qg.Solution(x, y, s)
    with pytest.raises(qg.NotDifferentiableError) as exc:
        qg.QCP(theta, sol)
    assert "cone block 0 (dpow)" in str(exc.value)


def test_validation_errors():
    rng = np.random.default_rng(5)
    theta, sol = kkt_instance(rng, [qg.ConeBlock.nonneg(3)], 4)
    with pytest.raises(qg.ValidationError):
        qg.jvp(theta, qg.Solution(np.zeros(3), np.zeros(3), np.zeros(3)), None)
    with pytest.raises(qg.ValidationError):
        qg.QCP(theta, sol).jvp("not a perturbation")
