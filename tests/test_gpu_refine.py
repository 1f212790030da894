"""GPU re-solving oracle (testkit.py: refine / fd_jvp).

Mirrors the reference's TestRefine / TestFdJvp (reference
tests/test_testkit.py:268-345) on recipe-conditioned synthetic instances:
the residual and the rank-one Jacobian LSMR against the oracle, refine's
convergence / stagnation / budget / domain behaviour, and fd_jvp against
the analytic jvp and the vary_x analytic path (testkit.py:356-393)."""

import numpy as np
import pytest

from fixtures import gap, synth_instance
from oracle import qcp as Q

pytestmark = pytest.mark.gpu
qg = pytest.importorskip("paper_2508_17522_b200")
from paper_2508_17522_b200 import testkit  # noqa: E402

CASES = {
    "nonneg": ([("nonneg", 14, 0, 0.0)], 9, 70),
    "soc": ([("soc", 4, 0, 0.0)] * 3 + [("nonneg", 2, 0, 0.0)], 9, 70),
    "psd": ([("psd", 6, 3, 0.0)] * 2, 8, 60),
    "exp": ([("exp", 3, 0, 0.0)] * 4, 8, 60),
    "dexp": ([("dexp", 3, 0, 0.0)] * 4, 8, 60),
    "pow": ([("pow", 3, 0, 0.4)] * 4, 8, 60),
    "mixed": ([("zero", 3, 0, 0.0), ("nonneg", 5, 0, 0.0), ("soc", 4, 0, 0.0), ("exp", 3, 0, 0.0),
               ("psd", 3, 2, 0.0)], 10, 90),
}


def _case(name, seed=21):
    cones, n, nnz = CASES[name]
    ora, prod = synth_instance((cones, n, nnz), seed=seed)
    return ora, prod


def _noisy(theta, sol, seed=5, scale=1e-4):
    rng = np.random.default_rng(seed)
    return qg.embed(sol) + scale * rng.standard_normal(theta.n + theta.m + 1)


@pytest.mark.parametrize("name", sorted(CASES))
def test_residual_matches_oracle(name):
    (th, osol, _, _), (theta, sol, _, _) = _case(name)
    z = _noisy(theta, sol, scale=1e-2)
    z[-1] = 1.3
    got = testkit.normalized_residual(theta, z)
    want = Q.residual(th, z) / abs(z[-1])
    assert gap(got, want) <= 1e-12
    # zero (to rounding) at the encoding of the exact solution
    assert np.linalg.norm(testkit.normalized_residual(theta, qg.embed(sol))) <= 1e-12


@pytest.mark.parametrize("name", ["soc", "exp", "psd", "mixed"])
def test_rank_one_jacobian_lsmr_matches_oracle(name):
    import torch

    (th, _, _, _), (theta, sol, _, _) = _case(name)
    z = _noisy(theta, sol, scale=1e-3)
    z[-1] = 0.9
    pt = testkit._Point(theta, z)
    try:
        zd = torch.from_numpy(z).cuda()
        pt.move(zd, True)
        r = pt.residual().cpu().numpy()
        scaled = r / z[-1]
        F = Q.make_F(th, z)

        def mv(w):
            return F.matvec(w) - scaled * w[-1]

        def rmv(w):
            out = F.rmatvec(w)
            out[-1] -= scaled @ w
            return out

        J = Q.Operator(mv, rmv, z.size)
        for K in (1, 2, 3):
            want = Q.lsmr(J, -r, 0.0, 0.0, K).x
            got, _ = pt.h.lsmr_jacobian_device(torch.from_numpy(-r).cuda(), torch.from_numpy(scaled).cuda(),
                                               atol=0.0, btol=0.0, max_iter=K)
            assert gap(got.cpu().numpy(), want) <= 1e-12, K
        # and F alone (rank1 = None)
        want = Q.lsmr(F, -r, 0.0, 0.0, 3).x
        got, _ = pt.h.lsmr_jacobian_device(torch.from_numpy(-r).cuda(), None, atol=0.0, btol=0.0, max_iter=3)
        assert gap(got.cpu().numpy(), want) <= 1e-12
    finally:
        pt.close()


def test_exact_point_returned_unchanged():
    _, (theta, sol, _, _) = _case("nonneg")
    z = qg.embed(sol)
    out = testkit.refine(theta, z, tol=1e-8)
    assert out is not z and np.array_equal(out, z)


@pytest.mark.parametrize("name", sorted(CASES))
def test_refine_recovers_from_noise(name):
    (th, _, _, _), (theta, sol, _, _) = _case(name)
    out = testkit.refine(theta, _noisy(theta, sol), tol=1e-10, max_iter=20)
    assert np.linalg.norm(testkit.normalized_residual(theta, out)) <= 1e-10
    assert np.linalg.norm(Q.residual(th, out) / abs(out[-1])) <= 1e-9   # the oracle agrees


def test_infeasible_problem_stagnates():
    theta = qg.ProblemData(qg.CscMatrix.from_dense(np.array([[1.0]])), qg.CscMatrix.from_dense(np.zeros((1, 1))),
                           np.zeros(1), np.array([1.0]), qg.ConeSpec([qg.ConeBlock.zero(1)]))
    with pytest.raises(qg.NumericalError, match="line search stagnated"):
        testkit.refine(theta, np.array([0.0, 0.0, 1.0]), tol=1e-10, max_iter=50)


def test_iteration_budget():
    _, (theta, sol, _, _) = _case("soc")
    with pytest.raises(qg.NumericalError, match="after 2 iterations"):
        testkit.refine(theta, _noisy(theta, sol, seed=2), tol=1e-16, max_iter=2)


def test_rejects_bad_start():
    _, (theta, sol, _, _) = _case("nonneg")
    bad = qg.embed(sol)
    bad[-1] = -1.0
    with pytest.raises(qg.DomainError):
        testkit.refine(theta, bad)
    with pytest.raises(qg.ValidationError, match="length"):
        testkit.refine(theta, np.zeros(3))


def _unit(theta, dtheta):
    s = np.sqrt(np.sum(dtheta.dP.values ** 2) + np.sum(dtheta.dA.values ** 2) + np.sum(dtheta.dq ** 2)
                + np.sum(dtheta.db ** 2))
    return qg.DataPerturbation(dtheta.dP.with_values(dtheta.dP.values / s), dtheta.dA.with_values(dtheta.dA.values / s),
                               dtheta.dq / s, dtheta.db / s)


def _dgap(a, b):
    d = np.concatenate([a.dx - b.dx, a.dy - b.dy, a.ds - b.ds])
    return float(np.linalg.norm(d))


def _dnorm(a):
    return float(np.linalg.norm(np.concatenate([a.dx, a.dy, a.ds])))


@pytest.mark.parametrize("name", sorted(CASES))
def test_fd_jvp_triangulates_jvp(name):
    _, (theta, sol, pert, _) = _case(name, seed=9)
    dtheta = _unit(theta, pert)
    fd = testkit.fd_jvp(theta, sol, dtheta, 1e-6)
    got, diag = qg.jvp(theta, sol, dtheta, atol=1e-13, btol=1e-13, max_iter=30000)
    assert not diag.derivative_unreliable
    assert _dgap(fd, got) <= 2e-4 * (1.0 + _dnorm(got))


def test_fd_jvp_vary_x_analytic_path():
    # dtheta = (0, 0, -P dx, A dx) moves the solution by exactly (dx, 0, 0)
    _, (theta, sol, _, _) = _case("mixed", seed=3)
    dx = np.random.default_rng(9).standard_normal(theta.n)
    dtheta = qg.DataPerturbation(theta.P.with_values(np.zeros(theta.P.nnz)), theta.A.with_values(np.zeros(theta.A.nnz)),
                                 -theta.P.matvec(dx), theta.A.matvec(dx))
    fd = testkit.fd_jvp(theta, sol, dtheta, 1e-6)
    assert np.max(np.abs(fd.dx - dx)) <= 2e-4 * (1 + np.max(np.abs(dx)))
    assert np.max(np.abs(fd.dy)) <= 2e-4 and np.max(np.abs(fd.ds)) <= 2e-4


def test_fd_jvp_zero_direction_and_validation():
    _, (theta, sol, _, _) = _case("nonneg")
    z = qg.DataPerturbation.zeros_like(theta)
    d = testkit.fd_jvp(theta, sol, z, 1e-6)
    assert _dnorm(d) == 0.0
    with pytest.raises(qg.ValidationError, match="positive real"):
        testkit.fd_jvp(theta, sol, z, 0.0)
