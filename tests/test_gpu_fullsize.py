"""Full-size parity (BASELINE.json configs) of the CUDA path against the CPU
oracle, run on the GPU box's host.

P2: at a fixed cap K=20 with atol=btol=0 both sides run
exactly K iterations; on these sizes the reference algorithm's own ulp
sensitivity at K=20 is ~1e-13 (measured), so <= 1e-6 is a real check.
P1: F w / F' w <= 1e-12.  P4 (model-free, tol 1e-14): JVP/VJP duality and
the analytic vary_x path.
"""

import numpy as np
import pytest

from fixtures import gap, synth_instance
from oracle import qcp as Q

pytestmark = pytest.mark.gpu
qg = pytest.importorskip("paper_2508_17522_b200")

C3_SCALED = ([("exp", 3, 0, 0.0)] * 667 + [("pow", 3, 0, 0.5)] * 667, 2000, 100_000)


@pytest.mark.parametrize("cfg", ["c2", "c5a", "c4", "c3s"])
def test_fixed_cap_k20_vs_oracle(cfg):
    ora, prod = synth_instance(C3_SCALED if cfg == "c3s" else cfg, seed=3,
                               **({"diag_P": False} if cfg == "c3s" else {}))
    th, sol, pert, de = ora
    theta, psol, ppert, pde = prod
    q = qg.QCP(theta, psol)
    z = Q.embed(sol)
    F = Q.make_F(th, z)
    rng = np.random.default_rng(0)
    w = rng.standard_normal(z.size)
    assert gap(q.apply_F(w), F.matvec(w)) <= 1e-12
    assert gap(q.apply_F(w, transpose=True), F.rmatvec(w)) <= 1e-12
    dl, dg = q.jvp(ppert, atol=0.0, btol=0.0, max_iter=20)
    ol, og, _ = Q.jvp(th, sol, pert, atol=0.0, btol=0.0, max_iter=20)
    assert dg.iterations == og.iterations == 20
    assert max(gap(dl.dx, ol.dx), gap(dl.dy, ol.dy), gap(dl.ds, ol.ds)) <= 1e-6
    assert abs(dg.residual_norm - og.residual_norm) <= 1e-6 * og.rhs_norm
    g, vg = q.vjp(pde, atol=0.0, btol=0.0, max_iter=20)
    ov, vog, _ = Q.vjp(th, sol, de, atol=0.0, btol=0.0, max_iter=20)
    assert vg.iterations == vog.iterations == 20
    assert max(gap(g.dP.values, ov.dP.values), gap(g.dA.values, ov.dA.values), gap(g.dq, ov.dq),
               gap(g.db, ov.db)) <= 1e-6


@pytest.mark.parametrize("cfg", ["c2", "c5a"])
def test_duality_and_analytic_path(cfg):
    # reference tests/test_solution_map.py:412-431 (duality) and
    # testkit.analytic_path 'vary_x' (testkit.py:356-393)
    _, prod = synth_instance(cfg, seed=5, diag_P=True)
    theta, sol, pert, de = prod
    q = qg.QCP(theta, sol)
    dl, dg = q.jvp(pert, atol=1e-14, btol=1e-14)
    g, vg = q.vjp(de, atol=1e-14, btol=1e-14)
    lhs, rhs = dl.dot(de), g.dot(pert)
    assert abs(lhs - rhs) <= 1e-6 * (1 + abs(lhs))
    rng = np.random.default_rng(9)
    dx = rng.standard_normal(theta.n)
    vary = qg.DataPerturbation(theta.P.with_values(np.zeros(theta.P.nnz)), theta.A.with_values(np.zeros(theta.A.nnz)),
                               -theta.P.matvec(dx), theta.A.matvec(dx))
    dl, dg = q.jvp(vary, atol=1e-14, btol=1e-14)
    assert dg.converged
    assert gap(dl.dx, dx) <= 1e-5 and np.max(np.abs(dl.dy)) <= 1e-5 * (1 + np.max(np.abs(dx)))
