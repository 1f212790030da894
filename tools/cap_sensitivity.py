"""GPU-vs-oracle vjp gap and the oracle's own operator-noise sensitivity
(1e-16 relative noise on every F / F' output) across LSMR caps:
    python tools/cap_sensitivity.py c4 5 10 15 19 20"""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2508_17522_b200 as qg
from fixtures import synth_instance, gap
from oracle import qcp as Q
cfg = sys.argv[1]
ora, prod = synth_instance(cfg, seed=3)
th, sol, pert, de = ora
theta, psol, ppert, pde = prod
q = qg.QCP(theta, psol)
z = Q.embed(sol); F = Q.make_F(th, z); u0 = Q.embedding_project(th, z)
dz = Q.dphi_adjoint(th, z, de)
rng = np.random.default_rng(0)
noisy = lambda f: (lambda w: (lambda r: r * (1 + 1e-16 * rng.standard_normal(r.size)))(f(w)))
Fn = Q.Operator(noisy(F.matvec), noisy(F.rmatvec), z.size)
for K in [int(k) for k in sys.argv[2:]]:
    g, _ = q.vjp(pde, atol=0.0, btol=0.0, max_iter=K)
    a = Q.dthetaq_adjoint(th, u0, Q.lsmr(F.T, -dz, 0, 0, K).x).dA.values
    b = Q.dthetaq_adjoint(th, u0, Q.lsmr(Fn.T, -dz, 0, 0, K).x).dA.values
    print(cfg, K, "gpu-vs-oracle %.1e   oracle op-noise %.1e" % (gap(g.dA.values, a), gap(b, a)), flush=True)
