"""GPU vs oracle vjp gap at small caps on several configs (diagnostic)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2508_17522_b200 as qg
from fixtures import synth_instance, gap
from oracle import qcp as Q
cfgs = {"c2": "c2", "c5a": "c5a", "psd_small": ([("nonneg", 20, 0, 0.0)] + [("psd", 21, 6, 0.0)] * 10, 300, 5000),
        "soc_small": ([("soc", 6, 0, 0.0)] * 40, 300, 5000), "nn_small": ([("nonneg", 200, 0, 0.0)], 300, 5000)}
for name in sys.argv[1:]:
    ora, prod = synth_instance(cfgs[name], seed=3)
    th, sol, pert, de = ora
    theta, psol, ppert, pde = prod
    q = qg.QCP(theta, psol)
    z = Q.embed(sol); F = Q.make_F(th, z)
    w = np.random.default_rng(1).standard_normal(z.size)
    print(name, "F %.1e FT %.1e" % (gap(q.apply_F(w), F.matvec(w)), gap(q.apply_F(w, True), F.rmatvec(w))))
    for K in (1, 2, 3):
        g, vg = q.vjp(pde, atol=0.0, btol=0.0, max_iter=K)
        ov, vog, _ = Q.vjp(th, sol, de, atol=0.0, btol=0.0, max_iter=K)
        dl, dg = q.jvp(ppert, atol=0.0, btol=0.0, max_iter=K)
        ol, og, _ = Q.jvp(th, sol, pert, atol=0.0, btol=0.0, max_iter=K)
        print(name, K, "vjp dP %.1e dA %.1e dq %.1e db %.1e | jvp dx %.1e dy %.1e ds %.1e" % (
            gap(g.dP.values, ov.dP.values), gap(g.dA.values, ov.dA.values), gap(g.dq, ov.dq), gap(g.db, ov.db),
            gap(dl.dx, ol.dx), gap(dl.dy, ol.dy), gap(dl.ds, ol.ds)), flush=True)
