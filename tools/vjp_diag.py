"""GPU vs oracle vjp/jvp gap as a function of the LSMR cap (diagnostic)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2508_17522_b200 as qg
from fixtures import synth_instance, gap
from oracle import qcp as Q
cfg = sys.argv[1]
ora, prod = synth_instance(cfg, seed=3)
th, sol, pert, de = ora
theta, psol, ppert, pde = prod
q = qg.QCP(theta, psol)
for K in [int(k) for k in sys.argv[2:]]:
    g, vg = q.vjp(pde, atol=0.0, btol=0.0, max_iter=K)
    ov, vog, _ = Q.vjp(th, sol, de, atol=0.0, btol=0.0, max_iter=K)
    dl, dg = q.jvp(ppert, atol=0.0, btol=0.0, max_iter=K)
    ol, og, _ = Q.jvp(th, sol, pert, atol=0.0, btol=0.0, max_iter=K)
    print(cfg, K, "vjp dP %.1e dA %.1e dq %.1e db %.1e | jvp dx %.1e dy %.1e | res %.3e %.3e" % (
        gap(g.dP.values, ov.dP.values), gap(g.dA.values, ov.dA.values), gap(g.dq, ov.dq), gap(g.db, ov.db),
        gap(dl.dx, ol.dx), gap(dl.dy, ol.dy), vg.residual_norm, vog.residual_norm), flush=True)
