import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2508_17522_b200 as qg
from fixtures import synth_instance, gap
from oracle import qcp as Q
cfg = sys.argv[1]; K = int(sys.argv[2])
ora, prod = synth_instance(cfg, seed=3)
th, sol, pert, de = ora
theta, psol, ppert, pde = prod
q = qg.QCP(theta, psol)
g1, _ = q.vjp(pde, atol=0.0, btol=0.0, max_iter=K)
g2, _ = q.vjp(pde, atol=0.0, btol=0.0, max_iter=K)
ov, _, _ = Q.vjp(th, sol, de, atol=0.0, btol=0.0, max_iter=K)
print(os.environ.get("QG_SELL_SIDE"), cfg, K, "repeat-identical", np.array_equal(g1.dA.values, g2.dA.values),
      "gap dA %.1e" % gap(g1.dA.values, ov.dA.values), flush=True)
