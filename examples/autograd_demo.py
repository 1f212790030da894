"""cvxpylayers-style use of the derivative (run on a GPU box):

    python examples/autograd_demo.py

A batch of QPs with their solutions (here: synthetic KKT-reverse instances,
in practice the output of any conic solver) is wrapped by
``torch_layer.qcp_solution``; a loss on the solutions back-propagates into
(P, A, q, b) through the batched vjp.  The directional derivative of the loss
along a random data direction is then checked three ways: the gradient's
inner product, forward-mode AD (batched jvp), and central differences of
re-solved problems (``testkit.fd_jvp``, GPU Gauss-Newton refine).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.autograd.forward_ad as fwAD  # noqa: E402

import paper_2508_17522_b200 as qg  # noqa: E402
from paper_2508_17522_b200 import synth, testkit  # noqa: E402
from paper_2508_17522_b200.torch_layer import QCPStructure, qcp_solution  # noqa: E402

cones = [("zero", 4, 0, 0.0), ("nonneg", 12, 0, 0.0), ("soc", 5, 0, 0.0), ("exp", 3, 0, 0.0)]
bt = synth.custom(cones, n=16, nnzA=120, seed=7, batch=8)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
struct = QCPStructure(bt.P_colptr, bt.P_rowidx, bt.A_colptr, bt.A_rowidx, bt.n, bt.m, bt.blocks,
                      atol=1e-13, btol=1e-13, max_iter=20000)
P, A, q, b = (dev(getattr(bt, k)).requires_grad_(True) for k in ("P_vals", "A_vals", "q", "b"))
x0, y0, s0 = (dev(getattr(bt, k)) for k in ("x", "y", "s"))

# reverse mode: loss on the solutions -> gradients on the data (batched vjp)
x, y, s = qcp_solution(struct, P, A, q, b, x0, y0, s0)
target = torch.zeros_like(x)
loss = 0.5 * ((x - target) ** 2).sum()
loss.backward()
print(f"loss {loss.item():.6f}  |dL/dq| {q.grad.norm():.4e}  |dL/dA| {A.grad.norm():.4e}")

# one data direction for every problem (dq only, for the finite-difference check)
rng = np.random.default_rng(3)
dq = rng.standard_normal(q.numel())
dq /= np.linalg.norm(dq)
lin = float((q.grad.cpu().numpy() * dq).sum())

# forward mode: the same directional derivative through the batched jvp
with fwAD.dual_level():
    qd = fwAD.make_dual(q.detach(), dev(dq))
    xf, _, _ = qcp_solution(struct, P.detach(), A.detach(), qd, b.detach(), x0, y0, s0)
    dx = fwAD.unpack_dual(xf).tangent
fwd = float((x0 * dx).sum())

# finite differences of re-solved problems, problem by problem (GPU refine)
fd = 0.0
xo, po, ao = np.concatenate([[0], np.cumsum(bt.n)]), np.concatenate([[0], np.cumsum(bt.P_nnz)]), \
    np.concatenate([[0], np.cumsum(bt.A_nnz)])
def objects(i):
    o = synth.problem_objects(bt, i, qg)
    n, m = o["n"], o["m"]
    blocks = [qg.ConeBlock(k, dim=d) if k in ("zero", "nonneg", "soc") else
              qg.ConeBlock(k, order=od) if k == "psd" else
              qg.ConeBlock(k, alpha=a) if k in ("pow", "dpow") else qg.ConeBlock(k) for k, d, od, a in o["blocks"]]
    theta = qg.ProblemData(qg.CscMatrix(n, n, *o["P"]), qg.CscMatrix(m, n, *o["A"]), o["q"], o["b"],
                           qg.ConeSpec(blocks))
    return theta, qg.Solution(o["x"], o["y"], o["s"])


for i in range(bt.B):
    theta, sol = objects(i)
    d_i = dq[xo[i]:xo[i + 1]]
    dtheta = qg.DataPerturbation(theta.P.with_values(np.zeros(theta.P.nnz)),
                                 theta.A.with_values(np.zeros(theta.A.nnz)), d_i, np.zeros(theta.m))
    delta = testkit.fd_jvp(theta, sol, dtheta)
    fd += float((sol.x * delta.dx).sum())

print(f"directional derivative  vjp {lin:+.8e}  jvp {fwd:+.8e}  finite differences {fd:+.8e}")
