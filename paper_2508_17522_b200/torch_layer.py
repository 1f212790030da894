"""PyTorch autograd binding of the batched derivative.

The cvxpylayers-style consumer of ``vjp``: a solver (any) produces the
primal-dual solution ``(x, y, s)`` of a batch of QCPs; ``qcp_solution``
attaches the solution map's derivative to it, so that a loss on ``x, y, s``
back-propagates into ``(P, A, q, b)`` -- the VJP of arXiv 2508.17522 §5 --
and forward-mode AD (``torch.func.jvp``) pushes data directions through the
JVP.  Everything stays on the device: no host round trip per step.

    struct = QCPStructure(P_colptr, P_rowidx, A_colptr, A_rowidx, n, m, cones)
    x, y, s = qcp_solution(struct, P_vals, A_vals, q, b, x_star, y_star, s_star)
    loss(x).backward()          # P_vals.grad, A_vals.grad, q.grad, b.grad

Tensors are concatenated over the batch exactly as in ``qg_batch_desc``;
P/A values live on the fixed sparsity patterns of the structure (the
reference's masked adjoint, embedding.py:295-334).
"""

import torch

from paper_2508_17522_b200.solution_map import QCPBatch


class QCPStructure:
    """Sparsity patterns, sizes and cones of a batch (fixed across steps)."""

    def __init__(self, P_colptr, P_rowidx, A_colptr, A_rowidx, n, m, cones, P_nnz=None, A_nnz=None,
                 atol=1e-10, btol=1e-10, max_iter=None):
        dev = torch.device("cuda", torch.cuda.current_device())
        self.P_colptr = torch.as_tensor(P_colptr, dtype=torch.int64, device=dev)
        self.P_rowidx = torch.as_tensor(P_rowidx, dtype=torch.int64, device=dev)
        self.A_colptr = torch.as_tensor(A_colptr, dtype=torch.int64, device=dev)
        self.A_rowidx = torch.as_tensor(A_rowidx, dtype=torch.int64, device=dev)
        self.n, self.m = [int(v) for v in n], [int(v) for v in m]
        self.cones = cones
        cp = lambda colptr, ncols: [int(colptr[sum(c + 1 for c in ncols[:i]) + ncols[i]]) for i in range(len(ncols))]
        self.P_nnz = list(P_nnz) if P_nnz is not None else cp(self.P_colptr.cpu().tolist(), self.n)
        self.A_nnz = list(A_nnz) if A_nnz is not None else cp(self.A_colptr.cpu().tolist(), self.n)
        self.opts = dict(atol=atol, btol=btol, max_iter=max_iter)

    def prepare(self, P_vals, A_vals, q, b, x, y, s):
        t = dict(P_colptr=self.P_colptr, P_rowidx=self.P_rowidx, P_vals=P_vals.detach().contiguous(),
                 A_colptr=self.A_colptr, A_rowidx=self.A_rowidx, A_vals=A_vals.detach().contiguous(),
                 q=q.detach().contiguous(), b=b.detach().contiguous(), x=x.detach().contiguous(),
                 y=y.detach().contiguous(), s=s.detach().contiguous())
        batch = QCPBatch.from_device(self.n, self.m, self.P_nnz, self.A_nnz, self.cones, t)
        batch._keep = t
        return batch


class _SolutionMap(torch.autograd.Function):
    @staticmethod
    def forward(struct, P_vals, A_vals, q, b, x, y, s):
        return x.detach().clone(), y.detach().clone(), s.detach().clone()

    @staticmethod
    def setup_context(ctx, inputs, output):
        struct, P_vals, A_vals, q, b, x, y, s = inputs
        ctx.struct = struct
        ctx.batch = struct.prepare(P_vals, A_vals, q, b, x, y, s)

    @staticmethod
    def backward(ctx, gx, gy, gs):
        z = lambda g, ref: torch.zeros_like(ref) if g is None else g.contiguous()
        batch = ctx.batch
        gx, gy, gs = z(gx, batch._keep["x"]), z(gy, batch._keep["y"]), z(gs, batch._keep["s"])
        dP, dA, dq, db, _ = batch.vjp_device(gx, gy, gs, **ctx.struct.opts)
        return None, dP, dA, dq, db, None, None, None

    @staticmethod
    def jvp(ctx, _struct, tP, tA, tq, tb, _tx, _ty, _ts):
        z = lambda t, n: torch.zeros(n, dtype=torch.float64, device="cuda") if t is None else t.contiguous()
        batch = ctx.batch
        dx, dy, ds, _ = batch.jvp_device(z(tP, sum(ctx.struct.P_nnz)), z(tA, sum(ctx.struct.A_nnz)),
                                         z(tq, sum(ctx.struct.n)), z(tb, sum(ctx.struct.m)),
                                         **ctx.struct.opts)
        return dx, dy, ds


def qcp_solution(struct, P_vals, A_vals, q, b, x, y, s):
    """Identity on the solution (x, y, s) that carries the solution map's
    derivative with respect to (P_vals, A_vals, q, b)."""
    return _SolutionMap.apply(struct, P_vals, A_vals, q, b, x, y, s)
