"""Fixed-cap oracle runs with the preparation done once (test helper).

For full-size parity (BASELINE configs at their real sizes) the oracle's
per-call preparation -- Pi_K*(z), D Pi (13,334 exp/pow root solves at C3),
the operator F -- dominates; this helper prepares once and then runs the
reference's fixed-cap LSMR for any number of caps and noise draws, mapping
the solutions through the same formulas as oracle.qcp.jvp / vjp
(reference solution_map.py:206-231, 325-385; embedding.py:295-334).

``noise``: every operator output perturbed by 1e-16 relative noise -- the
reference's own sensitivity at that cap: the GPU path is
compared only where that sensitivity is <= 1e-10.
"""

import numpy as np

from fixtures import gap
from oracle import cones as C
from oracle import qcp as Q


class OracleRuns:
    def __init__(self, th, sol, pert, de):
        self.th = th
        z = self.z = Q.embed(sol)
        n, m = Q.dims(th)
        self.n = n
        self.F = Q.make_F(th, z)
        self.u = Q.embedding_project(th, z)
        mid = z[n:-1]
        self.mid = mid
        self.proj = C.project(th.blocks, mid, dual=True)
        self.D = C.Derivative(th.blocks, mid, dual=True)
        self.rhs = -Q.dthetaq_apply(th, self.u, pert) / abs(z[-1])
        s = self.proj - mid
        dz = np.empty(z.shape[0])
        dz[:n] = de.dx
        dz[n:-1] = self.D.matvec(de.dy + de.ds) - de.ds
        dz[-1] = -(z[:n] @ de.dx) - self.proj @ de.dy - s @ de.ds
        self.dz = dz

    def _op(self, noise):
        if noise is None:
            return self.F
        f, ft = self.F.matvec, self.F.rmatvec
        nz = lambda r: r * (1 + 1e-16 * noise.standard_normal(r.size))
        return Q.Operator(lambda w: nz(f(w)), lambda w: nz(ft(w)), self.z.size)

    def run(self, K, noise=None):
        """(jvp output [dx|dy|ds], vjp output [dP|dA|dq|db]) at cap K."""
        F = self._op(noise)
        n, z = self.n, self.z
        x = Q.lsmr(F, self.rhs, 0.0, 0.0, K).x
        dmid = self.D.matvec(x[n:-1])
        dzN = x[-1]
        j = np.concatenate([x[:n] - dzN * z[:n], dmid - dzN * self.proj,
                            dmid - x[n:-1] - dzN * (self.proj - self.mid)])
        w = Q.lsmr(F.T, -self.dz, 0.0, 0.0, K).x
        g = Q.dthetaq_adjoint(self.th, self.u, w)
        return j, np.concatenate([g.dP.values, g.dA.values, g.dq, g.db])

    def stable_caps(self, caps, limit=1e-10, draws=(1, 2)):
        """{K: (jvp, vjp)} for the caps at which the reference is stable
        under 1e-16 operator noise (sensitivity <= limit)."""
        out = {}
        for K in caps:
            j0, v0 = self.run(K)
            sens = 0.0
            for seed in draws:
                j1, v1 = self.run(K, np.random.default_rng(seed))
                sens = max(sens, gap(j1, j0), gap(v1, v0))
            if sens <= limit:
                out[K] = (j0, v0)
        return out
