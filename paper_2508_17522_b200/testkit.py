"""Re-solving derivative oracle on the GPU operator.

``refine`` is testkit.refine (reference testkit.py:410-470): Gauss-Newton on
the normalized residual N(z) = R(z)/|z_N| from a warm start, each step the
least-squares model  min ||J d + N(z)||  with the full Jacobian
J = F - N(z) e_N' / z_N  (F of embedding.make_F plus the rank-one
normalization term), then a halving line search on ||N||.  ``fd_jvp`` is
testkit.fd_jvp (testkit.py:473-497): central differences of the refined
solutions at theta +- h dtheta.

Everything that scales with the problem runs in libqcpgrad: the point
preparation (Pi z, D Pi, P x) by ``qg_set_point``, the residual by
``qg_residual`` and the model solve by ``qg_lsmr_jacobian`` (the fused LSMR
kernels with the rank-one term folded into the F / F' steps).  The host
drives the (<= 50 x 30) iteration control exactly as the reference does.
"""

import numpy as np

from paper_2508_17522_b200 import _native as N
from paper_2508_17522_b200.embedding import DataPerturbation, ProblemData
from paper_2508_17522_b200.errors import ConegradError, NumericalError, ValidationError
from paper_2508_17522_b200.solution_map import QCPBatch, Solution, SolutionDelta, embed
from paper_2508_17522_b200.sparse import add_scaled


class _Point:
    """A single-problem handle movable to any embedding point."""

    def __init__(self, theta, z):
        n, m = theta.n, theta.m
        self.n, self.m = n, m
        # created at (x, y - s) = (z_x, z_mid) with z_N = 1, then moved to z
        self.h = QCPBatch([theta], [Solution(z[:n], z[n:n + m], np.zeros(m))])

    def move(self, z_dev, deriv):
        self.h.set_point_device(z_dev, want_deriv=deriv)

    def residual(self):
        return self.h.residual_device()

    def close(self):
        self.h.close()


def _norm(t):
    import torch

    return float(torch.linalg.vector_norm(t))


def refine(theta, z0, tol=1e-10, max_iter=50):
    """Drive the normalized residual to ``tol`` from the warm start ``z0``
    (reference testkit.py:410-470); returns z (NumPy).  NumericalError when
    the line search stagnates or ``max_iter`` steps leave it above ``tol``."""
    import torch

    if not isinstance(theta, ProblemData):
        raise ValidationError("theta must be a ProblemData")
    z = np.ascontiguousarray(z0, dtype=np.float64).copy()
    dim = theta.n + theta.m + 1
    if z.shape != (dim,):
        raise ValidationError(f"z0 must have length {dim}, got {z.shape}")
    if not np.all(np.isfinite(z)):
        raise ValidationError("z0 contains non-finite entries")
    pt = _Point(theta, z)
    try:
        zd = N.to_dev(z, torch.float64)
        pt.move(zd, False)
        res = pt.residual().clone()
        rn = _norm(res)
        for _ in range(max_iter):
            if rn <= tol:
                return zd.cpu().numpy()
            pt.move(zd, True)
            scaled = res / zd[-1]                       # d/dz [R/|z_N|] = F - N e_N'/z_N
            step, _ = pt.h.lsmr_jacobian_device(-res, scaled, atol=1e-12, btol=1e-12)
            step = step.clone()
            size = 1.0
            for _ in range(30):
                trial = zd + size * step
                try:
                    pt.move(trial, False)
                    tres = pt.residual().clone()
                except ConegradError:
                    size *= 0.5
                    continue
                tn = _norm(tres)
                if tn < rn:
                    break
                size *= 0.5
            else:
                raise NumericalError(f"line search stagnated: residual {rn:.3e} not reduced over 30 halvings")
            zd, res, rn = trial, tres, tn
        if rn <= tol:
            return zd.cpu().numpy()
        raise NumericalError(f"residual {rn:.3e} still above tolerance {tol:g} after {max_iter} iterations")
    finally:
        pt.close()


def normalized_residual(theta, z):
    """N(z) on the GPU (embedding.normalized_residual, embedding.py:391-396)."""
    import torch

    z = np.ascontiguousarray(z, dtype=np.float64)
    pt = _Point(theta, z)
    try:
        pt.move(N.to_dev(z, torch.float64), False)
        return pt.residual().cpu().numpy()
    finally:
        pt.close()


def _shifted(theta, dtheta, t):
    return ProblemData(add_scaled(theta.P, dtheta.dP, t), add_scaled(theta.A, dtheta.dA, t),
                       theta.q + t * dtheta.dq, theta.b + t * dtheta.db, theta.cone)


def _decode(theta, z):
    """phi(theta, z) through the GPU projection (solution_map.py:182-194)."""
    import torch

    n, m = theta.n, theta.m
    pt = _Point(theta, z)
    try:
        zd = N.to_dev(z, torch.float64)
        pt.move(zd, False)
        pz = pt.h.embedding_point_device().cpu().numpy()
    finally:
        pt.close()
    zN, mid, proj = z[-1], z[n:n + m], pz[n:n + m]
    return Solution(z[:n] / zN, proj / zN, (proj - mid) / zN)


def fd_jvp(theta, sol, dtheta, h=1e-6, *, tol=1e-11, max_iter=50):
    """Central-difference directional derivative of the solution map
    (reference testkit.py:473-497): refine at theta +- h dtheta from embed(sol)."""
    if not isinstance(theta, ProblemData):
        raise ValidationError("theta must be a ProblemData")
    if not isinstance(sol, Solution):
        raise ValidationError("sol must be a Solution")
    if not isinstance(dtheta, DataPerturbation):
        raise ValidationError("dtheta must be a DataPerturbation")
    if (dtheta.n, dtheta.m) != (theta.n, theta.m):
        raise ValidationError(f"perturbation dimensions ({dtheta.n}, {dtheta.m}) do not match "
                              f"problem dimensions ({theta.n}, {theta.m})")
    h = float(h)
    if not (np.isfinite(h) and h > 0.0):
        raise ValidationError(f"h must be a positive real, got {h}")
    z0 = embed(sol)
    plus, minus = _shifted(theta, dtheta, h), _shifted(theta, dtheta, -h)
    ahead = _decode(plus, refine(plus, z0, tol=tol, max_iter=max_iter))
    behind = _decode(minus, refine(minus, z0, tol=tol, max_iter=max_iter))
    f = 0.5 / h
    return SolutionDelta(f * (ahead.x - behind.x), f * (ahead.y - behind.y), f * (ahead.s - behind.s))
