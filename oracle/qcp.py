"""Oracle derivative path: sparse products, embedding operator, LSMR, jvp/vjp.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Restates, operation
for operation, the reference's

* CSC products in storage order      (``_kernels/_csc.pyx:17-50``, ``pyref.py:12-27``)
* embedding maps                     (``embedding.py:198-427``)
* LSMR (Fong-Saunders, damp = 0)     (``lsmr.py:38-184``)
* solution-map pipeline              (``solution_map.py:170-385``)

including the reference's redundant work per operator application (the
recomputed ``P x`` in ``duq_apply``/``duq_adjoint`` and three projection-
derivative applications per LSMR iteration), so that timing it is a fair
stand-in for timing the reference.  Matrices are any objects with
``nrows, ncols, col_ptr, row_idx, values``.
"""

import ctypes
import os
from collections import namedtuple

import numpy as np

from oracle import cones as C

Csc = namedtuple("Csc", "nrows ncols col_ptr row_idx values")
Problem = namedtuple("Problem", "P A q b blocks")
Sol = namedtuple("Sol", "x y s")
Pert = namedtuple("Pert", "dP dA dq db")
Delta = namedtuple("Delta", "dx dy ds")
LsmrOut = namedtuple("LsmrOut", "x itn converged normr normar")
Diag = namedtuple("Diag", "iterations converged residual_norm rhs_norm derivative_unreliable")

# ---------------------------------------------------------------------------
# CSC products.  The C restatement (oracle/csc.c) is used when built; the
# NumPy form below is bit-identical (np.add.at accumulates in index order).
# ---------------------------------------------------------------------------

_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(os.path.dirname(__file__), "_build", "liboracle_csc.so")
        if os.path.exists(path):
            lib = ctypes.CDLL(path)
            dp = ctypes.POINTER(ctypes.c_double)
            ip = ctypes.POINTER(ctypes.c_int64)
            lib.oracle_csc_spmv.argtypes = [ctypes.c_int64, ctypes.c_int64, ip, ip, dp, dp, dp]
            lib.oracle_csc_spmv_adjoint.argtypes = [ctypes.c_int64, ip, ip, dp, dp, dp]
            _LIB = lib
        else:
            _LIB = False
    return _LIB


def _ptr(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def spmv(M, x):
    """A @ x, storage-order scatter (_csc.pyx:17-32)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    lib = _lib()
    out = np.zeros(M.nrows)
    if lib:
        cp = np.ascontiguousarray(M.col_ptr, dtype=np.int64)
        ri = np.ascontiguousarray(M.row_idx, dtype=np.int64)
        va = np.ascontiguousarray(M.values, dtype=np.float64)
        lib.oracle_csc_spmv(M.nrows, M.ncols, _ptr(cp, ctypes.c_int64), _ptr(ri, ctypes.c_int64),
                            _ptr(va, ctypes.c_double), _ptr(x, ctypes.c_double),
                            _ptr(out, ctypes.c_double))
        return out
    cols = np.repeat(np.arange(M.ncols), np.diff(M.col_ptr))
    np.add.at(out, M.row_idx, M.values * x[cols])
    return out


def spmv_t(M, y):
    """A.T @ y, per-column gather in storage order (_csc.pyx:35-50)."""
    y = np.ascontiguousarray(y, dtype=np.float64)
    lib = _lib()
    out = np.zeros(M.ncols)
    if lib:
        cp = np.ascontiguousarray(M.col_ptr, dtype=np.int64)
        ri = np.ascontiguousarray(M.row_idx, dtype=np.int64)
        va = np.ascontiguousarray(M.values, dtype=np.float64)
        lib.oracle_csc_spmv_adjoint(M.ncols, _ptr(cp, ctypes.c_int64), _ptr(ri, ctypes.c_int64),
                                    _ptr(va, ctypes.c_double), _ptr(y, ctypes.c_double),
                                    _ptr(out, ctypes.c_double))
        return out
    cols = np.repeat(np.arange(M.ncols), np.diff(M.col_ptr))
    np.add.at(out, cols, M.values * y[M.row_idx])
    return out


def entry_cols(M):
    return np.repeat(np.arange(M.ncols, dtype=np.int64), np.diff(M.col_ptr))


def to_dense(M):
    D = np.zeros((M.nrows, M.ncols))
    D[M.row_idx, entry_cols(M)] = M.values
    return D


def from_dense(D):
    cols, rows = np.nonzero(D.T)
    cp = np.zeros(D.shape[1] + 1, dtype=np.int64)
    np.cumsum(np.bincount(cols, minlength=D.shape[1]), out=cp[1:])
    return Csc(D.shape[0], D.shape[1], cp, rows.astype(np.int64), D[rows, cols])


# ---------------------------------------------------------------------------
# Embedding (embedding.py)
# ---------------------------------------------------------------------------

def dims(th):
    return th.A.ncols, th.A.nrows


def embedding_project(th, z):                       # embedding.py:337-344
    n, m = dims(th)
    out = np.empty(n + m + 1)
    out[:n] = z[:n]
    out[n:n + m] = C.project(th.blocks, z[n:n + m], dual=True)
    out[-1] = max(z[-1], 0.0)
    return out


def duq_apply(th, u, du):                           # embedding.py:214-238
    n, m = dims(th)
    x, tau = u[:n], u[n + m]
    dx, dy, dt = du[:n], du[n:n + m], du[n + m]
    Px = spmv(th.P, x)
    out = np.empty(n + m + 1)
    out[:n] = spmv(th.P, dx) + spmv_t(th.A, dy) + dt * th.q
    out[n:n + m] = -spmv(th.A, dx) + dt * th.b
    out[-1] = (-(2.0 / tau) * (Px @ dx) - th.q @ dx - th.b @ dy
               + (x @ Px) / (tau * tau) * dt)
    return out


def duq_adjoint(th, u, w):                          # embedding.py:241-262
    n, m = dims(th)
    x, tau = u[:n], u[n + m]
    w1, w2, wN = w[:n], w[n:n + m], w[n + m]
    Px = spmv(th.P, x)
    out = np.empty(n + m + 1)
    out[:n] = spmv(th.P, w1) - spmv_t(th.A, w2) - ((2.0 / tau) * wN) * Px - wN * th.q
    out[n:n + m] = spmv(th.A, w1) - wN * th.b
    out[-1] = th.q @ w1 + th.b @ w2 + (x @ Px) / (tau * tau) * wN
    return out


def dthetaq_apply(th, u, d):                        # embedding.py:265-292
    n, m = dims(th)
    x, y, tau = u[:n], u[n:n + m], u[n + m]
    dPx = spmv(d.dP, x)
    out = np.empty(n + m + 1)
    out[:n] = dPx + spmv_t(d.dA, y) + tau * d.dq
    out[n:n + m] = -spmv(d.dA, x) + tau * d.db
    out[-1] = -(x @ dPx) / tau - d.dq @ x - d.db @ y
    return out


def dthetaq_adjoint(th, u, w):                      # embedding.py:295-334
    n, m = dims(th)
    x, y, tau = u[:n], u[n:n + m], u[n + m]
    w1, w2, wN = w[:n], w[n:n + m], w[n + m]
    r, c = th.P.row_idx, entry_cols(th.P)
    pv = 0.5 * (w1[r] * x[c] + x[r] * w1[c]) - (wN / tau) * (x[r] * x[c])
    r, c = th.A.row_idx, entry_cols(th.A)
    av = y[r] * w1[c] - w2[r] * x[c]
    return Pert(Csc(th.P.nrows, th.P.ncols, th.P.col_ptr, th.P.row_idx, pv),
                Csc(th.A.nrows, th.A.ncols, th.A.col_ptr, th.A.row_idx, av),
                tau * w1 - wN * x, tau * w2 - wN * y)


class EmbeddingDerivative:                          # embedding.py:347-371
    def __init__(self, th, z):
        n, m = dims(th)
        self.n, self.m = n, m
        self.mid = C.Derivative(th.blocks, z[n:n + m], dual=True)
        self.last = 1.0 if z[-1] > 0.0 else 0.0

    def matvec(self, w):
        n, m = self.n, self.m
        out = np.empty(n + m + 1)
        out[:n] = w[:n]
        out[n:n + m] = self.mid.matvec(w[n:n + m])
        out[-1] = self.last * w[-1]
        return out


class Operator:
    def __init__(self, matvec, rmatvec, dim):
        self.matvec, self.rmatvec, self.dim = matvec, rmatvec, dim

    @property
    def T(self):
        return Operator(self.rmatvec, self.matvec, self.dim)


def make_F(th, z):                                  # embedding.py:399-427
    pz = embedding_project(th, z)
    dpi = EmbeddingDerivative(th, z)
    zN = z[-1]

    def mv(w):
        v = dpi.matvec(w)
        return (duq_apply(th, pz, v) - v + w) / zN

    def rmv(w):
        return (dpi.matvec(duq_adjoint(th, pz, w)) - dpi.matvec(w) + w) / zN

    return Operator(mv, rmv, z.shape[0])


def residual(th, z):                                # embedding.py:198-211, 374-388
    n, m = dims(th)
    pz = embedding_project(th, z)
    x, y, tau = pz[:n], pz[n:n + m], pz[-1]
    Px = spmv(th.P, x)
    Q = np.empty(n + m + 1)
    Q[:n] = Px + spmv_t(th.A, y) + tau * th.q
    Q[n:n + m] = -spmv(th.A, x) + tau * th.b
    Q[-1] = -(x @ Px) / tau - th.q @ x - th.b @ y
    return Q - pz + z


# ---------------------------------------------------------------------------
# LSMR (lsmr.py)
# ---------------------------------------------------------------------------

def givens(a, b):                                   # lsmr.py:38-54
    if b == 0:
        return np.sign(a), 0.0, abs(a)
    if a == 0:
        return 0.0, np.sign(b), abs(b)
    if abs(b) > abs(a):
        t = a / b
        s = np.sign(b) / np.sqrt(1 + t * t)
        return s * t, s, b / s
    t = b / a
    c = np.sign(a) / np.sqrt(1 + t * t)
    return c, c * t, a / c


def lsmr(op, rhs, atol=1e-10, btol=1e-10, max_iter=None):   # lsmr.py:57-184
    dim = op.dim
    if max_iter is None:
        max_iter = 20 * dim
    x = np.zeros(dim)
    beta = float(np.linalg.norm(rhs))
    normb = beta
    if beta > 0:
        u = rhs / beta
        v = op.rmatvec(u)
        alpha = float(np.linalg.norm(v))
    else:
        u, v, alpha = rhs.copy(), np.zeros(dim), 0.0
    if alpha > 0:
        v = v / alpha
    if alpha * beta == 0:
        return LsmrOut(x, 0, True, beta, 0.0)
    zetabar, alphabar = alpha * beta, alpha
    rho = rhobar = cbar = 1.0
    sbar = 0.0
    h, hbar = v.copy(), np.zeros(dim)
    betadd, betad, rhodold = beta, 0.0, 1.0
    tautildeold = thetatilde = zeta = d = 0.0
    normA2 = alpha * alpha
    normr, normar = beta, alpha * beta
    itn = 0
    while itn < max_iter:
        itn += 1
        u = op.matvec(v) - alpha * u
        beta = float(np.linalg.norm(u))
        if beta > 0:
            u = u / beta
            v = op.rmatvec(u) - beta * v
            alpha = float(np.linalg.norm(v))
            if alpha > 0:
                v = v / alpha
        if not (np.isfinite(alpha) and np.isfinite(beta)):
            raise FloatingPointError(itn)
        chat, shat, alphahat = givens(alphabar, 0.0)
        rhoold = rho
        c, s, rho = givens(alphahat, beta)
        thetanew = s * alpha
        alphabar = c * alpha
        rhobarold = rhobar
        zetaold = zeta
        thetabar = sbar * rho
        rhotemp = cbar * rho
        cbar, sbar, rhobar = givens(rhotemp, thetanew)
        zeta = cbar * zetabar
        zetabar = -sbar * zetabar
        hbar = h - (thetabar * rho / (rhoold * rhobarold)) * hbar
        x = x + (zeta / (rho * rhobar)) * hbar
        h = v - (thetanew / rho) * h
        betaacute = chat * betadd
        betacheck = -shat * betadd
        betahat = c * betaacute
        betadd = -s * betaacute
        thetatildeold = thetatilde
        ctildeold, stildeold, rhotildeold = givens(rhodold, thetabar)
        thetatilde = stildeold * rhobar
        rhodold = ctildeold * rhobar
        betad = -stildeold * betad + ctildeold * betahat
        tautildeold = (zetaold - thetatildeold * tautildeold) / rhotildeold
        taud = (zeta - thetatilde * tautildeold) / rhodold
        d = d + betacheck * betacheck
        normr = float(np.sqrt(d + (betad - taud) ** 2 + betadd * betadd))
        normA2 = normA2 + beta * beta
        normA = float(np.sqrt(normA2))
        normA2 = normA2 + alpha * alpha
        normar = abs(zetabar)
        normx = float(np.linalg.norm(x))
        if not (np.isfinite(normr) and np.isfinite(normar) and np.isfinite(normx)):
            raise FloatingPointError(itn)
        if normar == 0:
            return LsmrOut(x, itn, True, normr, normar)
        test1 = normr / normb
        test2 = normar / (normA * normr) if normr > 0 else 0.0
        rtol = btol + atol * normA * normx / normb
        t1 = test1 / (1 + normA * normx / normb)
        if 1 + test2 <= 1 or 1 + t1 <= 1 or test2 <= atol or test1 <= rtol:
            return LsmrOut(x, itn, True, normr, normar)
    return LsmrOut(x, itn, False, normr, normar)


# ---------------------------------------------------------------------------
# Solution map (solution_map.py)
# ---------------------------------------------------------------------------

def embed(sol):                                     # solution_map.py:170-179
    return np.concatenate([sol.x, sol.y - sol.s, [1.0]])


def dphi_apply(th, z, dz):                          # solution_map.py:206-231
    n, _ = dims(th)
    mid = z[n:-1]
    proj = C.project(th.blocks, mid, dual=True)
    dmid = C.Derivative(th.blocks, mid, dual=True).matvec(dz[n:-1])
    dzN = dz[-1]
    return Delta(dz[:n] - dzN * z[:n], dmid - dzN * proj, dmid - dz[n:-1] - dzN * (proj - mid))


def dphi_adjoint(th, z, de):                        # solution_map.py:234-260
    n, _ = dims(th)
    mid = z[n:-1]
    proj = C.project(th.blocks, mid, dual=True)
    s = proj - mid
    D = C.Derivative(th.blocks, mid, dual=True)
    out = np.empty(z.shape[0])
    out[:n] = de.dx
    out[n:-1] = D.matvec(de.dy + de.ds) - de.ds
    out[-1] = -(z[:n] @ de.dx) - proj @ de.dy - s @ de.ds
    return out


def _diag(res, rhs_norm):                           # solution_map.py:313-322
    return Diag(res.itn, res.converged, float(res.normr), float(rhs_norm),
                bool(res.normr > 1e-6 * rhs_norm))


def jvp(th, sol, dth, atol=1e-10, btol=1e-10, max_iter=None):   # solution_map.py:325-355
    z = embed(sol)
    u = embedding_project(th, z)
    rhs = -dthetaq_apply(th, u, dth) / abs(z[-1])
    res = lsmr(make_F(th, z), rhs, atol, btol, max_iter)
    return dphi_apply(th, z, res.x), _diag(res, np.linalg.norm(rhs)), res


def vjp(th, sol, de, atol=1e-10, btol=1e-10, max_iter=None):    # solution_map.py:358-385
    z = embed(sol)
    dz = dphi_adjoint(th, z, de)
    res = lsmr(make_F(th, z).T, -dz, atol, btol, max_iter)
    u = embedding_project(th, z)
    g = dthetaq_adjoint(th, u, res.x)
    a = 1.0 / abs(z[-1])
    g = Pert(g.dP._replace(values=a * g.dP.values), g.dA._replace(values=a * g.dA.values),
             a * g.dq, a * g.db)
    return g, _diag(res, np.linalg.norm(dz)), res


def kkt(th, sol, tol=None):                         # solution_map.py:263-288
    x, y, s = sol.x, sol.y, sol.s
    if tol is None:
        nrm = np.sqrt(th.P.values @ th.P.values + th.A.values @ th.A.values
                      + th.q @ th.q + th.b @ th.b)
        tol = 1e-6 * (1.0 + nrm)
    primal = float(np.linalg.norm(spmv(th.A, x) + s - th.b))
    stat = float(np.linalg.norm(spmv(th.P, x) + spmv_t(th.A, y) + th.q))
    gap = float(abs(s @ y))
    sd = float(np.linalg.norm(s - C.project(th.blocks, s)))
    yd = float(np.linalg.norm(y - C.project(th.blocks, y, dual=True)))
    return dict(primal=primal, stationarity=stat, gap=gap, primal_cone_distance=sd,
                dual_cone_distance=yd, tol=float(tol),
                ok=max(primal, stat, gap, sd, yd) <= tol)
