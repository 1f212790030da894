"""Oracle cone calculus (test infrastructure; see ``oracle/__init__.py``).

Restates the reference's projections and projection derivatives for the
eight block kinds (``cones.py`` in the reference; lines cited per routine).
The arithmetic follows the reference operation for operation so that results
agree to rounding; only the code organisation differs.  A block is any object
with ``kind``, ``dim``, ``order`` and ``alpha`` attributes.
"""

import math
from collections import namedtuple

import numpy as np

KINDS = ("zero", "nonneg", "soc", "psd", "exp", "dexp", "pow", "dpow")

Block = namedtuple("Block", "kind dim order alpha")


class ConeFailure(Exception):
    """Raised where the reference raises NumericalError (code 'numerical')
    or NotDifferentiableError (code 'nondiff')."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def block(kind, dim=None, order=None, alpha=None):
    if kind == "psd":
        return Block(kind, order * (order + 1) // 2, order, None)
    if kind in ("exp", "dexp"):
        return Block(kind, 3, None, None)
    if kind in ("pow", "dpow"):
        return Block(kind, 3, None, float(alpha))
    return Block(kind, int(dim), None, None)


def offsets(blocks):
    out = [0]
    for b in blocks:
        out.append(out[-1] + b.dim)
    return out


# --- svec / smat (reference cones.py:176-202) -------------------------------

def _tri(order):
    cols, rows = np.triu_indices(order)
    return rows, cols, np.where(rows == cols, 1.0, math.sqrt(2.0))


def svec(Z):
    rows, cols, sc = _tri(Z.shape[0])
    return Z[rows, cols] * sc


def smat(v, order):
    rows, cols, sc = _tri(order)
    vals = np.asarray(v, dtype=np.float64) / sc
    Z = np.zeros((order, order))
    Z[rows, cols] = vals
    Z[cols, rows] = vals
    return Z


# --- exponential cone (reference cones.py:209-480) ---------------------------

def _exp_member(x, y, z):                          # cones.py:213-219
    if y > 0.0:
        with np.errstate(over="ignore"):
            return y * np.exp(x / y) <= z
    return y == 0.0 and x <= 0.0 and z >= 0.0


def _exp_polar_member(x, y, z):                    # cones.py:222-228
    if x > 0.0:
        with np.errstate(over="ignore"):
            return x * np.exp(y / x) <= -np.e * z
    return x == 0.0 and y <= 0.0 and z <= 0.0


def exp_ratio_eq(p, r):
    """h(rho) and h'(rho) of the ratio equation (cones.py:231-261)."""
    x, y, z = p
    if r <= 0.0:
        e1 = np.exp(r)
        e2 = e1 * e1
        a = 0.0 if e1 == 0.0 else z * e1 * (r * r - r + 1.0)
        ad = 0.0 if e1 == 0.0 else z * e1 * (r * r + r)
        return (x * (-1.0 - (1.0 - r) * e2) + y * (r + e2) - a,
                x * e2 * (2.0 * r - 1.0) + y * (1.0 + 2.0 * e2) - ad)
    e1 = np.exp(-r)
    e2 = e1 * e1
    a = 0.0 if e1 == 0.0 else z * e1 * (r * r - r + 1.0)
    ad = 0.0 if e1 == 0.0 else z * e1 * (r * r - 3.0 * r + 2.0)
    return (x * (r - 1.0 - e2) + y * (1.0 + r * e2) - a,
            x * (1.0 + 2.0 * e2) + y * e2 * (1.0 - 2.0 * r) + ad)


def _exp_candidate(p, r):                          # cones.py:264-294
    x, y, z = p
    if abs(r) > 1e150:
        yh = x / r
        return np.array([x, yh, 0.0]), yh, (-z if r < 0 else 0.0), 0.0
    if r <= 0.0:
        e1 = np.exp(r)
        yh = (r * x + y + z * e1) / (r * r + 1.0 + e1 * e1)
        zh = yh * e1
        mu = (x * e1 + y * (1.0 - r) * e1 - z) / (e1 * e1 * (1.0 + (1.0 - r) ** 2) + 1.0)
        mue = mu * e1
    else:
        e1 = np.exp(-r)
        e2 = e1 * e1
        den = (r * r + 1.0) * e2 + 1.0
        yh = ((r * x + y) * e2 + z * e1) / den
        zh = ((r * x + y) * e1 + z) / den
        dd = 1.0 + (1.0 - r) ** 2 + e2
        mu = ((x + y * (1.0 - r)) * e1 - z * e2) / dd
        mue = ((x + y * (1.0 - r)) - z * e1) / dd
    return np.array([r * yh, yh, zh]), yh, mu, mue


def _exp_worst_residual(p, r, ph, mu, mue):        # cones.py:297-308
    r4 = 0.0 if abs(r) > 700.0 else ph[1] * np.exp(r) - ph[2]
    return max(abs(ph[0] - p[0] + mue), abs(ph[1] - p[1] + mue * (1.0 - r)),
               abs(ph[2] - p[2] - mu), abs(r4))


def _exp_newton(p, lo, hi, flo):                   # cones.py:311-331
    r = 0.5 * (lo + hi)
    for _ in range(200):
        f, fp = exp_ratio_eq(p, r)
        if f == 0.0:
            return r
        if (f > 0.0) == (flo > 0.0):
            lo, flo = r, f
        else:
            hi = r
        nxt = r - f / fp if fp != 0.0 else 0.5 * (lo + hi)
        if not lo < nxt < hi:
            nxt = 0.5 * (lo + hi)
        if abs(nxt - r) <= 1e-14 * (1.0 + abs(r)):
            return nxt
        r = nxt
    return r


def exp_root(p):
    """Expanding 129-point sign scan + polish (cones.py:334-378).

    Returns (rho, phat, yhat, mu) or raises ConeFailure('numerical')."""
    tol = 1e-10 * (1.0 + float(np.linalg.norm(p)))
    x, y, _ = p
    lim = 4.0
    if y != 0.0:
        lim = max(lim, 4.0 * abs(x / y))
    if x != 0.0:
        lim = max(lim, 4.0 * abs(1.0 - y / x))
    lim = min(lim, 1e160)

    def accept(r):
        ph, yh, mu, mue = _exp_candidate(p, r)
        if yh > 0.0 and mu >= -tol and _exp_worst_residual(p, r, ph, mu, mue) <= tol:
            return r, ph, yh, mu
        return None

    span = 1.0
    while True:
        grid = np.linspace(-span, span, 129)
        hv = [exp_ratio_eq(p, g)[0] for g in grid]
        for i in range(128):
            if hv[i] == 0.0:
                got = accept(grid[i])
            elif hv[i] * hv[i + 1] < 0.0:
                got = accept(_exp_newton(p, grid[i], grid[i + 1], hv[i]))
            else:
                continue
            if got is not None:
                return got
        if hv[128] == 0.0:
            got = accept(grid[128])
            if got is not None:
                return got
        if span >= lim:
            raise ConeFailure("numerical", "exponential cone projection root-finding did not converge")
        span = min(2.0 * span, lim)


def _exp_soft(p, tol):                             # cones.py:396-402
    x, y, z = p
    if y > tol:
        with np.errstate(over="ignore"):
            return y * np.exp(x / y) <= z + tol
    return abs(y) <= tol and x <= tol and z >= -tol


def _exp_polar_soft(p, tol):                       # cones.py:405-411
    x, y, z = p
    if x > tol:
        with np.errstate(over="ignore"):
            return x * np.exp(y / x) <= -np.e * z + tol
    return abs(x) <= tol and y <= tol and z <= tol


def proj_exp(p):                                   # cones.py:414-433
    x, y, z = p
    if _exp_member(x, y, z):
        return p.copy()
    if _exp_polar_member(x, y, z):
        return np.zeros(3)
    if x <= 0.0 and y <= 0.0:
        return np.array([x, 0.0, max(z, 0.0)])
    try:
        return exp_root(p)[1]
    except ConeFailure:
        tol = 1e-9 * (1.0 + float(np.linalg.norm(p)))
        if _exp_soft(p, tol):
            return p.copy()
        if _exp_polar_soft(p, tol):
            return np.zeros(3)
        raise


def dproj_exp(p):
    """3x3 derivative of the exp-cone projection (cones.py:436-480)."""
    x, y, z = p
    if y > 0.0:
        with np.errstate(over="ignore"):
            if y * np.exp(x / y) < z:
                return np.eye(3)
    if _exp_polar_member(x, y, z):
        return np.zeros((3, 3))
    if x <= 0.0 and y <= 0.0:
        return np.diag([1.0, 0.0, 1.0 if z > 0.0 else 0.0])
    try:
        r, _, yh, mu = exp_root(p)
    except ConeFailure:
        tol = 1e-9 * (1.0 + float(np.linalg.norm(p)))
        if _exp_soft(p, tol):
            return np.eye(3)
        if _exp_polar_soft(p, tol):
            return np.zeros((3, 3))
        if x <= tol and y <= tol:
            return np.diag([1.0, 0.0, 1.0 if z > 0.0 else 0.0])
        raise
    if abs(r) > 700.0:
        raise ConeFailure("numerical", "exponential cone projection derivative overflows on the boundary ray")
    e = np.exp(r)
    k = mu * e / yh
    J = np.array([[1.0 + k, -r * k, 0.0, e],
                  [-r * k, 1.0 + r * r * k, 0.0, (1.0 - r) * e],
                  [0.0, 0.0, 1.0, -1.0],
                  [e, (1.0 - r) * e, -1.0, 0.0]])
    if not np.all(np.isfinite(J)):
        raise ConeFailure("numerical", "exponential cone derivative system is not finite")
    D = np.linalg.solve(J, np.eye(4)[:, :3])[:3, :]
    return 0.5 * (D + D.T)


# --- power cone (reference cones.py:487-722) ---------------------------------

def _pow_member(p, a):                              # cones.py:490-493
    x, y, z = p
    return x >= 0.0 and y >= 0.0 and x ** a * y ** (1.0 - a) >= abs(z)


def _pow_polar_member(p, a):                        # cones.py:496-501
    x, y, z = p
    if x > 0.0 or y > 0.0:
        return False
    return (-x / a) ** a * (-y / (1.0 - a)) ** (1.0 - a) >= abs(z)


def _pow_coord(w, c, r, az):                        # cones.py:504-514
    qq = 4.0 * c * r * (az - r)
    sq = np.sqrt(w * w + qq)
    return 0.5 * (w + sq) if w >= 0.0 else 0.5 * qq / (sq - w)


def pow_resid(p, a, r, az):                         # cones.py:517-531
    x, y, _ = p
    fx = _pow_coord(x, a, r, az)
    fy = _pow_coord(y, 1.0 - a, r, az)
    prod = fx ** a * fy ** (1.0 - a)
    if fx > 0.0 and fy > 0.0:
        dfx = a * (az - 2.0 * r) / np.sqrt(x * x + 4.0 * a * r * (az - r))
        dfy = (1.0 - a) * (az - 2.0 * r) / np.sqrt(y * y + 4.0 * (1.0 - a) * r * (az - r))
        return prod - r, prod * (a * dfx / fx + (1.0 - a) * dfy / fy) - 1.0
    return prod - r, None


def _pow_bracket(p, a):                             # cones.py:534-556
    x, y, z = p
    az = abs(z)
    fhi = pow_resid(p, a, az, az)[0]
    if fhi >= 0.0:
        return "cone", None
    if x > 0.0 and y > 0.0:
        return "root", (0.0, x ** a * y ** (1.0 - a), az, fhi)
    lo = 0.5 * az
    flo = pow_resid(p, a, lo, az)[0]
    for _ in range(200):
        if flo > 0.0:
            return "root", (lo, flo, az, fhi)
        lo *= 0.5
        flo = pow_resid(p, a, lo, az)[0]
    return "polar", None


def _pow_bisect(p, a, lo, hi, az, limit):
    """Shared bisection loop; returns (lo, hi, exact_root_or_None)."""
    for _ in range(limit):
        mid = 0.5 * (lo + hi)
        if mid <= lo or mid >= hi:
            break
        fm = pow_resid(p, a, mid, az)[0]
        if fm > 0.0:
            lo = mid
        elif fm < 0.0:
            hi = mid
        else:
            return lo, hi, mid
    return lo, hi, None


def pow_root(p, a, lo, flo, hi, fhi):               # cones.py:559-618
    az = abs(p[2])
    tol = 1e-12 * (1.0 + az)
    if flo == 0.0:
        return lo
    while hi - lo > 1e-14 * az:
        mid = 0.5 * (lo + hi)
        if mid <= lo or mid >= hi:
            break
        fm = pow_resid(p, a, mid, az)[0]
        if fm > 0.0:
            lo = mid
        elif fm < 0.0:
            hi = mid
        else:
            return mid
    r = 0.5 * (lo + hi)
    for _ in range(50):
        f, fp = pow_resid(p, a, r, az)
        if abs(f) <= 0.25 * tol:
            break
        if f > 0.0:
            lo = r
        else:
            hi = r
        nxt = r - f / fp if fp not in (None, 0.0) else 0.5 * (lo + hi)
        if not lo < nxt < hi:
            nxt = 0.5 * (lo + hi)
        if abs(nxt - r) <= 1e-17 * (1.0 + r):
            r = nxt
            break
        r = nxt
    f = pow_resid(p, a, r, az)[0]
    if abs(f) <= tol:
        return r
    if f > 0.0:
        lo = r
    else:
        hi = r
    lo, hi, exact = _pow_bisect(p, a, lo, hi, az, 80)
    if exact is not None:
        return exact
    flo = pow_resid(p, a, lo, az)[0]
    fhi = pow_resid(p, a, hi, az)[0]
    return lo if abs(flo) <= abs(fhi) else hi


def proj_pow(p, a):                                 # cones.py:647-663
    if _pow_member(p, a):
        return p.copy()
    if _pow_polar_member(p, a):
        return np.zeros(3)
    x, y, z = p
    if z == 0.0:
        return np.array([max(x, 0.0), max(y, 0.0), 0.0])
    az = abs(z)
    side, br = _pow_bracket(p, a)
    if side == "cone":
        return p.copy()
    if side == "polar":
        return np.zeros(3)
    r = pow_root(p, a, *br)
    return np.array([_pow_coord(x, a, r, az), _pow_coord(y, 1.0 - a, r, az), np.sign(z) * r])


def dproj_pow(p, a):                                # cones.py:666-722
    x, y, z = p
    if z == 0.0 and (x == 0.0 or y == 0.0):
        raise ConeFailure("nondiff", "power cone projection is not differentiable at z = 0 with x = 0 or y = 0")
    if _pow_member(p, a):
        return np.eye(3)
    if _pow_polar_member(p, a):
        return np.zeros((3, 3))
    if z != 0.0:
        az = abs(z)
        side, br = _pow_bracket(p, a)
        if side == "cone":
            return np.eye(3)
        if side == "polar":
            return np.zeros((3, 3))
        r = pow_root(p, a, *br)
        gx = 2.0 * _pow_coord(x, a, r, az) - x
        gy = 2.0 * _pow_coord(y, 1.0 - a, r, az) - y
        ratio = a * x / gx + (1.0 - a) * y / gy
        L = 2.0 * (az - r) / (az + (az - 2.0 * r) * ratio)
        sz = np.sign(z)
        D = np.empty((3, 3))
        D[0, 0] = 0.5 + x / (2.0 * gx) + a ** 2 * (az - 2.0 * r) * r * L / gx ** 2
        D[1, 1] = 0.5 + y / (2.0 * gy) + (1.0 - a) ** 2 * (az - 2.0 * r) * r * L / gy ** 2
        D[0, 1] = D[1, 0] = (a - a ** 2) * (az - 2.0 * r) * r * L / (gx * gy)
        D[0, 2] = D[2, 0] = sz * a * r * L / gx
        D[1, 2] = D[2, 1] = sz * (1.0 - a) * r * L / gy
        D[2, 2] = r / az - r / az * ratio * L
        return D
    if x > 0.0:
        d = 1.0 if a > 0.5 else (0.0 if a < 0.5 else x / (2.0 * abs(y) + x))
    else:
        d = 1.0 if a < 0.5 else (0.0 if a > 0.5 else y / (2.0 * abs(x) + y))
    return np.diag([1.0 if x > 0.0 else 0.0, 1.0 if y > 0.0 else 0.0, d])


# --- second-order and PSD blocks (reference cones.py:730-795) ----------------

def proj_soc(v):                                    # cones.py:730-737
    t, u = v[0], v[1:]
    nu = float(np.linalg.norm(u))
    if nu <= -t:
        return np.zeros_like(v)
    if nu <= t:
        return v.copy()
    return 0.5 * (1.0 + t / nu) * np.concatenate([[nu], u])


def dproj_soc(v):
    """Applier for the SOC derivative (cones.py:740-764)."""
    t, u = v[0], v[1:]
    nu = float(np.linalg.norm(u))
    if nu == 0.0 and t == 0.0:
        return lambda d: 0.5 * d
    if nu < -t:
        return lambda d: np.zeros_like(d)
    if nu < t:
        return lambda d: d.copy()

    def app(d):
        dt, du = d[0], d[1:]
        ud = float(u @ du)
        head = nu * dt + ud
        tail = u * dt + (t + nu) * du - (t / nu ** 2) * ud * u
        return np.concatenate([[head], tail]) / (2.0 * nu)
    return app


def proj_psd(v, order):                             # cones.py:767-769
    lam, V = np.linalg.eigh(smat(v, order))
    return svec((V * np.clip(lam, 0.0, None)) @ V.T)


def psd_weights(lam):
    """Scaling matrix B of the PSD derivative (cones.py:779-789)."""
    tol = 1e-12 * float(np.max(np.abs(lam))) if lam.size else 0.0
    pos = lam >= -tol
    B = np.zeros((lam.size, lam.size))
    B[pos[:, None] & pos[None, :]] = 1.0
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = lam[:, None] / (lam[:, None] - lam[None, :])
    cross = pos[:, None] & ~pos[None, :]
    B[cross] = ratio[cross]
    B[cross.T] = ratio.T[cross.T]
    return B


def dproj_psd(v, order):                            # cones.py:772-795
    lam, V = np.linalg.eigh(smat(v, order))
    B = psd_weights(lam)
    return lambda d: svec(V @ (B * (V.T @ smat(d, order) @ V)) @ V.T)


# --- block dispatch (reference cones.py:803-963) -----------------------------

def _mat(D):
    return lambda d: D @ d


def _cmat(D):
    return lambda d: d - D @ d


def proj_block(b, v, dual=False):
    """Primal (cones.py:803-819) or dual (cones.py:822-834) block projection."""
    k = b.kind
    if dual:
        if k == "zero":
            return v.copy()
        if k == "exp":
            return v + proj_exp(-v)
        if k == "dexp":
            return proj_exp(v)
        if k == "pow":
            return v + proj_pow(-v, b.alpha)
        if k == "dpow":
            return proj_pow(v, b.alpha)
    if k == "zero":
        return np.zeros_like(v)
    if k == "nonneg":
        return np.maximum(v, 0.0)
    if k == "soc":
        return proj_soc(v)
    if k == "psd":
        return proj_psd(v, b.order)
    if k == "exp":
        return proj_exp(v)
    if k == "dexp":
        return v + proj_exp(-v)
    if k == "pow":
        return proj_pow(v, b.alpha)
    return v + proj_pow(-v, b.alpha)


def nonneg_weights(v):                              # cones.py:837-840
    w = np.where(v > 0.0, 1.0, 0.0)
    w[v == 0.0] = 0.5
    return w


def dproj_block(b, v, dual=False):
    """Applier of the block derivative (cones.py:843-883)."""
    k = b.kind
    if dual:
        if k == "zero":
            return lambda d: d.copy()
        if k == "exp":
            return _cmat(dproj_exp(-v))
        if k == "dexp":
            return _mat(dproj_exp(v))
        if k == "pow":
            return _cmat(dproj_pow(-v, b.alpha))
        if k == "dpow":
            return _mat(dproj_pow(v, b.alpha))
    if k == "zero":
        return lambda d: np.zeros_like(d)
    if k == "nonneg":
        w = nonneg_weights(v)
        return lambda d: w * d
    if k == "soc":
        return dproj_soc(v)
    if k == "psd":
        return dproj_psd(v, b.order)
    if k == "exp":
        return _mat(dproj_exp(v))
    if k == "dexp":
        return _cmat(dproj_exp(-v))
    if k == "pow":
        return _mat(dproj_pow(v, b.alpha))
    return _cmat(dproj_pow(-v, b.alpha))


class BlockFailure(Exception):
    """Failure of block ``index`` (mirrors cones.py:916-922 wrapping)."""

    def __init__(self, index, kind, inner):
        super().__init__(f"cone block {index} ({kind}): {inner}")
        self.index, self.kind, self.code = index, kind, inner.code


def _each(blocks, v, fn):
    v = np.ascontiguousarray(v, dtype=np.float64)
    offs = offsets(blocks)
    out = []
    for i, b in enumerate(blocks):
        try:
            out.append((offs[i], offs[i + 1], fn(b, v[offs[i]:offs[i + 1]])))
        except ConeFailure as exc:
            raise BlockFailure(i, b.kind, exc) from exc
    return out


def project(blocks, v, dual=False):
    """Projection onto the product cone or its dual (cones.py:926-941)."""
    out = np.empty(sum(b.dim for b in blocks))
    for a, e, val in _each(blocks, v, lambda b, s: proj_block(b, s, dual)):
        out[a:e] = val
    return out


class Derivative:
    """Prepared blockwise derivative (cones.py:886-906, 944-953)."""

    def __init__(self, blocks, v, dual=False):
        self.dim = sum(b.dim for b in blocks)
        self.parts = _each(blocks, v, lambda b, s: dproj_block(b, s, dual))

    def matvec(self, d):
        d = np.ascontiguousarray(d, dtype=np.float64)
        out = np.empty(self.dim)
        for a, e, app in self.parts:
            out[a:e] = app(d[a:e])
        return out
