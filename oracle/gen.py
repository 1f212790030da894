"""Oracle instance generator -- TEST INFRASTRUCTURE ONLY.

Restates the reference's bit-reproducible generator (``testkit.py:95-343``):
SplitMix64 stream, Bernoulli-pattern Gaussian CSC matrices, the exact-sum
Gram ridge ``P = M'M + eps I``, and the KKT-reverse construction with the
margin test.  Used to rebuild configuration C1-ref (n=100, m=150,
zero(30)+nonneg(120), density 0.1) and the golden instances inside tests.
"""

import math

import numpy as np

from oracle import cones as C
from oracle import qcp as Q

_M64 = (1 << 64) - 1


class SplitMix64:                                   # testkit.py:95-151
    def __init__(self, seed):
        self.state = int(seed) & _M64

    def next_u64(self):
        self.state = (self.state + 0x9E3779B97F4A7C15) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def uniform(self):
        return (self.next_u64() >> 11) * 2.0 ** -53

    def normal(self):
        u1 = self.uniform()
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log1p(-u1)) * math.cos(2.0 * math.pi * u2)

    def normals(self, k, scale=1.0):
        return np.array([scale * self.normal() for _ in range(k)])


def _bernoulli_csc(rng, nrows, ncols, density, scale):   # testkit.py:205-216
    cp = np.zeros(ncols + 1, dtype=np.int64)
    rows = []
    for j in range(ncols):
        for i in range(nrows):
            if rng.uniform() < density:
                rows.append(i)
        cp[j + 1] = len(rows)
    rows = np.array(rows, dtype=np.int64)
    return Q.Csc(nrows, ncols, cp, rows, rng.normals(rows.size, scale))


def _gram_ridge(M, eps):                                  # testkit.py:219-246
    n = M.ncols
    sup = [M.row_idx[M.col_ptr[j]:M.col_ptr[j + 1]] for j in range(n)]
    val = [M.values[M.col_ptr[j]:M.col_ptr[j + 1]] for j in range(n)]
    cp = np.zeros(n + 1, dtype=np.int64)
    rows, vals = [], []
    for j in range(n):
        for i in range(n):
            common, ia, ib = np.intersect1d(sup[i], sup[j], assume_unique=True,
                                            return_indices=True)
            if common.size == 0 and i != j:
                continue
            v = math.fsum(val[i][ia] * val[j][ib])
            if i == j:
                v += eps
            rows.append(i)
            vals.append(v)
        cp[j + 1] = len(rows)
    return Q.Csc(n, n, cp, np.array(rows, dtype=np.int64), np.array(vals))


def _probes(dim):                                         # testkit.py:249-257
    pr = np.zeros((6, dim))
    pr[0, 0], pr[1, 0] = 1.0, -1.0
    pr[2] = 1.0 / math.sqrt(dim)
    pr[3] = -pr[2]
    pr[4] = np.where(np.arange(dim) % 2 == 0, 1.0, -1.0) / math.sqrt(dim)
    pr[5] = -pr[4]
    return pr


def _dmat(b, v):
    D = C.Derivative([b], v, dual=True)
    return np.stack([D.matvec(e) for e in np.eye(b.dim)], axis=1)


def stable_block(b, w, margin):                           # testkit.py:270-300
    t = margin * (1.0 + np.linalg.norm(w))
    if b.kind == "zero":
        return True
    if b.kind == "nonneg":
        return bool(np.min(np.abs(w)) >= t)
    if b.kind == "soc":
        tail = np.linalg.norm(w[1:])
        return bool(abs(tail - w[0]) >= t and abs(tail + w[0]) >= t)
    if b.kind == "psd":
        return bool(np.min(np.abs(np.linalg.eigvalsh(C.smat(w, b.order)))) >= t)
    try:
        ref = _dmat(b, -w)
        thr = 0.03 * (1.0 + np.linalg.norm(ref))
        for pr in _probes(b.dim):
            if np.linalg.norm(_dmat(b, -w + t * pr) - ref) > thr:
                return False
    except C.BlockFailure:
        return False
    return True


def generate(seed, n, m, blocks, density=0.3, scale=1.0, margin=1e-6):
    """testkit.generate (testkit.py:318-343).  Returns (Problem, Sol)."""
    rng = SplitMix64(seed)
    A = _bernoulli_csc(rng, m, n, density, scale)
    M = _bernoulli_csc(rng, n, n, density, scale)
    P = _gram_ridge(M, 1e-3 * scale)
    x = rng.normals(n, scale)
    w = np.empty(m)
    offs = C.offsets(blocks)
    for i, b in enumerate(blocks):
        for _ in range(100):
            cand = rng.normals(b.dim, scale)
            if stable_block(b, cand, margin):
                break
        else:
            raise RuntimeError(f"block {i}: no stable point")
        w[offs[i]:offs[i + 1]] = cand
    s = C.project(blocks, w)
    y = s - w
    b_ = Q.spmv(A, x) + s
    q = -(Q.spmv(P, x) + Q.spmv_t(A, y))
    return Q.Problem(P, A, q, b_, list(blocks)), Q.Sol(x, y, s), rng


def c1_ref(seed=0):
    """Configuration C1-ref of SURVEY.md §8(d)."""
    blocks = [C.block("zero", 30), C.block("nonneg", 120)]
    th, sol, _ = generate(seed, 100, 150, blocks, density=0.1)
    return th, sol


def golden_directions(th, seed):
    """Direction draws of the reference golden files (pkg/tests/golden/regenerate.py:336-360)."""
    rng = SplitMix64(seed)
    P = th.P
    drawn, pv = {}, np.zeros(P.values.size)
    for col in range(P.ncols):
        for k in range(P.col_ptr[col], P.col_ptr[col + 1]):
            key = (min(P.row_idx[k], col), max(P.row_idx[k], col))
            if key not in drawn:
                drawn[key] = rng.normal()
            pv[k] = drawn[key]
    dP = Q.Csc(P.nrows, P.ncols, P.col_ptr, P.row_idx, pv)
    dA = Q.Csc(th.A.nrows, th.A.ncols, th.A.col_ptr, th.A.row_idx, rng.normals(th.A.values.size))
    dq = rng.normals(P.ncols)
    db = rng.normals(th.A.nrows)
    de = Q.Delta(rng.normals(P.ncols), rng.normals(th.A.nrows), rng.normals(th.A.nrows))
    return Q.Pert(dP, dA, dq, db), de
