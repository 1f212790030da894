"""Synthetic QCP instances of the benchmark shapes.

KKT-reverse construction, vectorised in NumPy so batches of thousands of
problems build in seconds: draw a complementary pair (s in K, y in K*,
s'y = 0) per cone block, a primal x, then set b = A x + s and
q = -(P x + A'y) so (x, y, s) is optimal by construction.  Complementary
pairs are drawn analytically (boundary points with their normal cones, or
one side zero) so no projection has to be solved to build an instance.

Conditioning recipe: A's values are N(0,1)/sqrt(nnz per
row); P = I + (sparse Gram) or a positive diagonal.

Configurations (BASELINE.json ``configs``):
  c1  n=100,   m=150    zero(30)+nonneg(120), density 0.1
  c2  n=2000,  m=4000   500 x SOC(8), nnz(A) ~ 1e5
  c3  n=20000, m=40002  6667 x exp + 6667 x pow(0.5), nnz(A) ~ 1e6
  c4  n=20000, m=280336 512 x PSD(32) + nonneg(10000), nnz(A) ~ 2e6
  c5a batch of 4096 x (n=1000, m=1500: nonneg(500) + 100 x SOC(10), nnz(A) 1.5e4)
  c5b LASSO canonical form, features 10000 x 5000 dense: n = m = 20000, nnz(A) ~ 5.0e7
"""

from dataclasses import dataclass, field

import numpy as np

KIND_CODE = {"zero": 0, "nonneg": 1, "soc": 2, "psd": 3, "exp": 4, "dexp": 5, "pow": 6, "dpow": 7}


@dataclass
class Batch:
    """Concatenated batch in the C-ABI layout (qg_batch_desc), host side."""

    n: list
    m: list
    blocks: list                  # per problem: list of (kind, dim, order, alpha)
    P_colptr: np.ndarray
    P_rowidx: np.ndarray
    P_vals: np.ndarray
    A_colptr: np.ndarray
    A_rowidx: np.ndarray
    A_vals: np.ndarray
    q: np.ndarray
    b: np.ndarray
    x: np.ndarray
    y: np.ndarray
    s: np.ndarray
    P_nnz: list = field(default_factory=list)
    A_nnz: list = field(default_factory=list)

    @property
    def B(self):
        return len(self.n)


@dataclass
class Directions:
    dP: np.ndarray   # on P's pattern (symmetric), concatenated
    dA: np.ndarray
    dq: np.ndarray
    db: np.ndarray
    dx: np.ndarray
    dy: np.ndarray
    ds: np.ndarray


class _Block:
    __slots__ = ("kind", "dim", "order", "alpha")

    def __init__(self, kind, dim, order=None, alpha=None):
        self.kind, self.dim, self.order, self.alpha = kind, dim, order, alpha


# ---------------------------------------------------------------------------
# sparse pieces (one problem or a batch of identical shapes)
# ---------------------------------------------------------------------------

def _csc_batch(rng, B, nrows, ncols, nnz_target):
    """B random CSC patterns (rows strictly increasing per column)."""
    total = nrows * ncols
    k = min(int(nnz_target * 1.02) + 8, total)
    keys = rng.integers(0, total, size=(B, k), dtype=np.int64)
    keys += (np.arange(B, dtype=np.int64) * total)[:, None]
    keys = np.unique(keys.ravel())
    prob = keys // total
    loc = keys - prob * total
    col, row = loc // nrows, loc % nrows
    counts = np.bincount(prob * ncols + col, minlength=B * ncols).reshape(B, ncols)
    colptr = np.zeros((B, ncols + 1), dtype=np.int64)
    np.cumsum(counts, axis=1, out=colptr[:, 1:])
    nnz = colptr[:, -1].copy()
    return colptr.ravel(), row.astype(np.int64), nnz, prob


def _row_scale(rows_global, nrows_total, vals):
    cnt = np.bincount(rows_global, minlength=nrows_total).astype(np.float64)
    return vals / np.sqrt(np.maximum(cnt, 1.0))[rows_global]


def _gram_plus_identity(rng, n, per_col=4):
    """P = M'M + I with M sparse (per_col entries per column), CSC, full pattern."""
    import scipy.sparse as sp

    M = sp.random(n, n, density=per_col / n, format="csc", random_state=np.random.RandomState(rng.integers(2**31)),
                  data_rvs=rng.standard_normal)
    M.data /= np.sqrt(per_col)
    P = (M.T @ M + sp.identity(n)).tocsc()
    P = 0.5 * (P + P.T)
    P = P.tocsc()
    P.sort_indices()
    return P.indptr.astype(np.int64), P.indices.astype(np.int64), P.data.astype(np.float64)


# ---------------------------------------------------------------------------
# complementary pairs per cone kind (vectorised over blocks)
# ---------------------------------------------------------------------------

def _pairs(rng, blocks):
    """Return (s, y) for the concatenated blocks with s in K, y in K*, s'y = 0."""
    m = sum(b.dim for b in blocks)
    s, y = np.zeros(m), np.zeros(m)
    off = 0
    groups = {}
    for b in blocks:
        groups.setdefault((b.kind, b.dim, b.order, b.alpha), []).append(off)
        off += b.dim
    for (kind, dim, order, alpha), offs in groups.items():
        offs = np.array(offs)
        idx = offs[:, None] + np.arange(dim)[None, :]
        nb = len(offs)
        if kind == "zero":
            y[idx] = rng.standard_normal((nb, dim))
        elif kind == "nonneg":
            w = rng.standard_normal((nb, dim))
            w = np.where(np.abs(w) < 1e-3, 1e-3, w)
            s[idx], y[idx] = np.maximum(w, 0.0), np.maximum(-w, 0.0)
        elif kind == "soc":
            w = rng.standard_normal((nb, dim))
            t, u = w[:, 0], w[:, 1:]
            nu = np.linalg.norm(u, axis=1)
            proj = np.where((nu <= -t)[:, None], 0.0,
                            np.where((nu <= t)[:, None], w,
                                     0.5 * (1.0 + t / np.maximum(nu, 1e-300))[:, None]
                                     * np.concatenate([nu[:, None], u], axis=1)))
            s[idx], y[idx] = proj, proj - w
        elif kind == "psd":
            G = rng.standard_normal((nb, order, order))
            W = 0.5 * (G + np.swapaxes(G, 1, 2))
            lam, V = np.linalg.eigh(W)
            lam = np.where(np.abs(lam) < 1e-2, 1e-2, lam)
            Sp = (V * np.maximum(lam, 0.0)[:, None, :]) @ np.swapaxes(V, 1, 2)
            Sn = (V * np.maximum(-lam, 0.0)[:, None, :]) @ np.swapaxes(V, 1, 2)
            cols, rows = np.triu_indices(order)
            sc = np.where(rows == cols, 1.0, np.sqrt(2.0))
            s[idx], y[idx] = Sp[:, rows, cols] * sc, Sn[:, rows, cols] * sc
        else:
            base = "exp" if kind in ("exp", "dexp") else "pow"
            a = alpha if alpha else 0.5
            mode = rng.random(nb)
            t = rng.uniform(0.5, 2.0, nb)
            mu = rng.uniform(0.5, 2.0, nb)
            if base == "exp":
                rho = rng.uniform(-1.5, 1.5, nb)
                e = np.exp(rho)
                pk = t[:, None] * np.stack([rho, np.ones(nb), e], 1)            # on K_exp boundary
                pd = mu[:, None] * np.stack([-e, (rho - 1.0) * e, np.ones(nb)], 1)  # normal, in K_exp*
                ik = np.stack([-t, t, 2.0 * t], 1)                               # interior of K_exp
                idl = np.stack([-t, np.ones(nb) * 0.5 * t, 2.0 * t], 1)          # interior of K_exp*
            else:
                xx, yy = rng.uniform(0.5, 2.0, nb), rng.uniform(0.5, 2.0, nb)
                sg = np.where(rng.random(nb) < 0.5, -1.0, 1.0)
                zz = sg * xx ** a * yy ** (1 - a)
                pk = np.stack([xx, yy, zz], 1)
                pd = mu[:, None] * np.stack([a * xx ** (a - 1) * yy ** (1 - a),
                                             (1 - a) * xx ** a * yy ** (-a), -sg], 1)
                ik = np.stack([xx, yy, 0.3 * zz], 1)
                idl = np.stack([a * xx, (1 - a) * yy, 0.3 * zz], 1)
            sk, yk = pk.copy(), pd.copy()
            inter = mode < 0.1     # s interior, y = 0
            dint = (mode >= 0.1) & (mode < 0.2)   # s = 0, y interior of K*
            sk[inter], yk[inter] = ik[inter], 0.0
            sk[dint], yk[dint] = 0.0, idl[dint]
            if kind in ("dexp", "dpow"):   # K is the dual cone: roles swap
                sk, yk = yk, sk
            s[idx], y[idx] = sk, yk
    return s, y


def _spmv_csc(colptr, rowidx, vals, nrows, x):
    import scipy.sparse as sp

    M = sp.csc_matrix((vals, rowidx, colptr), shape=(nrows, len(colptr) - 1))
    return M @ x, M


# ---------------------------------------------------------------------------
# configurations
# ---------------------------------------------------------------------------

def _cones(config):
    if config == "c1":
        return [_Block("zero", 30), _Block("nonneg", 120)], 100, 150, 1600
    if config == "c2":
        return [_Block("soc", 8) for _ in range(500)], 2000, 4000, 100_000
    if config == "c3":
        return ([_Block("exp", 3) for _ in range(6667)] + [_Block("pow", 3, alpha=0.5) for _ in range(6667)],
                20000, 40002, 1_000_000)
    if config == "c4":
        return ([_Block("nonneg", 10000)] + [_Block("psd", 528, order=32) for _ in range(512)],
                20000, 10000 + 512 * 528, 2_000_000)
    if config == "c5a":
        return [_Block("nonneg", 500)] + [_Block("soc", 10) for _ in range(100)], 1000, 1500, 15_000
    raise ValueError(config)


def _canonical(blocks):
    order = {k: i for i, k in enumerate(KIND_CODE)}
    return sorted(blocks, key=lambda b: order[b.kind])


def custom(cones, n, nnzA, seed=0, batch=1, diag_P=True):
    """A batch of problems with the given cone list [(kind, dim, order, alpha)]."""
    blocks = [_Block(k, d, o or None, a or None) for (k, d, o, a) in cones]
    m = sum(b.dim for b in blocks)
    return generate(None, seed=seed, batch=batch, diag_P=diag_P, _shape=(blocks, n, m, nnzA))


def generate(config, seed=0, batch=1, diag_P=None, _shape=None):
    """Build a Batch of ``batch`` problems of configuration ``config``."""
    if config == "c5b":
        if batch != 1:
            raise ValueError("c5b is a single problem")
        return _lasso(seed)
    rng = np.random.default_rng(seed)
    blocks, n, m, nnzA = _shape if _shape is not None else _cones(config)
    blocks = _canonical(blocks)
    B = batch
    if diag_P is None:
        diag_P = config in ("c1", "c5a")
    # A: Bernoulli-like pattern, values N(0,1)/sqrt(nnz per row)
    A_colptr, A_rowidx, A_nnz, A_prob = _csc_batch(rng, B, m, n, nnzA)
    vals = rng.standard_normal(A_rowidx.size)
    A_vals = _row_scale(A_prob * m + A_rowidx, B * m, vals)
    # P
    if diag_P:
        P_colptr = np.tile(np.arange(n + 1, dtype=np.int64), B)
        P_rowidx = np.tile(np.arange(n, dtype=np.int64), B)
        P_vals = 1.0 + np.abs(rng.standard_normal(B * n))
        P_nnz = [n] * B
    else:
        cps, ris, vs, P_nnz = [], [], [], []
        for _ in range(B):
            cp, ri, v = _gram_plus_identity(rng, n)
            cps.append(cp), ris.append(ri), vs.append(v), P_nnz.append(int(cp[-1]))
        P_colptr, P_rowidx, P_vals = np.concatenate(cps), np.concatenate(ris), np.concatenate(vs)
    # KKT-reverse
    x = rng.standard_normal(B * n)
    s = np.zeros(B * m)
    y = np.zeros(B * m)
    for p in range(B):
        sp_, yp = _pairs(rng, blocks)
        s[p * m:(p + 1) * m], y[p * m:(p + 1) * m] = sp_, yp
    q = np.empty(B * n)
    b = np.empty(B * m)
    po = np.concatenate([[0], np.cumsum(P_nnz)])
    ao = np.concatenate([[0], np.cumsum(A_nnz)])
    for p in range(B):
        xs, ys = slice(p * n, (p + 1) * n), slice(p * m, (p + 1) * m)
        Ax, Am = _spmv_csc(A_colptr[p * (n + 1):(p + 1) * (n + 1)], A_rowidx[ao[p]:ao[p + 1]],
                           A_vals[ao[p]:ao[p + 1]], m, x[xs])
        Px, _ = _spmv_csc(P_colptr[p * (n + 1):(p + 1) * (n + 1)], P_rowidx[po[p]:po[p + 1]],
                          P_vals[po[p]:po[p + 1]], n, x[xs])
        b[ys] = Ax + s[ys]
        q[xs] = -(Px + Am.T @ y[ys])
    blk = [(bb.kind, bb.dim, bb.order or 0, bb.alpha or 0.0) for bb in blocks]
    return Batch([n] * B, [m] * B, [blk] * B, P_colptr, P_rowidx, P_vals, A_colptr, A_rowidx, A_vals,
                 q, b, x, y, s, list(map(int, P_nnz)), list(map(int, A_nnz)))


def _lasso(seed):
    """LASSO canonical form: F in R^{10000 x 5000} dense,
    A = [[F, 0, -I], [I, -I, 0], [-I, -I, 0]] over (w, t, r), P = blkdiag(0, 0, I),
    cones zero(10000) + nonneg(10000); n = m = 20000, nnz(A) ~ 5.0e7."""
    rng = np.random.default_rng(seed)
    p_rows, p_feat = 10000, 5000
    n = p_feat + p_feat + p_rows
    m = p_rows + 2 * p_feat
    Fd = rng.standard_normal((p_rows, p_feat)) / np.sqrt(p_feat)
    # CSC column by column: w_j column = [F[:, j]; e_j; -e_j], t_j = [0; -e_j; -e_j], r_i = [-e_i; 0; 0]
    cols_ptr = [0]
    rows, vals = [], []
    ar = np.arange(p_rows, dtype=np.int64)
    colw_rows = np.concatenate([np.tile(ar, (p_feat, 1)),
                                (p_rows + np.arange(p_feat, dtype=np.int64))[:, None],
                                (p_rows + p_feat + np.arange(p_feat, dtype=np.int64))[:, None]], axis=1)
    colw_vals = np.concatenate([Fd.T, np.ones((p_feat, 1)), -np.ones((p_feat, 1))], axis=1)
    rows.append(colw_rows.ravel()), vals.append(colw_vals.ravel())
    t_rows = np.stack([p_rows + np.arange(p_feat), p_rows + p_feat + np.arange(p_feat)], 1).astype(np.int64)
    rows.append(t_rows.ravel()), vals.append(-np.ones(2 * p_feat))
    rows.append(ar.copy()), vals.append(-np.ones(p_rows))
    counts = np.concatenate([np.full(p_feat, p_rows + 2), np.full(p_feat, 2), np.full(p_rows, 1)])
    A_colptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    A_rowidx = np.concatenate(rows)
    A_vals = np.concatenate(vals)
    P_colptr = np.concatenate([np.zeros(2 * p_feat + 1, dtype=np.int64),
                               np.arange(1, p_rows + 1, dtype=np.int64)])
    P_rowidx = np.arange(2 * p_feat, n, dtype=np.int64)
    P_vals = np.ones(p_rows)
    blocks = [_Block("zero", p_rows), _Block("nonneg", 2 * p_feat)]
    s, y = _pairs(rng, blocks)
    x = rng.standard_normal(n)
    Ax, Am = _spmv_csc(A_colptr, A_rowidx, A_vals, m, x)
    Px, _ = _spmv_csc(P_colptr, P_rowidx, P_vals, n, x)
    b = Ax + s
    q = -(Px + Am.T @ y)
    blk = [(bb.kind, bb.dim, 0, 0.0) for bb in blocks]
    del cols_ptr
    return Batch([n], [m], [blk], P_colptr, P_rowidx, P_vals, A_colptr, A_rowidx, A_vals, q, b, x, y, s,
                 [int(P_colptr[-1])], [int(A_colptr[-1])])


def directions(batch, seed=1):
    """Random data / solution directions; dP symmetric on P's pattern."""
    rng = np.random.default_rng(seed)
    dP = np.empty(batch.P_vals.size)
    off = 0
    cpo = 0
    for p in range(batch.B):
        n, nnz = batch.n[p], batch.P_nnz[p]
        cp = batch.P_colptr[cpo:cpo + n + 1]
        ri = batch.P_rowidx[off:off + nnz]
        cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(cp))
        key = np.minimum(ri, cols) * n + np.maximum(ri, cols)
        uniq, inv = np.unique(key, return_inverse=True)
        dP[off:off + nnz] = rng.standard_normal(uniq.size)[inv]
        off += nnz
        cpo += n + 1
    NX, NY = sum(batch.n), sum(batch.m)
    return Directions(dP, rng.standard_normal(batch.A_vals.size), rng.standard_normal(NX), rng.standard_normal(NY),
                      rng.standard_normal(NX), rng.standard_normal(NY), rng.standard_normal(NY))


def problem_objects(batch, p, pkg):
    """Problem p of a batch as (ProblemData, Solution) objects of ``pkg``
    (the product package or the oracle's namedtuples)."""
    n, m = batch.n[p], batch.m[p]
    cpo = sum(batch.n[:p]) + p
    po, ao = sum(batch.P_nnz[:p]), sum(batch.A_nnz[:p])
    xo, yo = sum(batch.n[:p]), sum(batch.m[:p])
    Pc = (batch.P_colptr[cpo:cpo + n + 1], batch.P_rowidx[po:po + batch.P_nnz[p]], batch.P_vals[po:po + batch.P_nnz[p]])
    Ac = (batch.A_colptr[cpo:cpo + n + 1], batch.A_rowidx[ao:ao + batch.A_nnz[p]], batch.A_vals[ao:ao + batch.A_nnz[p]])
    return dict(n=n, m=m, P=Pc, A=Ac, q=batch.q[xo:xo + n], b=batch.b[yo:yo + m], x=batch.x[xo:xo + n],
                y=batch.y[yo:yo + m], s=batch.s[yo:yo + m], blocks=batch.blocks[p],
                slices=(xo, yo, po, ao))
