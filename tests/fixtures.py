"""Load the committed parity fixtures (tests/golden/*.npz) into plain
structures shared by the oracle tests and the GPU parity tests."""

from pathlib import Path

import numpy as np

from oracle import cones as C
from oracle import qcp as Q

GOLDEN = Path(__file__).resolve().parent / "golden"
KINDS = ("zero", "nonneg", "soc", "psd", "exp", "dexp", "pow", "dpow")


def load(name):
    with np.load(GOLDEN / name) as f:
        return {k: f[k] for k in f.files}


def csc(d, prefix):
    r, c = (int(v) for v in d[f"{prefix}_shape"])
    return Q.Csc(r, c, d[f"{prefix}_colptr"], d[f"{prefix}_rowidx"], d[f"{prefix}_vals"])


def blocks(d):
    out = []
    for k, dim, order, alpha in zip(d["cone_kind"], d["cone_dim"], d["cone_order"], d["cone_alpha"]):
        kind = KINDS[int(k)]
        out.append(C.block(kind, dim=int(dim), order=int(order), alpha=float(alpha)))
    return out


def instance(d):
    th = Q.Problem(csc(d, "P"), csc(d, "A"), d["q"], d["b"], blocks(d))
    sol = Q.Sol(d["x"], d["y"], d["s"])
    pert = Q.Pert(csc(d, "dP"), csc(d, "dA"), d["dq"], d["db"])
    de = Q.Delta(d["dx"], d["dy"], d["ds"])
    return th, sol, pert, de


def gap(got, want):
    """Relative-scaled max gap (reference tests/helpers.py:37-43)."""
    got, want = np.asarray(got, float), np.asarray(want, float)
    assert got.shape == want.shape, (got.shape, want.shape)
    if got.size == 0:
        return 0.0
    return float(np.max(np.abs(got - want))) / (1.0 + float(np.max(np.abs(want))))


def kat_block(tag):
    kind, _, alpha = tag.partition("_")
    if kind == "psd":
        return C.block("psd", order=3)
    if kind in ("pow", "dpow"):
        return C.block(kind, alpha=float(alpha))
    if kind in ("exp", "dexp"):
        return C.block(kind)
    return C.block(kind, dim=5)


def kat_tags():
    d = load("cones_kat.npz")
    return sorted({k.split("__")[0] for k in d})


def product_instance(d):
    """The same fixture as product objects (paper_2508_17522_b200)."""
    import paper_2508_17522_b200 as qg

    def m(prefix):
        r, c = (int(v) for v in d[f"{prefix}_shape"])
        return qg.CscMatrix(r, c, d[f"{prefix}_colptr"], d[f"{prefix}_rowidx"], d[f"{prefix}_vals"])

    blks = []
    for k, dim, order, alpha in zip(d["cone_kind"], d["cone_dim"], d["cone_order"], d["cone_alpha"]):
        kind = KINDS[int(k)]
        blks.append(qg.ConeBlock(kind, dim=int(dim)) if kind in ("zero", "nonneg", "soc") else
                    qg.ConeBlock(kind, order=int(order)) if kind == "psd" else
                    qg.ConeBlock(kind, alpha=float(alpha)) if kind in ("pow", "dpow") else qg.ConeBlock(kind))
    theta = qg.ProblemData(m("P"), m("A"), d["q"], d["b"], qg.ConeSpec(blks))
    sol = qg.Solution(d["x"], d["y"], d["s"])
    pert = qg.DataPerturbation(m("dP"), m("dA"), d["dq"], d["db"])
    delta = qg.SolutionDelta(d["dx"], d["dy"], d["ds"])
    return theta, sol, pert, delta


def product_block(tag):
    import paper_2508_17522_b200 as qg

    kind, _, alpha = tag.partition("_")
    if kind == "psd":
        return qg.ConeBlock.psd(3)
    if kind in ("pow", "dpow"):
        return qg.ConeBlock(kind, alpha=float(alpha))
    if kind in ("exp", "dexp"):
        return qg.ConeBlock(kind)
    return qg.ConeBlock(kind, dim=5)


def synth_instance(cfg, seed=0, **kw):
    """A synthetic instance (paper_2508_17522_b200.synth) as both oracle and
    product objects: returns (oracle tuple, product tuple) of
    (theta, sol, perturbation, delta)."""
    import paper_2508_17522_b200 as qg
    from paper_2508_17522_b200 import synth

    if isinstance(cfg, tuple):
        bt = synth.custom(*cfg, seed=seed, **kw)
    else:
        bt = synth.generate(cfg, seed=seed, **kw)
    dirs = synth.directions(bt, seed=seed + 1)
    o = synth.problem_objects(bt, 0, None)
    n, m = o["n"], o["m"]
    xo, yo, po, ao = o["slices"]
    dPv, dAv = dirs.dP[po:po + o["P"][1].size], dirs.dA[ao:ao + o["A"][1].size]
    dq, db = dirs.dq[xo:xo + n], dirs.db[yo:yo + m]
    dx, dy, ds = dirs.dx[xo:xo + n], dirs.dy[yo:yo + m], dirs.ds[yo:yo + m]
    P, A = Q.Csc(n, n, *o["P"]), Q.Csc(m, n, *o["A"])
    oblocks = [C.block(k, dim=dm, order=od, alpha=al) for (k, dm, od, al) in o["blocks"]]
    ora = (Q.Problem(P, A, o["q"], o["b"], oblocks), Q.Sol(o["x"], o["y"], o["s"]),
           Q.Pert(Q.Csc(n, n, P.col_ptr, P.row_idx, dPv), Q.Csc(m, n, A.col_ptr, A.row_idx, dAv), dq, db),
           Q.Delta(dx, dy, ds))
    pblocks = []
    for k, dm, od, al in o["blocks"]:
        pblocks.append(qg.ConeBlock(k, dim=dm) if k in ("zero", "nonneg", "soc") else
                       qg.ConeBlock(k, order=od) if k == "psd" else
                       qg.ConeBlock(k, alpha=al) if k in ("pow", "dpow") else qg.ConeBlock(k))
    Pm, Am = qg.CscMatrix(n, n, *o["P"]), qg.CscMatrix(m, n, *o["A"])
    theta = qg.ProblemData(Pm, Am, o["q"], o["b"], qg.ConeSpec(pblocks))
    prod = (theta, qg.Solution(o["x"], o["y"], o["s"]),
            qg.DataPerturbation(Pm.with_values(dPv), Am.with_values(dAv), dq, db), qg.SolutionDelta(dx, dy, ds))
    return ora, prod
