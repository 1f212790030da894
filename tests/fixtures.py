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
