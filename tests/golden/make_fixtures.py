"""Generate the committed parity fixtures from the REAL reference.

Run in the build container (the only place /root/reference exists)::

    python tests/golden/make_fixtures.py

It imports ``conegrad`` straight from ``/root/reference/pkg/src`` (its
pure-NumPy kernel backend is bit-identical to the Cython one, see
``_kernels/pyref.py:1-7``) and writes ``tests/golden/*.npz``:

* ``golden_<kind>.npz`` -- the reference's own committed golden instances
  (``pkg/tests/golden/<kind>_*.json``) with their frozen jvp/vjp outputs,
  plus outputs of the reference run here: ``F w`` / ``F' w`` for random
  ``w``, fixed-cap (K=20, atol=btol=0) jvp/vjp, and the dual projection and
  its derivative at the embedding point.
* ``cones_kat.npz`` -- projections and projection derivatives (primal and
  dual) for every cone kind on seeded random and edge-case points.
* ``c1ref.npz`` -- configuration C1-ref (``testkit.generate`` seed 0, n=100,
  m=150, zero(30)+nonneg(120), density 0.1) with golden-style directions
  and the reference's K=20 and K=200 fixed-cap jvp/vjp outputs.

Nothing under tests/ reads /root/reference at run time; only these files.
"""

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

import conegrad  # noqa: E402
from conegrad import cones, jsonio, lsmr as lsmr_mod, solution_map as sm  # noqa: E402
from conegrad.embedding import _embedding_project, make_F, dthetaq_adjoint  # noqa: E402
from conegrad.errors import ConegradError  # noqa: E402
from conegrad.testkit import GeneratorConfig, generate  # noqa: E402

OUT = Path(__file__).resolve().parent
KINDS = ("zero", "nonneg", "soc", "psd", "exp", "dexp", "pow", "dpow")
KCODE = {k: i for i, k in enumerate(KINDS)}


def cone_arrays(spec):
    kinds = np.array([KCODE[b.kind] for b in spec.blocks], dtype=np.int64)
    dims = np.array([b.dim for b in spec.blocks], dtype=np.int64)
    orders = np.array([b.order if b.order else 0 for b in spec.blocks], dtype=np.int64)
    alphas = np.array([b.alpha if b.alpha else 0.0 for b in spec.blocks])
    return dict(cone_kind=kinds, cone_dim=dims, cone_order=orders, cone_alpha=alphas)


def csc_arrays(prefix, M):
    return {f"{prefix}_shape": np.array(M.shape, dtype=np.int64),
            f"{prefix}_colptr": M.col_ptr.copy(), f"{prefix}_rowidx": M.row_idx.copy(),
            f"{prefix}_vals": M.values.copy()}


def problem_arrays(theta, sol):
    d = cone_arrays(theta.cone)
    d.update(csc_arrays("P", theta.P))
    d.update(csc_arrays("A", theta.A))
    d.update(q=theta.q, b=theta.b, x=sol.x, y=sol.y, s=sol.s)
    return d


def run_fixed(theta, sol, dtheta, delta, K):
    out = {}
    dl, dg = sm.jvp(theta, sol, dtheta, atol=0.0, btol=0.0, max_iter=K, check=False)
    out.update({f"k{K}_jvp_dx": dl.dx, f"k{K}_jvp_dy": dl.dy, f"k{K}_jvp_ds": dl.ds,
                f"k{K}_jvp_its": np.int64(dg.iterations), f"k{K}_jvp_res": dg.residual_norm})
    g, vg = sm.vjp(theta, sol, delta, atol=0.0, btol=0.0, max_iter=K, check=False)
    out.update({f"k{K}_vjp_dP": g.dP.values, f"k{K}_vjp_dA": g.dA.values,
                f"k{K}_vjp_dq": g.dq, f"k{K}_vjp_db": g.db,
                f"k{K}_vjp_its": np.int64(vg.iterations), f"k{K}_vjp_res": vg.residual_norm})
    return out


def run_tol(theta, sol, dtheta, delta, tol, tag):
    out = {}
    dl, dg = sm.jvp(theta, sol, dtheta, atol=tol, btol=tol)
    out.update({f"{tag}_jvp_dx": dl.dx, f"{tag}_jvp_dy": dl.dy, f"{tag}_jvp_ds": dl.ds,
                f"{tag}_jvp_its": np.int64(dg.iterations), f"{tag}_jvp_res": dg.residual_norm})
    g, vg = sm.vjp(theta, sol, delta, atol=tol, btol=tol)
    out.update({f"{tag}_vjp_dP": g.dP.values, f"{tag}_vjp_dA": g.dA.values,
                f"{tag}_vjp_dq": g.dq, f"{tag}_vjp_db": g.db,
                f"{tag}_vjp_its": np.int64(vg.iterations), f"{tag}_vjp_res": vg.residual_norm})
    return out


def operator_probes(theta, sol, rng, count=3):
    z = sm.embed(sol)
    F = make_F(theta, z)
    W = rng.standard_normal((count, z.size))
    Fw = np.stack([F.matvec(w) for w in W])
    FTw = np.stack([F.rmatvec(w) for w in W])
    pz = _embedding_project(theta, z)
    mid = z[theta.n:-1]
    D = cones.dprojection_dual(theta.cone, mid)
    dmid = np.stack([D.matvec(w[theta.n:-1]) for w in W])
    return dict(op_w=W, op_Fw=Fw, op_FTw=FTw, op_pz=pz, op_dpi_mid=dmid)


def golden_file(kind):
    load = lambda s: json.loads((REF / "tests" / "golden" / f"{kind}_{s}.json").read_text())
    prob, soln = load("problem"), load("solution")
    theta = jsonio.parse_problem(prob)
    sol = jsonio.parse_solution(soln, theta.n, theta.m)
    dtheta = jsonio.parse_perturbation(load("perturbation"), theta.n, theta.m)
    delta = jsonio.parse_delta(load("delta"), theta.n, theta.m)
    jv, vj = load("jvp"), load("vjp")
    d = problem_arrays(theta, sol)
    d.update(csc_arrays("dP", dtheta.dP))
    d.update(csc_arrays("dA", dtheta.dA))
    d.update(dq=dtheta.dq, db=dtheta.db, dx=delta.dx, dy=delta.dy, ds=delta.ds)
    # frozen outputs committed by the reference
    d.update(jvp_dx=np.array(jv["dx"]), jvp_dy=np.array(jv["dy"]), jvp_ds=np.array(jv["ds"]),
             jvp_its=np.int64(jv["diagnostics"]["lsmr_iterations"]),
             jvp_res=jv["diagnostics"]["lsmr_residual"],
             jvp_conv=np.int64(jv["diagnostics"]["converged"]),
             jvp_unrel=np.int64(jv["diagnostics"]["derivative_unreliable"]),
             vjp_dP=np.array(vj["dP"]["values"]), vjp_dA=np.array(vj["dA"]["values"]),
             vjp_dq=np.array(vj["dq"]), vjp_db=np.array(vj["db"]),
             vjp_its=np.int64(vj["diagnostics"]["lsmr_iterations"]),
             vjp_res=vj["diagnostics"]["lsmr_residual"],
             vjp_conv=np.int64(vj["diagnostics"]["converged"]),
             vjp_unrel=np.int64(vj["diagnostics"]["derivative_unreliable"]))
    # rerun here: the frozen outputs must reproduce (reference test_golden TOL 1e-9)
    dl, dg = sm.jvp(theta, sol, dtheta)
    assert np.max(np.abs(dl.dx - d["jvp_dx"])) <= 1e-9 * (1 + np.max(np.abs(d["jvp_dx"])))
    assert dg.iterations == d["jvp_its"]
    rng = np.random.default_rng(KCODE[kind] + 100)
    d.update(operator_probes(theta, sol, rng))
    d.update(run_fixed(theta, sol, dtheta, delta, 3))
    d.update(run_tol(theta, sol, dtheta, delta, 1e-14, "t14"))
    d.update(kkt=np.array([v for k, v in sm.check_solution(theta, sol).as_dict().items()
                           if k not in ("tol", "ok")]))
    np.savez_compressed(OUT / f"golden_{kind}.npz", **d)
    return d


def cone_points(kind, rng, count):
    dim = 3 if kind in ("exp", "dexp", "pow", "dpow") else (6 if kind == "psd" else 5)
    pts = [rng.standard_normal(dim) * rng.choice([0.3, 1.0, 4.0]) for _ in range(count)]
    edge = [np.zeros(dim)]
    if kind == "soc":
        edge += [np.array([5.0, 3.0, 4.0, 0.0, 0.0]), np.array([-5.0, 3.0, 4.0, 0.0, 0.0]),
                 np.array([0.0, 3.0, 4.0, 0.0, 0.0]), np.array([1.0, 0.0, 0.0, 0.0, 0.0])]
    if kind == "nonneg":
        edge += [np.array([0.0, 1.0, -1.0, 0.0, 2.0])]
    if kind in ("exp", "dexp"):
        edge += [np.array([0.0, 1.0, 1.0]), np.array([-1.0, -1.0, 2.0]), np.array([-1.0, -2.0, -1.0]),
                 np.array([1.0, 1.0, -3.0]), np.array([0.5, 0.0, 1.0])]
    if kind in ("pow", "dpow"):
        edge += [np.array([0.0, 0.0, 2.0]), np.array([1.0, 2.0, 0.5]), np.array([1.0, -2.0, 0.0]),
                 np.array([-1.0, 2.0, 0.0]), np.array([-1.0, -1.0, 0.3])]
    return edge + pts


def cones_kat():
    rng = np.random.default_rng(7)
    rec = {}
    for kind in KINDS:
        for alpha in ((0.3, 0.5, 0.8) if kind in ("pow", "dpow") else (None,)):
            tag = kind if alpha is None else f"{kind}_{alpha}"
            if kind == "psd":
                blk = cones.ConeBlock.psd(3)
            elif kind in ("pow", "dpow"):
                blk = cones.ConeBlock(kind, alpha=alpha)
            elif kind in ("exp", "dexp"):
                blk = cones.ConeBlock(kind)
            else:
                blk = cones.ConeBlock(kind, dim=5)
            spec = cones.ConeSpec([blk])
            P, PP, PD, DD, DP, OK = [], [], [], [], [], []
            for p in cone_points(kind, rng, 120):
                dirs = rng.standard_normal((2, p.size))
                try:
                    pp = cones.project(spec, p)
                    pd = cones.project_dual(spec, p)
                    dd = np.stack([cones.dprojection_dual(spec, p).matvec(e) for e in dirs])
                    dp = np.stack([cones.dprojection(spec, p).matvec(e) for e in dirs])
                    ok = 1
                except ConegradError:
                    pp = pd = np.full(p.size, np.nan)
                    dd = dp = np.full((2, p.size), np.nan)
                    ok = 0
                P.append(np.concatenate([p, dirs.ravel()]))
                PP.append(pp), PD.append(pd), DD.append(dd), DP.append(dp), OK.append(ok)
            rec[f"{tag}__pts"] = np.array(P)
            rec[f"{tag}__proj"] = np.array(PP)
            rec[f"{tag}__projdual"] = np.array(PD)
            rec[f"{tag}__dprojdual"] = np.array(DD)
            rec[f"{tag}__dproj"] = np.array(DP)
            rec[f"{tag}__ok"] = np.array(OK)
    # known-answer points from the reference's tests (tests/test_cones.py:229-307)
    np.savez_compressed(OUT / "cones_kat.npz", **rec)


def c1ref():
    spec = cones.ConeSpec([cones.ConeBlock.zero(30), cones.ConeBlock.nonneg(120)])
    theta, sol = generate(GeneratorConfig(0, 100, 150, spec, density=0.1))
    sys.path.insert(0, str(REF / "tests" / "golden"))
    from regenerate import directions
    dtheta, delta = directions(theta, 1042)
    d = problem_arrays(theta, sol)
    d.update(csc_arrays("dP", dtheta.dP))
    d.update(csc_arrays("dA", dtheta.dA))
    d.update(dq=dtheta.dq, db=dtheta.db, dx=delta.dx, dy=delta.dy, ds=delta.ds)
    d.update(run_fixed(theta, sol, dtheta, delta, 3))
    d.update(operator_probes(theta, sol, np.random.default_rng(5)))
    np.savez_compressed(OUT / "c1ref.npz", **d)


# Small instances built with the conditioning recipe by the
# product's synthetic generator; outputs from the reference at atol=btol=1e-14
# (the matched tolerance at which outputs are insensitive to summation order).
RECIPES = {
    "r_qp": ([("zero", 20, 0, 0.0), ("nonneg", 70, 0, 0.0)], 60, 900, True),
    "r_soc": ([("soc", 6, 0, 0.0)] * 12, 60, 1000, False),
    "r_exppow": ([("exp", 3, 0, 0.0)] * 8 + [("dexp", 3, 0, 0.0)] * 8 + [("pow", 3, 0, 0.3)] * 8
                 + [("dpow", 3, 0, 0.7)] * 8, 80, 1400, True),
    "r_psd": ([("nonneg", 10, 0, 0.0)] + [("psd", 21, 6, 0.0)] * 3, 60, 900, False),
    "r_mixed": ([("zero", 5, 0, 0.0), ("nonneg", 10, 0, 0.0), ("soc", 5, 0, 0.0), ("soc", 4, 0, 0.0),
                 ("psd", 10, 4, 0.0), ("exp", 3, 0, 0.0), ("exp", 3, 0, 0.0), ("dexp", 3, 0, 0.0),
                 ("pow", 3, 0, 0.4), ("dpow", 3, 0, 0.6)], 70, 900, True),
}


def recipe(name):
    sys.path.insert(0, str(OUT.parent.parent))
    from paper_2508_17522_b200 import synth
    from conegrad.embedding import DataPerturbation, ProblemData
    from conegrad.solution_map import Solution, SolutionDelta
    from conegrad.sparse import CscMatrix

    cones_, n, nnzA, diagP = RECIPES[name]
    bt = synth.custom(cones_, n, nnzA, seed=11, diag_P=diagP)
    dirs = synth.directions(bt, seed=12)
    o = synth.problem_objects(bt, 0, None)
    m = o["m"]
    blocks = []
    for k, dm, od, al in o["blocks"]:
        blocks.append(cones.ConeBlock(k, dim=dm) if k in ("zero", "nonneg", "soc") else
                      cones.ConeBlock(k, order=od) if k == "psd" else
                      cones.ConeBlock(k, alpha=al) if k in ("pow", "dpow") else cones.ConeBlock(k))
    P = CscMatrix(n, n, *o["P"])
    A = CscMatrix(m, n, *o["A"])
    theta = ProblemData(P, A, o["q"], o["b"], cones.ConeSpec(blocks))
    sol = Solution(o["x"], o["y"], o["s"])
    dtheta = DataPerturbation(P.with_values(dirs.dP), A.with_values(dirs.dA), dirs.dq, dirs.db)
    delta = SolutionDelta(dirs.dx, dirs.dy, dirs.ds)
    d = problem_arrays(theta, sol)
    d.update(csc_arrays("dP", dtheta.dP))
    d.update(csc_arrays("dA", dtheta.dA))
    d.update(dq=dtheta.dq, db=dtheta.db, dx=delta.dx, dy=delta.dy, ds=delta.ds)
    d.update(run_tol(theta, sol, dtheta, delta, 1e-14, "t14"))
    d.update(run_fixed(theta, sol, dtheta, delta, 3))
    d.update(operator_probes(theta, sol, np.random.default_rng(3)))
    np.savez_compressed(OUT / f"{name}.npz", **d)


if __name__ == "__main__":
    for kind in KINDS:
        golden_file(kind)
        print("golden", kind)
    cones_kat()
    print("cones_kat")
    c1ref()
    print("c1ref")
    for name in RECIPES:
        recipe(name)
        print(name)
