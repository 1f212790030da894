"""The reference's own reproducibility on its golden files at its DEFAULT
LSMR tolerance (atol = btol = 1e-10): run the oracle (pinned to the goldens
with exact iteration counts, tests/test_oracle.py) with every F / F' output
perturbed by 1e-16 relative noise -- what any implementation with another
summation order sees -- and record, per kind, the worst relative-scaled gap
to the frozen golden (helpers.py:37-44 metric) and the iteration spread.

    python tools/golden_noise.py > tests/golden/golden_noise.json

integration/conegrad_plugin.py relaxes the golden comparisons of the
reference's own suite to max(1e-6, 10 x this spread) per kind (SURVEY §8(c):
zero ~1e-6, nonneg ~1e-3 measured reachable).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from fixtures import instance, load  # noqa: E402
from oracle import qcp as Q  # noqa: E402

KINDS = ["zero", "nonneg", "soc", "psd", "exp", "dexp", "pow", "dpow"]


def sgap(got, want):
    got, want = np.asarray(got, float), np.asarray(want, float)
    return float(np.max(np.abs(got - want))) / (1.0 + float(np.max(np.abs(want)))) if want.size else 0.0


def main(draws=16):
    out = {}
    make_F = Q.make_F
    for kind in KINDS:
        d = load(f"golden_{kind}.npz")
        th, sol, pert, de = instance(d)
        worst_j = worst_v = 0.0
        its_j, its_v = [], []
        flags_j, flags_v = set(), set()
        for seed in range(draws):
            rng = np.random.default_rng(seed)

            def noisy_F(th_, z_, rng=rng):
                F = make_F(th_, z_)
                nz = lambda r: r * (1 + 1e-16 * rng.standard_normal(r.size))
                return Q.Operator(lambda w: nz(F.matvec(w)), lambda w: nz(F.rmatvec(w)), z_.size)

            Q.make_F = noisy_F
            try:
                dl, diag_j, dj = Q.jvp(th, sol, pert)
                gv, diag_v, dv = Q.vjp(th, sol, de)
                flags_j.add((bool(diag_j.converged), bool(diag_j.derivative_unreliable)))
                flags_v.add((bool(diag_v.converged), bool(diag_v.derivative_unreliable)))
            finally:
                Q.make_F = make_F
            worst_j = max(worst_j, sgap(dl.dx, d["jvp_dx"]), sgap(dl.dy, d["jvp_dy"]), sgap(dl.ds, d["jvp_ds"]))
            worst_v = max(worst_v, sgap(gv.dP.values, d["vjp_dP"]), sgap(gv.dA.values, d["vjp_dA"]),
                          sgap(gv.dq, d["vjp_dq"]), sgap(gv.db, d["vjp_db"]))
            its_j.append(dj.itn)
            its_v.append(dv.itn)
        out[kind] = {"jvp_gap": worst_j, "vjp_gap": worst_v, "jvp_its": [min(its_j), max(its_j)],
                     "vjp_its": [min(its_v), max(its_v)], "golden_its": [int(d["jvp_its"]), int(d["vjp_its"])],
                     # (converged, derivative_unreliable) pairs the reference itself produced
                     "jvp_flags": sorted([list(f) for f in flags_j]), "vjp_flags": sorted([list(f) for f in flags_v]),
                     "draws": draws}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
