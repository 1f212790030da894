"""Binary ingest (binio.py): bit-exact round trips of every object the
reference's JSON carries (jsonio.py:21-33), the batch layout, and the same
validation failures (unknown keys, bad structure) -- host only, no GPU."""

import numpy as np
import pytest

import paper_2508_17522_b200 as qg
from paper_2508_17522_b200 import binio, synth

from fixtures import load, product_instance


def test_problem_and_friends_roundtrip(tmp_path):
    theta, sol, pert, delta = product_instance(load("golden_psd.npz"))
    binio.save_problem(tmp_path / "p.npz", theta)
    binio.save_solution(tmp_path / "s.npz", sol)
    binio.save_perturbation(tmp_path / "d.npz", pert)
    binio.save_delta(tmp_path / "e.npz", delta)
    t2 = binio.load_problem(tmp_path / "p.npz")
    for a, b in ((t2.P, theta.P), (t2.A, theta.A), (pert.dP, binio.load_perturbation(tmp_path / "d.npz").dP)):
        assert a.shape == b.shape and np.array_equal(a.col_ptr, b.col_ptr)
        assert np.array_equal(a.row_idx, b.row_idx) and np.array_equal(a.values, b.values)
    assert np.array_equal(t2.q, theta.q) and np.array_equal(t2.b, theta.b)
    assert [(b.kind, b.dim, b.order, b.alpha) for b in t2.cone.blocks] == \
           [(b.kind, b.dim, b.order, b.alpha) for b in theta.cone.blocks]
    s2 = binio.load_solution(tmp_path / "s.npz")
    assert np.array_equal(s2.x, sol.x) and np.array_equal(s2.s, sol.s)
    e2 = binio.load_delta(tmp_path / "e.npz")
    assert np.array_equal(e2.dy, delta.dy)


def test_all_cone_kinds_roundtrip():
    spec = qg.ConeSpec([qg.ConeBlock.zero(2), qg.ConeBlock.nonneg(3), qg.ConeBlock.soc(4), qg.ConeBlock.psd(3),
                        qg.ConeBlock.exp(), qg.ConeBlock.dual_exp(), qg.ConeBlock.power(0.3),
                        qg.ConeBlock.dual_power(0.7)])
    back = binio.cone_spec(binio.cone_table(spec))
    assert [(b.kind, b.dim, b.order, b.alpha) for b in back.blocks] == \
           [(b.kind, b.dim, b.order, b.alpha) for b in spec.blocks]


def test_batch_roundtrip(tmp_path):
    bt = synth.custom([("nonneg", 7, 0, 0.0), ("soc", 4, 0, 0.0), ("pow", 3, 0, 0.4)], n=9, nnzA=50, seed=2,
                      batch=3)
    arrays = {k: getattr(bt, k) for k in binio._BATCH_ARRAYS}
    binio.save_batch(tmp_path / "b.npz", bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks, arrays)
    n, m, pn, an, blocks, arr = binio.load_batch(tmp_path / "b.npz")
    assert (n, m, pn, an) == (list(bt.n), list(bt.m), list(bt.P_nnz), list(bt.A_nnz))
    assert blocks == [[(k, d, o, a) for (k, d, o, a) in bl] for bl in bt.blocks]
    for k in binio._BATCH_ARRAYS:
        assert np.array_equal(arr[k], arrays[k])


def test_validation(tmp_path):
    theta, sol, _, _ = product_instance(load("golden_soc.npz"))
    np.savez(tmp_path / "bad.npz", x=sol.x, y=sol.y, s=sol.s, extra=np.zeros(1))
    with pytest.raises(qg.ValidationError, match="unknown keys"):
        binio.load_solution(tmp_path / "bad.npz")
    binio.save_problem(tmp_path / "p.npz", theta)
    with np.load(tmp_path / "p.npz") as z:
        d = {k: z[k] for k in z.files}
    d["A.row_idx"] = d["A.row_idx"][::-1].copy()     # rows no longer increasing per column
    np.savez(tmp_path / "p2.npz", **d)
    with pytest.raises(qg.ValidationError):
        binio.load_problem(tmp_path / "p2.npz")
    d = {k: v for k, v in d.items() if k != "q"}
    np.savez(tmp_path / "p3.npz", **d)
    with pytest.raises(qg.ValidationError, match="missing keys"):
        binio.load_problem(tmp_path / "p3.npz")
