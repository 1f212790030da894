"""The PyTorch autograd binding (torch_layer.py): reverse mode equals the
batched vjp, forward mode equals the batched jvp, bit for bit (same kernels,
same order), and the chain rule composes with ordinary torch ops."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2508_17522_b200 import QCPBatch, synth  # noqa: E402
from paper_2508_17522_b200.torch_layer import QCPStructure, qcp_solution  # noqa: E402

CONES = [("zero", 4, 0, 0.0), ("nonneg", 10, 0, 0.0), ("soc", 5, 0, 0.0), ("exp", 3, 0, 0.0),
         ("pow", 3, 0, 0.4), ("psd", 6, 3, 0.0)]
OPTS = dict(atol=1e-12, btol=1e-12, max_iter=400)


def _setup(seed=3, batch=3):
    bt = synth.custom(CONES, n=24, nnzA=120, seed=seed, batch=batch)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    st = QCPStructure(bt.P_colptr, bt.P_rowidx, bt.A_colptr, bt.A_rowidx, bt.n, bt.m, bt.blocks, **OPTS)
    data = {k: dev(getattr(bt, k)) for k in ("P_vals", "A_vals", "q", "b", "x", "y", "s")}
    return bt, st, data


def _batch(bt, data):
    t = {k: torch.from_numpy(np.ascontiguousarray(getattr(bt, k))).cuda()
         for k in ("P_colptr", "P_rowidx", "A_colptr", "A_rowidx")}
    t.update(data)
    return QCPBatch.from_device(bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks, t)


def test_structure_nnz():
    bt, st, _ = _setup()
    assert st.P_nnz == list(bt.P_nnz) and st.A_nnz == list(bt.A_nnz)


def test_backward_is_vjp():
    bt, st, data = _setup()
    leaves = {k: data[k].clone().requires_grad_(True) for k in ("P_vals", "A_vals", "q", "b")}
    x, y, s = qcp_solution(st, leaves["P_vals"], leaves["A_vals"], leaves["q"], leaves["b"],
                           data["x"], data["y"], data["s"])
    assert torch.equal(x, data["x"]) and torch.equal(s, data["s"])
    g = torch.Generator(device="cuda").manual_seed(7)
    wx, wy, ws = (torch.randn(t.shape, generator=g, device="cuda", dtype=torch.float64) for t in (x, y, s))
    ((wx * x).sum() + (wy * y).sum() + (ws * s).sum()).backward()
    dP, dA, dq, db, _ = _batch(bt, data).vjp_device(wx, wy, ws, **OPTS)
    assert torch.equal(leaves["P_vals"].grad, dP) and torch.equal(leaves["A_vals"].grad, dA)
    assert torch.equal(leaves["q"].grad, dq) and torch.equal(leaves["b"].grad, db)


def test_backward_chain_rule_and_missing_grads():
    bt, st, data = _setup(seed=5)
    q = data["q"].clone().requires_grad_(True)
    x, _, _ = qcp_solution(st, data["P_vals"], data["A_vals"], q, data["b"], data["x"], data["y"], data["s"])
    (0.5 * (x * x).sum()).backward()  # y, s unused: their cotangents are zero
    z = lambda t: torch.zeros_like(t)
    _, _, dq, _, _ = _batch(bt, data).vjp_device(data["x"].clone(), z(data["y"]), z(data["s"]), **OPTS)
    assert torch.equal(q.grad, dq)


def test_forward_mode_is_jvp():
    import torch.autograd.forward_ad as fwAD

    bt, st, data = _setup(seed=9)
    dirs = synth.directions(bt, seed=11)
    tan = {k: torch.from_numpy(np.ascontiguousarray(getattr(dirs, k))).cuda() for k in ("dP", "dA", "dq", "db")}
    with fwAD.dual_level():
        P = fwAD.make_dual(data["P_vals"], tan["dP"])
        A = fwAD.make_dual(data["A_vals"], tan["dA"])
        qd = fwAD.make_dual(data["q"], tan["dq"])
        bd = fwAD.make_dual(data["b"], tan["db"])
        x, y, s = qcp_solution(st, P, A, qd, bd, data["x"], data["y"], data["s"])
        tx, ty, ts = (fwAD.unpack_dual(t).tangent for t in (x, y, s))
    dx, dy, ds, _ = _batch(bt, data).jvp_device(tan["dP"], tan["dA"], tan["dq"], tan["db"], **OPTS)
    assert torch.equal(tx, dx) and torch.equal(ty, dy) and torch.equal(ts, ds)


def test_adjoint_identity_through_autograd():
    """<w, J v> == <J' w, v> within the LSMR tolerance, both through torch."""
    import torch.autograd.forward_ad as fwAD

    bt, st, data = _setup(seed=13)
    dirs = synth.directions(bt, seed=17)
    v = {k: torch.from_numpy(np.ascontiguousarray(getattr(dirs, k))).cuda() for k in ("dP", "dA", "dq", "db")}
    w = {k: torch.from_numpy(np.ascontiguousarray(getattr(dirs, k))).cuda() for k in ("dx", "dy", "ds")}
    with fwAD.dual_level():
        duals = [fwAD.make_dual(data[k], v[t]) for k, t in
                 (("P_vals", "dP"), ("A_vals", "dA"), ("q", "dq"), ("b", "db"))]
        outs = qcp_solution(st, *duals, data["x"], data["y"], data["s"])
        jv = [fwAD.unpack_dual(t).tangent for t in outs]
    lhs = sum(float((a * b).sum()) for a, b in zip((w["dx"], w["dy"], w["ds"]), jv))
    leaves = [data[k].clone().requires_grad_(True) for k in ("P_vals", "A_vals", "q", "b")]
    outs = qcp_solution(st, *leaves, data["x"], data["y"], data["s"])
    sum((a * b).sum() for a, b in zip((w["dx"], w["dy"], w["ds"]), outs)).backward()
    rhs = sum(float((l.grad * v[t]).sum()) for l, t in zip(leaves, ("dP", "dA", "dq", "db")))
    assert abs(lhs - rhs) <= 1e-6 * (1.0 + abs(lhs))
