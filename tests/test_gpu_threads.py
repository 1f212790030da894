"""Threading contract (reference SPEC: pure and thread-safe):
concurrent jvp / vjp calls from several host threads -- on one shared
handle (serialised by the handle) and on one handle per thread (truly
concurrent, each on its own stream) -- return exactly the serial results."""

import threading

import numpy as np
import pytest

from fixtures import load, product_instance

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
qg = pytest.importorskip("paper_2508_17522_b200")

KINDS = ("soc", "psd", "exp", "pow")


def _serial():
    out = {}
    for k in KINDS:
        theta, sol, pert, delta = product_instance(load(f"golden_{k}.npz"))
        q = qg.QCP(theta, sol)
        d, _ = q.jvp(pert)
        g, _ = q.vjp(delta)
        out[k] = (d.dx.copy(), d.dy.copy(), g.dA.values.copy(), g.dq.copy())
    return out


def _run_threads(fn, n):
    errs, th = [], []

    def wrap(i):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                fn(i)
        except Exception as e:  # surfaced below
            errs.append(e)

    for i in range(n):
        th.append(threading.Thread(target=wrap, args=(i,), daemon=True))
        th[-1].start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs


def test_handle_per_thread_concurrent():
    ref = _serial()
    got = {}

    def work(i):
        k = KINDS[i % len(KINDS)]
        theta, sol, pert, delta = product_instance(load(f"golden_{k}.npz"))
        q = qg.QCP(theta, sol)
        for _ in range(3):
            d, _ = q.jvp(pert)
            g, _ = q.vjp(delta)
        got[i] = (k, d.dx.copy(), d.dy.copy(), g.dA.values.copy(), g.dq.copy())

    _run_threads(work, 8)
    for k, *vals in got.values():
        for a, b in zip(vals, ref[k]):
            assert np.array_equal(a, b)


def test_shared_handle_concurrent():
    theta, sol, pert, delta = product_instance(load("golden_soc.npz"))
    q = qg.QCP(theta, sol)
    d0, _ = q.jvp(pert)
    g0, _ = q.vjp(delta)
    got = []

    def work(i):
        for _ in range(3):
            d, _ = q.jvp(pert) if i % 2 == 0 else (None, None)
            g, _ = q.vjp(delta) if i % 2 == 1 else (None, None)
            got.append((d.dx.copy() if d is not None else None, g.dq.copy() if g is not None else None))

    _run_threads(work, 6)
    assert len(got) == 18
    for dx, dq in got:
        if dx is not None:
            assert np.array_equal(dx, d0.dx)
        if dq is not None:
            assert np.array_equal(dq, g0.dq)
