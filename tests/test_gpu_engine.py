"""The problem-resident LSMR engine (csrc/engine.cu): which batches take it,
and parity with the oracle and with the 4-launch graph loop.

Small problems (<= 16k stored entries per operator side) and large batches
(>= 296 problems) run every solve problem-resident by default, so the
golden / recipe / edge-case suites already exercise the engine; these tests
pin the choice, the bench workload (c5a at >= 296 problems), large SOC
blocks (warp path), exp / pow blocks (3x3 path), convergence (stop tests)
and cap-0 / zero-rhs edges -- each against the oracle and the graph loop
(QG_ENGINE=0) on the same inputs.
"""

import numpy as np
import pytest

from fixtures import gap, synth_instance
from oracle import qcp as Q
from oracle_runs import OracleRuns

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2508_17522_b200 as qg  # noqa: E402
from paper_2508_17522_b200 import QCPBatch, synth  # noqa: E402
from test_gpu_configs_full import _batch, _check_problems, _dev, _run  # noqa: E402


def test_engine_choice(monkeypatch):
    bt = synth.generate("c5a", seed=21, batch=300)
    assert _batch(bt).resident()                       # large batch of small problems
    bt8 = synth.generate("c5a", seed=21, batch=8)
    assert not _batch(bt8).resident()                  # 8 x 31k entries: the graph loop fills the GPU better
    monkeypatch.setenv("QG_ENGINE", "1")
    assert _batch(bt8).resident()
    monkeypatch.setenv("QG_ENGINE", "0")
    bt1 = synth.generate("c5a", seed=21, batch=1)
    assert not _batch(bt1).resident()
    monkeypatch.setenv("QG_ENGINE", "1")              # PSD blocks: never resident, even when asked
    _, prod = synth_instance(([("nonneg", 5, 0, 0.0), ("psd", 6, 3, 0.0)], 8, 40), seed=3)
    assert not qg.QCP(*prod[:2]).resident()
    monkeypatch.delenv("QG_ENGINE")
    _, prod = synth_instance("c1", seed=3)             # one tiny problem: resident by default
    assert qg.QCP(*prod[:2]).resident()


def test_c5a_resident_batch_vs_oracle():
    """The bench's path: a c5a batch of 300 (resident by default), sampled
    problems against the oracle at stable caps; F w through the same handle."""
    bt = synth.generate("c5a", seed=22, batch=300)
    dirs = synth.directions(bt, seed=23)
    b = _batch(bt)
    assert b.resident()
    _check_problems(bt, dirs, b, probs=(0, 151, 299), caps=(5, 10, 20))


def _engine_vs_graph(monkeypatch, bt, dirs, kw, bound):
    monkeypatch.setenv("QG_ENGINE", "1")
    be = _batch(bt)
    assert be.resident()
    monkeypatch.setenv("QG_ENGINE", "0")
    bg = _batch(bt)
    assert not bg.resident()
    outs, diags = [], []
    for b in (be, bg):
        j = b.jvp_device(_dev(dirs.dP), _dev(dirs.dA), _dev(dirs.dq), _dev(dirs.db), **kw)
        v = b.vjp_device(_dev(dirs.dx), _dev(dirs.dy), _dev(dirs.ds), **kw)
        outs.append([t.cpu().numpy() for t in j[:3]] + [t.cpu().numpy() for t in v[:4]])
        diags.append((j[3], v[4]))
    for a, c in zip(*outs):
        assert gap(a, c) <= bound
    for de, dg in zip(*diags):
        for x, y in zip(de, dg):
            # long tolerance-driven solves: the reference itself moves its stop by
            # ~1% under 1e-16 operator noise (c5a at tol 1e-12: 1402..1420)
            assert abs(x.iterations - y.iterations) <= max(3, 0.02 * y.iterations)
            assert x.converged == y.converged
    return diags[0]


def test_engine_vs_graph_fixed_cap(monkeypatch):
    """Same fixed cap through both loops, at a cap where the reference
    itself is stable under 1e-16 operator noise (at unstable
    caps any two summation orders legitimately differ by far more)."""
    from oracle import cpu_bench

    bt = synth.generate("c5a", seed=24, batch=2)
    dirs = synth.directions(bt, seed=25)
    stable = set.intersection(*(set(OracleRuns(*cpu_bench.problem(bt, dirs, p)).stable_caps((5, 8, 10, 20)))
                                for p in range(bt.B)))
    assert stable, "no common stable cap"
    K = min(stable)
    dj, dv = _engine_vs_graph(monkeypatch, bt, dirs, dict(atol=0.0, btol=0.0, max_iter=K), 1e-6)
    assert all(d.iterations == K for d in dj) and all(d.iterations == K for d in dv)


def test_engine_vs_graph_converged(monkeypatch):
    """Tolerance-driven stop (lsmr.py:173-182) inside the resident loop."""
    bt = synth.generate("c5a", seed=26, batch=4)
    dirs = synth.directions(bt, seed=27)
    dj, dv = _engine_vs_graph(monkeypatch, bt, dirs, dict(atol=1e-12, btol=1e-12), 1e-6)
    assert all(d.converged for d in dj) and all(d.converged for d in dv)


def test_engine_cap_zero_and_zero_rhs(monkeypatch):
    monkeypatch.setenv("QG_ENGINE", "1")
    bt = synth.generate("c5a", seed=28, batch=3)
    dirs = synth.directions(bt, seed=29)
    b = _batch(bt)
    assert b.resident()
    j = b.jvp_device(_dev(dirs.dP), _dev(dirs.dA), _dev(dirs.dq), _dev(dirs.db), max_iter=0)
    assert all(d.iterations == 0 for d in j[3])
    z = lambda a: _dev(np.zeros_like(a))
    j = b.jvp_device(z(dirs.dP), z(dirs.dA), z(dirs.dq), z(dirs.db))
    assert all(d.iterations == 0 and d.converged for d in j[3])
    assert all(float(t.abs().max()) == 0.0 for t in j[:3])


@pytest.mark.parametrize("blocks", [
    [("nonneg", 40, 0, 0.0), ("soc", 70, 0, 0.0), ("soc", 45, 0, 0.0)],          # SOC > 32: warp path
    [("zero", 6, 0, 0.0)] + [("exp", 3, 0, 0.0)] * 12 + [("pow", 3, 0, 0.3)] * 12 + [("dexp", 3, 0, 0.0)] * 4,
])
def test_engine_cone_paths_vs_oracle(monkeypatch, blocks):
    monkeypatch.setenv("QG_ENGINE", "1")
    ora, prod = synth_instance((blocks, 60, 2500), seed=5, diag_P=False)
    th, sol, pert, de = ora
    theta, psol, ppert, pde = prod
    q = qg.QCP(theta, psol)
    assert q.resident()
    runs = OracleRuns(th, sol, pert, de).stable_caps((3, 5, 8, 12))
    assert runs, "no stable cap"
    for K, (jo, vo) in runs.items():
        dl, dg = q.jvp(ppert, atol=0.0, btol=0.0, max_iter=K)
        g, vg = q.vjp(pde, atol=0.0, btol=0.0, max_iter=K)
        assert dg.iterations == K and vg.iterations == K
        assert gap(np.concatenate([dl.dx, dl.dy, dl.ds]), jo) <= 1e-6
        assert gap(np.concatenate([g.dP.values, g.dA.values, g.dq, g.db]), vo) <= 1e-6
    # converged at a matched tight tolerance
    dl, dg = q.jvp(ppert, atol=1e-13, btol=1e-13)
    ol, og, _ = Q.jvp(th, sol, pert, atol=1e-13, btol=1e-13)
    assert dg.converged and abs(dg.iterations - og.iterations) <= max(3, og.iterations // 20)
    assert max(gap(dl.dx, ol.dx), gap(dl.dy, ol.dy), gap(dl.ds, ol.ds)) <= 1e-6


def test_engine_deterministic(monkeypatch):
    monkeypatch.setenv("QG_ENGINE", "1")
    bt = synth.generate("c5a", seed=30, batch=5)
    dirs = synth.directions(bt, seed=31)
    b = _batch(bt)
    r1 = _run(b, dirs, 7)
    r2 = _run(b, dirs, 7)
    for a, c in zip(r1[0] + r1[1], r2[0] + r2[1]):
        assert np.array_equal(a, c)


@pytest.mark.parametrize("kw", [dict(atol=0.0, btol=0.0, max_iter=10), dict(atol=1e-12, btol=1e-12),
                                dict(atol=0.0, btol=0.0, max_iter=3)])
def test_device_terminated_graph_loop_matches_host_loop(monkeypatch, kw):
    """The graph loop's conditional WHILE node (k_loop_cond re-arms it while a
    problem is active and the cap is not reached) runs the same kernels in
    the same order as the host-polled chunk loop: bit-identical outputs and
    iteration counts, including caps that are not a multiple of its chunk."""
    monkeypatch.setenv("QG_ENGINE", "0")
    bt = synth.generate("c5a", seed=32, batch=3)
    dirs = synth.directions(bt, seed=33)
    res = []
    for host in ("0", "1"):
        monkeypatch.setenv("QG_HOST_LOOP", host)
        b = _batch(bt)
        assert not b.resident()
        j = b.jvp_device(_dev(dirs.dP), _dev(dirs.dA), _dev(dirs.dq), _dev(dirs.db), **kw)
        v = b.vjp_device(_dev(dirs.dx), _dev(dirs.dy), _dev(dirs.ds), **kw)
        res.append(([t.cpu().numpy() for t in j[:3]] + [t.cpu().numpy() for t in v[:4]],
                    [d.iterations for d in j[3]] + [d.iterations for d in v[4]]))
    for a, c in zip(res[0][0], res[1][0]):
        assert np.array_equal(a, c)
    assert res[0][1] == res[1][1]
