"""Parity on the configurations and kernel variants the performance numbers
come from (BASELINE.json configs at their real sizes):

* the batched c5a handle of bench.py -- SELL-32 on BOTH sides
  (``layout()`` asserts it), including the X-side two-matrix SELL walk
  (P + A') -- on >= 128 problems, sampled problems against the oracle;
  and QG_SELL=1 forcing SELL on a small batch;
* full C3 (n=20k, m=40,002: 6,667 exp + 6,667 pow blocks): projections and
  D Pi per block, F w / F' w, fixed-cap jvp / vjp;
* full C5b (LASSO, nnz(A) = 5.0e7, the CTA-per-row MODE_WIDE units):
  F w / F' w, fixed-cap jvp / vjp; and its row-partitioned mode (LocalComm
  worlds 2..4) against the unpartitioned handle.

Tolerances (north star): P1 cone projections / D Pi / F w <= 1e-12
relative; P2 jvp / vjp <= 1e-6 at matched caps, compared only at caps where
the reference itself is stable under 1e-16 operator noise.
"""

import re
import threading

import numpy as np
import pytest

from fixtures import gap
from oracle import cones as C
from oracle import cpu_bench
from oracle import qcp as Q
from oracle_runs import OracleRuns

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2508_17522_b200 import QCPBatch, dist, synth  # noqa: E402

KEYS = ("P_colptr", "P_rowidx", "P_vals", "A_colptr", "A_rowidx", "A_vals", "q", "b", "x", "y", "s")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _batch(bt):
    return QCPBatch.from_device(bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks, {k: _dev(getattr(bt, k)) for k in KEYS})


def _run(b, dirs, K):
    kw = dict(atol=0.0, btol=0.0, max_iter=K)
    j = b.jvp_device(_dev(dirs.dP), _dev(dirs.dA), _dev(dirs.dq), _dev(dirs.db), **kw)
    v = b.vjp_device(_dev(dirs.dx), _dev(dirs.dy), _dev(dirs.ds), **kw)
    assert all(d.iterations == K for d in j[3]) and all(d.iterations == K for d in v[4])
    return [t.cpu().numpy() for t in j[:3]], [t.cpu().numpy() for t in v[:4]]


def _slices(bt, p):
    xo, yo = sum(bt.n[:p]), sum(bt.m[:p])
    po, ao = sum(bt.P_nnz[:p]), sum(bt.A_nnz[:p])
    return (slice(xo, xo + bt.n[p]), slice(yo, yo + bt.m[p]), slice(po, po + bt.P_nnz[p]),
            slice(ao, ao + bt.A_nnz[p]))


def _check_problems(bt, dirs, b, probs, caps):
    """F w / F' w of the whole batch at once, then fixed-cap jvp / vjp, for
    the sampled problems against the oracle."""
    NX, NY = sum(bt.n), sum(bt.m)
    rng = np.random.default_rng(0)
    w = rng.standard_normal(NX + NY + bt.B)
    Fw = [b.apply_F_device(_dev(w), transpose=t).cpu().numpy() for t in (False, True)]
    runs = {}
    for p in probs:
        th, sol, pert, de = cpu_bench.problem(bt, dirs, p)
        xs, ys, _, _ = _slices(bt, p)
        wp = np.concatenate([w[xs], w[NX + ys.start:NX + ys.stop], w[NX + NY + p:NX + NY + p + 1]])
        F = Q.make_F(th, Q.embed(sol))
        for k, ref in ((0, F.matvec(wp)), (1, F.rmatvec(wp))):
            got = np.concatenate([Fw[k][xs], Fw[k][NX + ys.start:NX + ys.stop], Fw[k][NX + NY + p:NX + NY + p + 1]])
            assert gap(got, ref) <= 1e-12, (p, k)                                   # P1
        runs[p] = OracleRuns(th, sol, pert, de).stable_caps(caps)
    checked = 0
    for K in caps:
        if not any(K in r for r in runs.values()):
            continue
        j, v = _run(b, dirs, K)
        for p in probs:
            if K not in runs[p]:
                continue
            xs, ys, ps, as_ = _slices(bt, p)
            mine_j = np.concatenate([j[0][xs], j[1][ys], j[2][ys]])
            mine_v = np.concatenate([v[0][ps], v[1][as_], v[2][xs], v[3][ys]])
            j0, v0 = runs[p][K]
            assert gap(mine_j, j0) <= 1e-6 and gap(mine_v, v0) <= 1e-6, (p, K)      # P2
            checked += 1
    assert checked >= len(probs)


def test_c5a_batched_sell_both_sides():
    """The bench's kernel variant: >= 128 c5a problems put both sides on SELL."""
    bt = synth.generate("c5a", seed=11, batch=128)
    dirs = synth.directions(bt, seed=12)
    b = _batch(bt)
    sx, sy = b.layout()
    assert sx > 0 and sy > 0, (sx, sy)
    _check_problems(bt, dirs, b, probs=(0, 37, 64, 127), caps=(5, 10, 20))


def test_c5a_forced_sell_small_batch(monkeypatch):
    monkeypatch.setenv("QG_SELL", "1")
    bt = synth.generate("c5a", seed=13, batch=6)
    dirs = synth.directions(bt, seed=14)
    b = _batch(bt)
    sx, sy = b.layout()
    assert sx > 0 and sy > 0
    _check_problems(bt, dirs, b, probs=(0, 5), caps=(5, 10, 20))
    monkeypatch.setenv("QG_SELL", "0")
    b0 = _batch(bt)
    assert b0.layout() == (0, 0)
    # SELL vs CSR: the operator to ulp level (different summation trees) ...
    w = _dev(np.random.default_rng(1).standard_normal(sum(bt.n) + sum(bt.m) + bt.B))
    for t in (False, True):
        assert gap(b.apply_F_device(w, transpose=t).cpu().numpy(),
                   b0.apply_F_device(w, transpose=t).cpu().numpy()) <= 1e-13
    # ... and fixed-cap jvp / vjp at the P2 bound (K=3 amplifies ulp
    # differences to ~1e-8 here: the reference's own cap sensitivity)
    j1, v1 = _run(b, dirs, 3)
    j0, v0 = _run(b0, dirs, 3)
    for a, c in zip(j1 + v1, j0 + v0):
        assert gap(a, c) <= 1e-6


@pytest.fixture(scope="module")
def c3():
    bt = synth.generate("c3", seed=3)
    return bt, synth.directions(bt, seed=4)


def test_c3_full_cones(c3):
    """Pi_K* and D Pi on every one of the 13,334 exp / pow blocks (root
    finders of cones.py:334-378, 559-618) <= 1e-12."""
    import paper_2508_17522_b200 as qg

    bt, _ = c3
    th, sol, _, _ = cpu_bench.problem(bt, synth.directions(bt, seed=4), 0)
    spec = qg.ConeSpec([qg.ConeBlock(k, alpha=a) if k in ("pow", "dpow") else qg.ConeBlock(k)
                        for (k, d, o, a) in bt.blocks[0]])
    mid = sol.y - sol.s
    rng = np.random.default_rng(5)
    for z in (mid, mid * (1.0 + 1e-6 * rng.standard_normal(mid.size))):
        for dual in (True, False):
            try:
                want = C.project(th.blocks, z, dual=dual)
            except C.BlockFailure as e:
                # Pi_K (primal, off the path) of these points: the reference
                # itself fails on block 2927 ("exponential cone projection
                # root-finding did not converge", checked against conegrad
                # 0.1.0) -- the GPU must fail the same way on the same block
                with pytest.raises(qg.NumericalError, match=re.escape(str(e))):
                    (qg.project_dual if dual else qg.project)(spec, z)
                continue
            got = (qg.project_dual if dual else qg.project)(spec, z)
            assert gap(got, want) <= 1e-12
        dz = rng.standard_normal(mid.size)
        got = qg.dprojection_dual(spec, z).matvec(dz)
        want = C.Derivative(th.blocks, z, dual=True).matvec(dz)
        assert gap(got, want) <= 1e-12


def test_c3_full_operator_and_caps(c3):
    bt, dirs = c3
    _check_problems(bt, dirs, _batch(bt), probs=(0,), caps=(5, 10, 20))


@pytest.fixture(scope="module")
def c5b():
    bt = synth.generate("c5b", seed=7)
    return bt, synth.directions(bt, seed=8)


def test_c5b_full_wide_rows(c5b):
    """LASSO, nnz(A) = 5.0e7: MODE_WIDE (CTA per dense row) on the GPU."""
    bt, dirs = c5b
    b = _batch(bt)
    _check_problems(bt, dirs, b, probs=(0,), caps=(2, 3, 5))


def _apply_rank(shard, comm, w, out, errs):
    try:
        with torch.cuda.stream(torch.cuda.Stream()):
            b = dist.partitioned_batch(shard, comm)
            n = shard.n
            wl = np.concatenate([w[:n], w[n + shard.lo:n + shard.hi], w[-1:]])
            out[shard.rank] = [b.apply_F_device(_dev(wl), transpose=t).cpu().numpy() for t in (False, True)]
            b.close()
    except Exception as e:  # surfaced by the main thread
        errs.append(e)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_c5b_row_partitioned_operator(c5b, world):
    """c5b's row-partitioned mode (dist.py) at full scale: the shards' F w /
    F' w, reassembled, equal the unpartitioned handle's (<= 1e-13)."""
    bt, _ = c5b
    n, m = bt.n[0], bt.m[0]
    w = np.random.default_rng(4).standard_normal(n + m + 1)
    one = _batch(bt)
    ref = [one.apply_F_device(_dev(w), transpose=t).cpu().numpy() for t in (False, True)]
    one.close()
    comms = dist.Comm.local(world)
    shards = [dist.make_shard(bt, r, world) for r in range(world)]
    out, errs = [None] * world, []
    th = [threading.Thread(target=_apply_rank, args=(shards[r], comms[r], w, out, errs), daemon=True)
          for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in comms:
        c.close()
    assert not errs, errs
    for k in range(2):
        got = np.concatenate([out[0][k][:n]] + [o[k][n:n + s.m] for o, s in zip(out, shards)] + [out[0][k][-1:]])
        assert gap(got, ref[k]) <= 1e-13


def _c4_small(seed):
    """c4's cone mix at 1/8 of its PSD blocks: nonneg + 64 x PSD(32), Gram P."""
    cones = [("nonneg", 1250, 0, 0)] + [("psd", 528, 32, 0)] * 64
    return synth.custom(cones, n=2500, nnzA=250_000, seed=seed, diag_P=False)


def test_psd_split_kernel_matches_inline_path(monkeypatch):
    """c4-shaped PSD handle: the F' step's PSD units as their own 256-thread
    kernel (k_step_psd, default) against the same units inside k_step
    (QG_PSD_SPLIT=0).  Same per-entry expressions and product tiles: the X
    and Y outputs are bit-identical; the T entry (partial sums in another
    order) agrees to ulp level; fixed-cap jvp / vjp at the P2 bound."""
    bt = _c4_small(seed=5)
    dirs = synth.directions(bt, seed=6)
    monkeypatch.setenv("QG_PSD_SPLIT", "1")
    b1 = _batch(bt)
    monkeypatch.setenv("QG_PSD_SPLIT", "0")
    b0 = _batch(bt)
    NE = sum(bt.n) + sum(bt.m) + bt.B
    w = _dev(np.random.default_rng(2).standard_normal(NE))
    for t in (False, True):
        o1 = b1.apply_F_device(w, transpose=t).cpu().numpy()
        o0 = b0.apply_F_device(w, transpose=t).cpu().numpy()
        assert np.array_equal(o1[:NE - bt.B], o0[:NE - bt.B]), t
        assert gap(o1, o0) <= 1e-13
    j1, v1 = _run(b1, dirs, 3)
    j0, v0 = _run(b0, dirs, 3)
    for a, c in zip(j1 + v1, j0 + v0):
        assert gap(a, c) <= 1e-6


@pytest.mark.parametrize("cfg", ["c4", "c5a"])
def test_graph_path_bit_deterministic(monkeypatch, cfg):
    """Repeated fixed-cap solves on the graph path (SELL units with dynamic
    slice claims, the split PSD kernel) are bit-identical."""
    monkeypatch.setenv("QG_ENGINE", "0")
    monkeypatch.setenv("QG_SELL", "1")
    bt = _c4_small(seed=7) if cfg == "c4" else synth.generate(cfg, seed=7, batch=8)
    dirs = synth.directions(bt, seed=8)
    b = _batch(bt)
    r1 = _run(b, dirs, 20)
    r2 = _run(b, dirs, 20)
    for a, c in zip(r1[0] + r1[1], r2[0] + r2[1]):
        assert np.array_equal(a, c)
