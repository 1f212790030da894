"""Row-partitioned mode (dist.py) on one GPU.

The partitioned algorithm runs as `world` shards on the device, one host
thread each (LocalComm: host barrier + fixed-order sum kernel, no kernel
waits on another shard), and must reproduce the unpartitioned handle:
bit for bit at world 1 (the X_PARTIAL / X_FINISH split and the reduced
finalize keep every summation order), and to rounding at world 2..4 (only
the order of the A' partial sums changes).  A one-rank NCCL communicator
exercises ncclAllReduce recorded inside the LSMR graphs.
"""

import os
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2508_17522_b200 import QCPBatch, dist, synth  # noqa: E402

CONES = [("nonneg", 37, 0, 0.0), ("soc", 5, 0, 0.0), ("soc", 7, 0, 0.0), ("zero", 11, 0, 0.0),
         ("exp", 3, 0, 0.0), ("pow", 3, 0, 0.3), ("psd", 6, 3, 0.0), ("nonneg", 41, 0, 0.0),
         ("soc", 4, 0, 0.0), ("dexp", 3, 0, 0.0)]


def _problem(seed=21):
    bt = synth.custom(CONES, n=60, nnzA=700, seed=seed)
    dirs = synth.directions(bt, seed=seed + 1)
    return bt, dirs


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _single(bt, dirs, kw):
    keys = ("P_colptr", "P_rowidx", "P_vals", "A_colptr", "A_rowidx", "A_vals", "q", "b", "x", "y", "s")
    b = QCPBatch.from_device(bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks, {k: _dev(getattr(bt, k)) for k in keys})
    j = b.jvp_device(_dev(dirs.dP), _dev(dirs.dA), _dev(dirs.dq), _dev(dirs.db), **kw)
    v = b.vjp_device(_dev(dirs.dx), _dev(dirs.dy), _dev(dirs.ds), **kw)
    return [t.cpu().numpy() for t in j[:3]], [t.cpu().numpy() for t in v[:4]], j[3], v[4]


def _rank_run(shard, comm, dirs, kw, out, errs):
    try:
        with torch.cuda.stream(torch.cuda.Stream()):
            b = dist.partitioned_batch(shard, comm)
            lo, hi = shard.lo, shard.hi
            dA = _dev(dirs.dA[shard.global_positions])
            j = b.jvp_device(_dev(dirs.dP), dA, _dev(dirs.dq), _dev(dirs.db[lo:hi]), **kw)
            v = b.vjp_device(_dev(dirs.dx), _dev(dirs.dy[lo:hi]), _dev(dirs.ds[lo:hi]), **kw)
            torch.cuda.current_stream().synchronize()
            out[shard.rank] = ([t.cpu().numpy() for t in j[:3]], [t.cpu().numpy() for t in v[:4]], j[3], v[4])
            b.close()
    except Exception as e:  # surfaced by the main thread
        errs.append(e)


def _partitioned(bt, dirs, world, kw):
    comms = dist.Comm.local(world)
    shards = [dist.make_shard(bt, r, world) for r in range(world)]
    out, errs = [None] * world, []
    th = [threading.Thread(target=_rank_run, args=(shards[r], comms[r], dirs, kw, out, errs), daemon=True)
          for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    assert all(o is not None for o in out)
    for c in comms:
        c.close()
    # replicated outputs agree bit for bit across ranks
    for o in out[1:]:
        assert np.array_equal(o[0][0], out[0][0][0])                   # dx
        assert np.array_equal(o[1][0], out[0][1][0]) and np.array_equal(o[1][2], out[0][1][2])  # dP, dq
        assert o[2][0].iterations == out[0][2][0].iterations
    dx = out[0][0][0]
    dy = np.concatenate([o[0][1] for o in out])
    ds = np.concatenate([o[0][2] for o in out])
    dA = np.zeros(bt.A_vals.size)
    for s, o in zip(shards, out):
        dA[s.global_positions] = o[1][1]
    db = np.concatenate([o[1][3] for o in out])
    return [dx, dy, ds], [out[0][1][0], dA, out[0][1][2], db], out[0][2], out[0][3]


def _gap(a, b):
    return float(np.max(np.abs(a - b))) / (1.0 + float(np.max(np.abs(b)))) if b.size else 0.0


def test_shards_cover_and_balance():
    bt, _ = _problem()
    for world in (2, 3, 4):
        shards = [dist.make_shard(bt, r, world) for r in range(world)]
        assert shards[0].lo == 0 and shards[-1].hi == bt.m[0]
        assert all(a.hi == b.lo for a, b in zip(shards, shards[1:]))
        assert sum(s.A_nnz for s in shards) == bt.A_vals.size


def test_world1_bitwise():
    bt, dirs = _problem()
    kw = dict(atol=1e-12, btol=1e-12, max_iter=300)
    j0, v0, d0, _ = _single(bt, dirs, kw)
    j1, v1, d1, _ = _partitioned(bt, dirs, 1, kw)
    assert d0[0].iterations == d1[0].iterations
    for a, b in zip(j0 + v0, j1 + v1):
        assert np.array_equal(a, b)


def _apply_rank(shard, comm, w, out, errs):
    try:
        with torch.cuda.stream(torch.cuda.Stream()):
            b = dist.partitioned_batch(shard, comm)
            n = shard.n
            wl = np.concatenate([w[:n], w[n + shard.lo:n + shard.hi], w[-1:]])
            out[shard.rank] = [b.apply_F_device(_dev(wl), transpose=t).cpu().numpy() for t in (False, True)]
            b.close()
    except Exception as e:
        errs.append(e)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_partitioned_operator(world):
    """F w and F' w of the shards, reassembled, equal the whole problem's."""
    bt, _ = _problem()
    keys = ("P_colptr", "P_rowidx", "P_vals", "A_colptr", "A_rowidx", "A_vals", "q", "b", "x", "y", "s")
    one = QCPBatch.from_device(bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks, {k: _dev(getattr(bt, k)) for k in keys})
    n, m = bt.n[0], bt.m[0]
    w = np.random.default_rng(4).standard_normal(n + m + 1)
    ref = [one.apply_F_device(_dev(w), transpose=t).cpu().numpy() for t in (False, True)]
    comms = dist.Comm.local(world)
    shards = [dist.make_shard(bt, r, world) for r in range(world)]
    out, errs = [None] * world, []
    th = [threading.Thread(target=_apply_rank, args=(shards[r], comms[r], w, out, errs), daemon=True)
          for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    for k in range(2):
        got = np.concatenate([out[0][k][:n]] + [o[k][n:n + s.m] for o, s in zip(out, shards)] + [out[0][k][-1:]])
        assert _gap(got, ref[k]) <= 1e-13
        assert all(np.array_equal(o[k][:n], out[0][k][:n]) and o[k][-1] == out[0][k][-1] for o in out)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_partitioned_matches_single(world):
    bt, dirs = _problem()
    # fixed small cap: the iterates themselves must agree to rounding (larger
    # caps amplify rounding: F is rank-deficient, see test_gpu_fullsize.py)
    kw = dict(atol=0.0, btol=0.0, max_iter=2)
    j0, v0, _, _ = _single(bt, dirs, kw)
    j1, v1, _, _ = _partitioned(bt, dirs, world, kw)
    for a, b in zip(j1 + v1, j0 + v0):
        assert _gap(a, b) <= 1e-12
    # converged at a tight tolerance
    kw = dict(atol=1e-13, btol=1e-13, max_iter=2000)
    j0, v0, d0, e0 = _single(bt, dirs, kw)
    j1, v1, d1, e1 = _partitioned(bt, dirs, world, kw)
    assert d0[0].converged and d1[0].converged and e1[0].converged
    for a, b in zip(j1 + v1, j0 + v0):
        assert _gap(a, b) <= 1e-7


def test_nccl_one_rank_graphs():
    import torch.distributed as tdist

    if not tdist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        tdist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        bt, dirs = _problem(seed=33)
        kw = dict(atol=1e-12, btol=1e-12, max_iter=300)
        j0, v0, d0, _ = _single(bt, dirs, kw)
        comm = dist.Comm.nccl()
        shard = dist.make_shard(bt, 0, 1)
        b = dist.partitioned_batch(shard, comm)
        j = b.jvp_device(_dev(dirs.dP), _dev(dirs.dA), _dev(dirs.dq), _dev(dirs.db), **kw)
        v = b.vjp_device(_dev(dirs.dx), _dev(dirs.dy), _dev(dirs.ds), **kw)
        assert j[3][0].iterations == d0[0].iterations
        for a, ref in zip([t.cpu().numpy() for t in j[:3]] + [t.cpu().numpy() for t in v[:4]], j0 + v0):
            assert np.array_equal(a, ref)
        t = torch.arange(8, dtype=torch.float64, device="cuda")
        assert torch.equal(comm.allreduce_(t.clone()), t)
        b.close()
        comm.close()
    finally:
        tdist.destroy_process_group()
