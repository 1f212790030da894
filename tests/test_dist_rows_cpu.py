"""Host logic of the row-partitioned mode (dist.py) on CPU:
shard boundaries (never inside a SOC / PSD / exp / pow block, anywhere in
zero / nonneg blocks, balanced by nnz), exact reconstruction of A from the
row shards, and the exchange identity the kernels rely on -- the sum over
ranks of A_r' w_r is A' w -- through a real gloo allreduce at world 2."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from oracle import qcp as Q
from paper_2508_17522_b200 import dist, synth

CONES = [("nonneg", 37, 0, 0.0), ("soc", 5, 0, 0.0), ("soc", 7, 0, 0.0), ("zero", 11, 0, 0.0),
         ("exp", 3, 0, 0.0), ("pow", 3, 0, 0.3), ("psd", 6, 3, 0.0), ("nonneg", 41, 0, 0.0),
         ("soc", 4, 0, 0.0), ("dexp", 3, 0, 0.0)]


def _problem(seed=21):
    return synth.custom(CONES, n=60, nnzA=700, seed=seed)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_allowed_cuts():
    blocks = [("nonneg", 3, 0, 0.0), ("soc", 4, 0, 0.0), ("zero", 2, 0, 0.0), ("psd", 3, 2, 0.0)]
    ok = dist.allowed_cuts(12, blocks)
    assert ok.tolist() == [True, True, True, True, False, False, False, True, True, True, False, False, True]
    with pytest.raises(ValueError):
        dist.allowed_cuts(11, blocks)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shards_reconstruct(world):
    bt = _problem()
    n, m = bt.n[0], bt.m[0]
    shards = [dist.make_shard(bt, r, world) for r in range(world)]
    assert shards[0].lo == 0 and shards[-1].hi == m
    assert all(a.hi == b.lo for a, b in zip(shards, shards[1:]))
    ok = dist.allowed_cuts(m, bt.blocks[0])
    assert all(ok[s.lo] for s in shards)
    # blocks: concatenation re-covers the rows; no non-elementwise block split
    assert sum(sum(b[1] for b in s.blocks) for s in shards) == m
    assert all(sum(b[1] for b in s.blocks) == s.m for s in shards)
    # A: every entry lands in exactly one shard, values and order preserved
    pos = np.concatenate([s.global_positions for s in shards])
    assert np.array_equal(np.sort(pos), np.arange(bt.A_vals.size))
    dense = np.zeros((m, n))
    for s in shards:
        cp, ri, va = s.arrays["A_colptr"], s.arrays["A_rowidx"], s.arrays["A_vals"]
        assert np.all(np.diff(cp) >= 0) and cp[-1] == va.size
        col = np.repeat(np.arange(n), np.diff(cp))
        dense[s.lo + ri, col] = va
        assert np.array_equal(va, bt.A_vals[s.global_positions])
        assert np.array_equal(s.arrays["b"], bt.b[s.lo:s.hi])
    ref = np.zeros((m, n))
    ref[bt.A_rowidx, np.repeat(np.arange(n), np.diff(bt.A_colptr))] = bt.A_vals
    assert np.array_equal(dense, ref)


def test_balance_on_elementwise_rows():
    # a LASSO-like cone list (two elementwise blocks) splits into near-equal nnz
    bt = synth.custom([("zero", 400, 0, 0.0), ("nonneg", 400, 0, 0.0)], n=300, nnzA=20000, seed=3)
    world = 4
    nnz = [dist.make_shard(bt, r, world).A_nnz for r in range(world)]
    assert max(nnz) - min(nnz) <= 0.05 * sum(nnz) / world + 40


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    bt = _problem(seed=5)   # every rank builds the same problem, keeps its rows
    s = dist.make_shard(bt, rank, world)
    n = s.n
    A_r = Q.Csc(s.m, n, s.arrays["A_colptr"], s.arrays["A_rowidx"], s.arrays["A_vals"])
    rng = np.random.default_rng(9)
    w = rng.standard_normal(bt.m[0])
    x = rng.standard_normal(n)
    part = torch.from_numpy(np.array(Q.spmv_t(A_r, w[s.lo:s.hi])))
    tdist.all_reduce(part)                    # the X_PARTIAL -> X_FINISH exchange
    A = Q.Csc(bt.m[0], n, bt.A_colptr, bt.A_rowidx, bt.A_vals)
    out[rank] = (float(np.max(np.abs(part.numpy() - Q.spmv_t(A, w)))),
                 float(np.max(np.abs(Q.spmv(A_r, x) - Q.spmv(A, x)[s.lo:s.hi]))) if s.m else 0.0,
                 s.lo, s.hi)
    tdist.barrier()
    tdist.destroy_process_group()


def test_exchange_identity_gloo_world2():
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    (e0, f0, lo0, hi0), (e1, f1, lo1, hi1) = out[0], out[1]
    assert lo0 == 0 and hi0 == lo1 and hi1 == _problem(seed=5).m[0]
    assert e0 <= 1e-12 and e1 <= 1e-12 and f0 == 0.0 and f1 == 0.0
