"""Dry run of bench.py's multi-rank plumbing on CPU (gloo, world 2): the
c5b row-shard branch (bench.row_shard over a small LASSO-shaped problem)
covers every row of A exactly once with whole cone blocks, the shards'
directions are the matching slices, and the max / sum over ranks that
bench.py uses for device time and problem counts agree on every rank.
(The NCCL launch itself needs GPUs: bench.py --gpus N under torchrun.)"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as tdist
import torch.multiprocessing as mp

import bench
from paper_2508_17522_b200 import synth


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = synth.custom([("zero", 40, 0, 0.0), ("nonneg", 50, 0, 0.0)], n=30, nnzA=900, seed=5)
        dirs = synth.directions(full, seed=6)
        bt, d = bench.row_shard(full, dirs, rank, world)
        s = bt.shard
        mx = bench.max_over_ranks(tdist, float(rank + 1))
        tot = bench.sum_over_ranks(tdist, float(bt.m[0]))
        out[rank] = dict(lo=s.lo, hi=s.hi, m=bt.m[0], nnz=bt.A_nnz[0], db=d.db.copy(), mx=mx, tot=tot,
                         rows=bt.A_rowidx.copy(), vals=bt.A_vals.copy(), pos=s.global_positions.copy())
    finally:
        tdist.destroy_process_group()


def test_bench_row_shard_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    full = synth.custom([("zero", 40, 0, 0.0), ("nonneg", 50, 0, 0.0)], n=30, nnzA=900, seed=5)
    dirs = synth.directions(full, seed=6)
    r0, r1 = out[0], out[1]
    assert r0["lo"] == 0 and r0["hi"] == r1["lo"] and r1["hi"] == full.m[0]
    assert r0["m"] + r1["m"] == full.m[0] and r0["nnz"] + r1["nnz"] == full.A_nnz[0]
    assert r0["mx"] == r1["mx"] == 2.0 and r0["tot"] == r1["tot"] == full.m[0]
    np.testing.assert_array_equal(np.concatenate([r0["db"], r1["db"]]), dirs.db)
    # every entry of A lands on exactly one rank, with its value
    pos = np.concatenate([r0["pos"], r1["pos"]])
    assert np.array_equal(np.sort(pos), np.arange(full.A_nnz[0]))
    vals = np.concatenate([r0["vals"], r1["vals"]])
    np.testing.assert_array_equal(vals, full.A_vals[pos])
