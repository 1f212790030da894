"""Multi-process (gloo, world size 2) coverage of the N>1 host logic of
bench.py: batch sharding into disjoint contiguous ranges, and the
max-over-ranks device-time / sum-over-ranks reductions.  The data path has
no collective (independent problems), so nothing else crosses ranks."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, _ = bench.dist_env()
    assert (r, w) == (rank, world)
    lo, hi = bench.shard_range(10, rank, world)
    # each rank owns its shard; timing is max-reduced, counts sum-reduced
    t = bench.max_over_ranks(dist, float(rank + 1))
    n = bench.sum_over_ranks(dist, float(hi - lo))
    bt, dirs, total, here, scaling = bench.build_workload("c5a", rank, world, batch_override=6, strong=True)
    wk = bench.build_workload("c5a", rank, world, batch_override=3)
    out[rank] = (lo, hi, t, n, total, here, scaling, bt.B, float(bt.x[0]), (wk[2], wk[3], wk[4], wk[0].B))
    dist.barrier()
    dist.destroy_process_group()


def test_sharding_and_reductions_world2():
    world = 2
    port = _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    (lo0, hi0, t0, n0, tot0, h0, sc0, b0, x0, w0), (lo1, hi1, t1, n1, tot1, h1, sc1, b1, x1, w1) = out[0], out[1]
    assert (lo0, hi0, lo1, hi1) == (0, 5, 5, 10)          # disjoint, contiguous, covering
    assert t0 == t1 == 2.0                                  # max over ranks
    assert n0 == n1 == 10.0                                 # every problem counted once
    assert tot0 == tot1 == 6 and h0 + h1 == 6 and b0 + b1 == 6   # --strong: one batch sharded
    assert sc0 == sc1 == "strong"
    assert x0 != x1                                         # ranks build different problems
    # default (weak): every rank its own batch of 3, 6 evaluated in total
    assert w0 == w1 == (6, 3, "weak", 3)


def test_shard_range_balanced():
    for total in (1, 7, 4096):
        for world in (1, 2, 4, 8):
            ranges = [bench.shard_range(total, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [h - l for l, h in ranges]
            assert max(sizes) - min(sizes) <= 1
