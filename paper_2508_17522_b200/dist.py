"""Row-partitioned derivative of one large QCP over several GPUs
(configuration C5b).

A single problem too large for one GPU's bandwidth budget is split by the
rows of A: rank r holds rows [lo_r, hi_r) of A, b, y, s and the cone blocks
covering them (a zero / nonneg block may be cut anywhere -- its projection
is elementwise; every other block stays whole), plus the full X side
(P, q, x) and the T coordinate.  Every rank runs the same LSMR; the only
exchange is one sum-allreduce of the n-vector of A_r' partial products per
operator step (and of a few per-problem partial sums per finalize), issued
by the library on the compute stream (``NcclComm``: captured inside the
LSMR CUDA graphs).

Outputs per rank: dx, dq, dP replicated; dy, ds, db and dA (the entries of
the local rows, CSC order of the local A) local.  ``global_positions`` maps
the local dA entries into the CSC order of the whole A.

The reference is single-process (no counterpart); the partition follows
SURVEY §8(e).  Host-side shard construction is plain NumPy (data placement,
not the hot path) and is covered by CPU tests; the kernels are the batch
kernels of libqcpgrad with the X_PARTIAL / X_FINISH split.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from paper_2508_17522_b200 import _native as N

ELEMENTWISE = ("zero", "nonneg")


def _kind(b):
    return b[0] if isinstance(b, tuple) else b.kind


def _dim(b):
    return int(b[1]) if isinstance(b, tuple) else int(b.dim)


def allowed_cuts(m, blocks):
    """Boolean [m+1]: may a shard boundary sit before row i?"""
    total = sum(_dim(b) for b in blocks)
    if total != m:
        raise ValueError(f"cone blocks cover {total} rows, expected {m}")
    ok = np.zeros(m + 1, dtype=bool)
    ok[0] = ok[m] = True
    r = 0
    for b in blocks:
        d = _dim(b)
        if _kind(b) in ELEMENTWISE:
            ok[r:r + d + 1] = True
        else:
            ok[r] = ok[r + d] = True
        r += d
    if r != m:
        raise ValueError(f"cone blocks cover {r} rows, expected {m}")
    return ok


def row_cuts(m, blocks, row_weight, world):
    """Shard boundaries 0 = c_0 <= c_1 <= ... <= c_world = m at allowed rows,
    balanced by the cumulative ``row_weight`` (nnz of the row + 1)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    ok = allowed_cuts(m, blocks)
    cum = np.concatenate([[0.0], np.cumsum(np.asarray(row_weight, dtype=np.float64))])
    pos = np.flatnonzero(ok)
    cuts = [0]
    for k in range(1, world):
        target = cum[-1] * k / world
        i = int(np.searchsorted(cum[pos], target))
        cands = [pos[j] for j in (i - 1, i) if 0 <= j < len(pos)]
        best = min(cands, key=lambda c: (abs(cum[c] - target), c))
        cuts.append(max(int(best), cuts[-1]))
    cuts.append(m)
    return cuts


def shard_blocks(blocks, lo, hi):
    """The blocks covering rows [lo, hi) as (kind, dim, order, alpha) tuples;
    elementwise blocks are clipped to the range."""
    out, r = [], 0
    for b in blocks:
        t = b if isinstance(b, tuple) else (b.kind, b.dim, getattr(b, "order", 0) or 0, getattr(b, "alpha", 0.0) or 0.0)
        d = int(t[1])
        a, e = max(r, lo), min(r + d, hi)
        if a < e:
            if _kind(t) not in ELEMENTWISE and (a != r or e != r + d):
                raise ValueError(f"shard [{lo}, {hi}) cuts a {_kind(t)} block at rows [{r}, {r + d})")
            out.append((t[0], e - a, t[2], t[3]))
        r += d
    return out


def shard_csc_rows(n, colptr, rowidx, vals, lo, hi):
    """Rows [lo, hi) of a CSC matrix (renumbered from 0) and the CSC
    positions of the kept entries in the original."""
    colptr = np.asarray(colptr, dtype=np.int64)
    rowidx = np.asarray(rowidx, dtype=np.int64)
    keep = (rowidx >= lo) & (rowidx < hi)
    col = np.repeat(np.arange(n, dtype=np.int64), np.diff(colptr))
    counts = np.bincount(col[keep], minlength=n)
    cp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=cp[1:])
    return cp, rowidx[keep] - lo, np.asarray(vals)[keep], np.flatnonzero(keep)


@dataclass
class RowShard:
    """One rank's share of a single problem (host arrays, ``qg_batch_desc`` keys)."""

    rank: int
    world: int
    lo: int
    hi: int
    n: int
    m: int                    # local rows
    blocks: list              # (kind, dim, order, alpha)
    arrays: dict              # P_*, A_* (local rows), q, b, x, y, s
    global_positions: np.ndarray   # local dA entry -> CSC position in the whole A

    @property
    def P_nnz(self):
        return int(self.arrays["P_vals"].size)

    @property
    def A_nnz(self):
        return int(self.arrays["A_vals"].size)


def make_shard(problem, rank, world, cuts=None):
    """Rank ``rank``'s shard of ``problem``: a dict with n, m, blocks and the
    ``qg_batch_desc`` arrays of ONE problem (synth.Batch with B = 1 works)."""
    g = (lambda k: problem[k]) if isinstance(problem, dict) else (lambda k: getattr(problem, k))
    one = lambda v: int(v[0]) if isinstance(v, (list, tuple, np.ndarray)) else int(v)
    n, m = one(g("n")), one(g("m"))
    blocks = g("blocks")
    if blocks and isinstance(blocks[0], list):   # synth.Batch: one block list per problem
        blocks = blocks[0]
    rowidx = np.asarray(g("A_rowidx"), dtype=np.int64)
    if cuts is None:
        cuts = row_cuts(m, blocks, np.bincount(rowidx, minlength=m) + 1, world)
    lo, hi = cuts[rank], cuts[rank + 1]
    cp, ri, va, pos = shard_csc_rows(n, g("A_colptr"), rowidx, g("A_vals"), lo, hi)
    arrays = {k: np.asarray(g(k)) for k in ("P_colptr", "P_rowidx", "P_vals", "q", "x")}
    arrays.update(A_colptr=cp, A_rowidx=ri, A_vals=va)
    for k in ("b", "y", "s"):
        arrays[k] = np.asarray(g(k))[lo:hi]
    return RowShard(rank, world, lo, hi, n, hi - lo, shard_blocks(blocks, lo, hi), arrays, pos)


# ------------------------------------------------------------ communicator --
class Comm:
    """A ``qg_comm``: the sum-allreduce the partitioned handles use."""

    def __init__(self, ptr):
        self.ptr = ptr
        r, w = ctypes.c_int(), ctypes.c_int()
        N.check(N.lib().qg_comm_rank(ptr, ctypes.byref(r), ctypes.byref(w)))
        self.rank, self.world = r.value, w.value

    @classmethod
    def nccl(cls, group=None):
        """One rank per GPU over NCCL; the unique id travels over the
        initialised ``torch.distributed`` process group."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        buf = (ctypes.c_ubyte * 128)()
        if rank == 0:
            N.check(N.lib().qg_comm_nccl_id(buf))
        box = [bytes(buf) if rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = (ctypes.c_ubyte * 128).from_buffer_copy(box[0])
        p = N.c_vp()
        N.check(N.lib().qg_comm_create_nccl(ctypes.byref(p), uid, world, rank))
        return cls(p)

    @classmethod
    def local(cls, world):
        """``world`` shards on the current device, to be driven by one host
        thread each (tests and single-GPU runs of the partitioned path)."""
        arr = (N.c_vp * world)()
        N.check(N.lib().qg_comm_create_local(arr, world))
        return [cls(N.c_vp(arr[r])) for r in range(world)]

    def allreduce_(self, t):
        """In-place sum over ranks of a float64 CUDA tensor (synchronous)."""
        N.check(N.lib().qg_comm_allreduce(self.ptr, N.ptr(t), int(t.numel()), N.stream_ptr()))
        return t

    def close(self):
        if getattr(self, "ptr", None):
            N.lib().qg_comm_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def partitioned_batch(shard, comm, tensors=None):
    """The ``QCPBatch`` over ``shard`` on this rank (``comm.rank`` must be
    ``shard.rank``); ``tensors``: the shard's arrays already on the device."""
    import torch

    from paper_2508_17522_b200.solution_map import QCPBatch

    if comm.rank != shard.rank or comm.world != shard.world:
        raise ValueError("communicator rank / world do not match the shard")
    if tensors is None:
        tensors = {k: N.to_dev(v, torch.int64 if k.endswith(("colptr", "rowidx")) else torch.float64)
                   for k, v in shard.arrays.items()}
    b = QCPBatch.from_device([shard.n], [shard.m], [shard.P_nnz], [shard.A_nnz], [shard.blocks], tensors, comm=comm)
    b._keep_tensors = tensors
    return b
