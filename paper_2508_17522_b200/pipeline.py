"""Host-buffer batch evaluation with copy / compute overlap.

``evaluate_host`` is the end-to-end entry for a batch that lives in (pinned)
host memory: problem data, solutions and directions in, jvp and vjp outputs
out.  The batch is cut into ``chunks`` contiguous problem ranges; chunk k+1's
host-to-device copies and chunk k-1's device-to-host copies run on two copy
streams (one per copy engine) while chunk k's preparation + jvp + vjp run on
the compute stream, so
PCIe time hides behind the kernels instead of adding to them.

Problems are independent, so per-problem results equal a whole-batch call up
to rounding (the work-unit partition, and with it the order of the partial
sums, depends on the batch size).

The next chunk's upload is issued after the current chunk's preparation
(whose small row-pointer / unit-table copies would otherwise queue behind
it in the copy engine), and the LSMR setup does no host-to-device copy (the
caps are computed on the device), so the uploads overlap only kernels.
Round 1 issued the upload first and measured 324 / 324 / 353 / 406 ms at
1 / 2 / 4 / 8 chunks vs 307 ms for the whole-batch path.
"""

import numpy as np

from paper_2508_17522_b200.solution_map import QCPBatch

_DATA = ("P_colptr", "P_rowidx", "P_vals", "A_colptr", "A_rowidx", "A_vals", "q", "b", "x", "y", "s")


def _offsets(n, m, P_nnz, A_nnz):
    cs = lambda v: np.concatenate([[0], np.cumsum(np.asarray(v, dtype=np.int64))])
    n, m = np.asarray(n, np.int64), np.asarray(m, np.int64)
    return dict(n=cs(n), m=cs(m), pc=cs(n + 1), pn=cs(P_nnz), an=cs(A_nnz))


def _ranges(o, lo, hi):
    """slice of each concatenated array for problems [lo, hi)."""
    return dict(P_colptr=(o["pc"][lo], o["pc"][hi]), A_colptr=(o["pc"][lo], o["pc"][hi]),
                P_rowidx=(o["pn"][lo], o["pn"][hi]), P_vals=(o["pn"][lo], o["pn"][hi]),
                A_rowidx=(o["an"][lo], o["an"][hi]), A_vals=(o["an"][lo], o["an"][hi]),
                q=(o["n"][lo], o["n"][hi]), x=(o["n"][lo], o["n"][hi]),
                b=(o["m"][lo], o["m"][hi]), y=(o["m"][lo], o["m"][hi]), s=(o["m"][lo], o["m"][hi]),
                dP=(o["pn"][lo], o["pn"][hi]), dA=(o["an"][lo], o["an"][hi]),
                dq=(o["n"][lo], o["n"][hi]), db=(o["m"][lo], o["m"][hi]),
                dx=(o["n"][lo], o["n"][hi]), dy=(o["m"][lo], o["m"][hi]), ds=(o["m"][lo], o["m"][hi]))


def chunk_bounds(B, chunks):
    """Problem ranges of the pipeline: a short first chunk (1/16 of the
    batch, >= 148 problems: one per SM of the resident engine) so the one
    upload nothing can hide behind is short, then equal chunks.  The first
    chunk's kernels cover the second chunk's upload when the rest is cut into
    chunks - 1 pieces of <= ~5x its size."""
    chunks = max(int(chunks), 1)
    if chunks == 1 or B < 2 * 148:
        edges = [B * c // chunks for c in range(chunks + 1)]
    else:
        first = max(148, B // 16)
        rest = B - first
        edges = [0] + [first + rest * c // (chunks - 1) for c in range(chunks)]
    return [e for i, e in enumerate(edges) if i == 0 or e > edges[i - 1]]


def evaluate_host(n, m, P_nnz, A_nnz, blocks, data, dirs, *, chunks=4, atol=1e-10, btol=1e-10, max_iter=None,
                  out=None):
    """jvp and vjp of every problem of a host batch.

    data: ``qg_batch_desc`` arrays (torch CPU tensors, ideally pinned);
    dirs: dP, dA, dq, db (jvp directions) and dx, dy, ds (vjp cotangents),
    concatenated like the data.  Returns a dict of host tensors
    (dx, dy, ds from jvp; gP, gA, gq, gb from vjp), reusing ``out`` when given,
    and the per-problem diagnostics lists (jvp, vjp)."""
    import torch

    B = len(n)
    o = _offsets(n, m, P_nnz, A_nnz)
    shapes = dict(dx=o["n"][-1], dy=o["m"][-1], ds=o["m"][-1], gP=o["pn"][-1], gA=o["an"][-1],
                  gq=o["n"][-1], gb=o["m"][-1])
    if out is None:
        out = {k: torch.empty(int(v), dtype=torch.float64, pin_memory=True) for k, v in shapes.items()}
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream()   # host -> device
    down = torch.cuda.Stream()   # device -> host (the other copy engine: runs beside the uploads)
    bounds = chunk_bounds(B, chunks)
    f64, i64 = torch.float64, torch.int64
    kw = dict(atol=atol, btol=btol, max_iter=max_iter)

    # Device buffers are allocated on the compute stream and only written by
    # the copy stream (ordered by events); device results are kept referenced
    # until the copy stream has drained, so the caching allocator never needs
    # cross-stream bookkeeping.
    def upload(lo, hi):
        r = _ranges(o, lo, hi)
        t = {}
        for k in _DATA + ("dP", "dA", "dq", "db", "dx", "dy", "ds"):
            a, b = (int(v) for v in r[k])
            t[k] = torch.empty(b - a, dtype=i64 if k.endswith(("colptr", "rowidx")) else f64, device="cuda")
        copy.wait_stream(comp)  # buffers' previous users on the compute stream are done
        with torch.cuda.stream(copy):
            for k, dst in t.items():
                a, b = (int(v) for v in r[k])
                dst.copy_((data if k in _DATA else dirs)[k][a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
        return t, ev

    diags_j, diags_v, keep = [], [], []
    pending = upload(bounds[0], bounds[1])
    for c in range(len(bounds) - 1):
        lo, hi = bounds[c], bounds[c + 1]
        t, ev = pending
        comp.wait_event(ev)
        b = QCPBatch.from_device(n[lo:hi], m[lo:hi], P_nnz[lo:hi], A_nnz[lo:hi], blocks[lo:hi],
                                 {k: t[k] for k in _DATA})
        # the next chunk's H2D starts only now, overlapping this chunk's
        # jvp / vjp kernels: the preparation's own small copies (row
        # pointers, unit tables) must not queue behind it in the copy engine
        if c + 2 < len(bounds):
            pending = upload(bounds[c + 1], bounds[c + 2])
        dx, dy, ds, dj = b.jvp_device(t["dP"], t["dA"], t["dq"], t["db"], **kw)
        gP, gA, gq, gb, dv = b.vjp_device(t["dx"], t["dy"], t["ds"], **kw)
        b.close()
        diags_j += dj
        diags_v += dv
        r = _ranges(o, lo, hi)
        res = dict(dx=(dx, "dx"), dy=(dy, "dy"), ds=(ds, "ds"), gP=(gP, "dP"), gA=(gA, "dA"), gq=(gq, "dq"),
                   gb=(gb, "db"))
        down.wait_stream(comp)
        with torch.cuda.stream(down):
            for k, (v, rk) in res.items():
                a, e = (int(x) for x in r[rk])
                out[k][a:e].copy_(v[:e - a], non_blocking=True)
        keep.append((t, res))
    copy.synchronize()
    down.synchronize()
    comp.synchronize()
    del keep
    return out, diags_j, diags_v
