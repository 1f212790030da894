"""pipeline.evaluate_host: chunked host-buffer evaluation with overlapped
copies equals one whole-batch device call (to rounding: the work-unit
partition depends on the batch size)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2508_17522_b200 import QCPBatch, synth  # noqa: E402
from paper_2508_17522_b200.pipeline import evaluate_host  # noqa: E402

KEYS = ("P_colptr", "P_rowidx", "P_vals", "A_colptr", "A_rowidx", "A_vals", "q", "b", "x", "y", "s")


def _gap(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b))) / (1.0 + float(np.max(np.abs(b)))) if b.size else 0.0


@pytest.mark.parametrize("chunks", [1, 3, 7])
def test_pipeline_matches_whole_batch(chunks):
    bt = synth.custom([("nonneg", 9, 0, 0.0), ("soc", 5, 0, 0.0), ("exp", 3, 0, 0.0), ("psd", 3, 2, 0.0)],
                      n=12, nnzA=90, seed=4, batch=7)
    dirs = synth.directions(bt, seed=5)
    host = {k: torch.from_numpy(np.ascontiguousarray(getattr(bt, k))).pin_memory() for k in KEYS}
    hdir = {k: torch.from_numpy(np.ascontiguousarray(getattr(dirs, k))).pin_memory()
            for k in ("dP", "dA", "dq", "db", "dx", "dy", "ds")}
    sizes = (bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks)
    whole = QCPBatch.from_device(*sizes, {k: v.cuda() for k, v in host.items()})
    d = {k: v.cuda() for k, v in hdir.items()}
    for kw, tol in ((dict(atol=0.0, btol=0.0, max_iter=2), 1e-12), (dict(atol=1e-12, btol=1e-12, max_iter=500), 1e-8)):
        jx, jy, js, _ = whole.jvp_device(d["dP"], d["dA"], d["dq"], d["db"], **kw)
        gP, gA, gq, gb, _ = whole.vjp_device(d["dx"], d["dy"], d["ds"], **kw)
        out, dj, dv = evaluate_host(*sizes, host, hdir, chunks=chunks, **kw)
        assert len(dj) == len(dv) == bt.B
        for k, ref in (("dx", jx), ("dy", jy), ("ds", js), ("gP", gP), ("gA", gA), ("gq", gq), ("gb", gb)):
            assert _gap(out[k].numpy(), ref.cpu().numpy()) <= tol, k
