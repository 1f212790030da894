"""Wall time of the host-buffer paths on c5a (diagnostic): whole-batch
from_host + jvp_host + vjp_host vs pipeline.evaluate_host at several chunk
counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_17522_b200 import QCPBatch  # noqa: E402
from paper_2508_17522_b200.pipeline import evaluate_host  # noqa: E402

bt, dirs, *_ = bench.build_workload("c5a", 0, 1, None)
kw = dict(atol=0.0, btol=0.0, max_iter=100)
sizes = (bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks)
pin = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in bench.batch_bytes(bt).items()}
pdir = {k: torch.from_numpy(np.ascontiguousarray(getattr(dirs, k))).pin_memory()
        for k in ("dP", "dA", "dq", "db", "dx", "dy", "ds")}


def whole():
    b = QCPBatch.from_host(*sizes, pin)
    b.jvp_host(pdir["dP"], pdir["dA"], pdir["dq"], pdir["db"], **kw)
    b.vjp_host(pdir["dx"], pdir["dy"], pdir["ds"], **kw)
    b.close()


def tm(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t) / reps


print(f"whole-batch host path {tm(whole):.1f} ms", flush=True)
for c in (1, 2, 4, 8):
    out = [None]

    def pip():
        out[0] = evaluate_host(*sizes, pin, pdir, chunks=c, out=out[0][0] if out[0] else None, **kw)
    print(f"pipeline chunks={c} {tm(pip):.1f} ms", flush=True)
