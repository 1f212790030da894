"""Per-LSMR-iteration device time of one config on the graph path, split
into the two step kernels (event-timed back to back, qg_time_kernel) and the
rest (finalizes, launch gaps): (t(K2) - t(K1)) / (K2 - K1) of fixed-cap
jvp and vjp solves, CUDA events around each solve.  Diagnostic only.

    python tools/iter_breakdown.py c2 [K1 K2]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_17522_b200 import QCPBatch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
K1 = int(sys.argv[2]) if len(sys.argv) > 2 else 50
K2 = int(sys.argv[3]) if len(sys.argv) > 3 else 150
bt, dirs, *_ = bench.build_workload(cfg, 0, 1, None)
dev = torch.device("cuda")
t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in bench.batch_bytes(bt).items()}
d = {k: torch.from_numpy(np.ascontiguousarray(getattr(dirs, k))).to(dev)
     for k in ("dP", "dA", "dq", "db", "dx", "dy", "ds")}
b = QCPBatch.from_device(bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks, t)


def solve_ms(which, K, reps=5):
    kw = dict(atol=0.0, btol=0.0, max_iter=K)
    fn = (lambda: b.jvp_device(d["dP"], d["dA"], d["dq"], d["db"], **kw)) if which == "jvp" else \
        (lambda: b.vjp_device(d["dx"], d["dy"], d["ds"], **kw))
    fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


f, ft = b.time_kernel(0, reps=50), b.time_kernel(1, reps=50)
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("QG_"))
for which in ("jvp", "vjp"):
    a1, a2 = solve_ms(which, K1), solve_ms(which, K2)
    it = (a2 - a1) / (K2 - K1) * 1e3
    loop = b.loop_time()[0 if which == "jvp" else 1]
    print(f"{cfg} [{env}] {which}: {it:.1f} us/iter (loop events: {loop / K2 * 1e3:.1f}) = F {f * 1e3:.1f} + "
          f"F' {ft * 1e3:.1f} + rest {it - (f + ft) * 1e3:.1f} us (solve K={K2}: {a2:.2f} ms, "
          f"resident={b.resident()}, layout={b.layout()})", flush=True)
