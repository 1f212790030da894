"""Event-timed F / F' / update kernel times and achieved GB/s for one config
(diagnostic; run several times under different QG_* environment settings).

    python tools/kernel_times.py [config] [batch] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_17522_b200 import QCPBatch  # noqa: E402
from paper_2508_17522_b200 import _native as N  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5a"
B = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
bt, dirs, *_ = bench.build_workload(cfg, 0, 1, B)
t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in bench.batch_bytes(bt).items()}
b = QCPBatch.from_device(bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks, t)
ab = bench.alg_bytes(bt)
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("QG_"))
for _ in range(2):
    f, ft, up = (b.time_kernel(w, reps=reps) for w in (0, 1, 2))
    lay = b.layout() if hasattr(N.lib(), "qg_handle_layout") else "?"
    print(f"{cfg} [{env}] layout={lay} F {f:.4f} ms {ab['F'] / f / 1e6:.0f} GB/s | "
          f"F' {ft:.4f} ms {ab['FT'] / ft / 1e6:.0f} GB/s | update {up:.4f} ms", flush=True)
