"""Per-stage wall time of QCPBatch creation (QG_TRACE) for one config."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if "notrace" not in sys.argv:  # `notrace`: total wall time only (the trace points synchronise the stream)
    os.environ["QG_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_17522_b200 import QCPBatch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5a"
bt, dirs, *_ = bench.build_workload(cfg, 0, 1, None)
t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in bench.batch_bytes(bt).items()}
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b = QCPBatch.from_device(bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks, t)
    torch.cuda.synchronize()
    print(f"--- create {i}: {1e3 * (time.perf_counter() - t0):.2f} ms", file=sys.stderr, flush=True)
    b.close()
