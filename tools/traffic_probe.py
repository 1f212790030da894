"""Target of bench.py's in-run DRAM-traffic capture: builds the bench's own
workload (same generator, seeds and batch) and runs the hot path once, so
that `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum` filtered to
the dominant kernel measures that kernel's traffic per launch in the same
run as the timing.  Not a benchmark (prints nothing of interest).

    python tools/traffic_probe.py --config c5a [--batch 4096] [--iters 100] [--which engine|ft]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5a")
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--iters", type=int, default=100)
ap.add_argument("--which", default="engine", choices=["engine", "ft", "f", "fin"])
args = ap.parse_args()

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_17522_b200 import QCPBatch  # noqa: E402

bt, dirs, *_ = bench.build_workload(args.config, 0, 1, args.batch)
dev = torch.device("cuda")
t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in bench.batch_bytes(bt).items()}
d = {k: torch.from_numpy(np.ascontiguousarray(getattr(dirs, k))).to(dev) for k in ("dP", "dA", "dq", "db")}
b = QCPBatch.from_device(bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks, t)
if args.which in ("engine", "fin"):
    b.jvp_device(d["dP"], d["dA"], d["dq"], d["db"], atol=0.0, btol=0.0, max_iter=args.iters)
else:
    b.time_kernel(1 if args.which == "ft" else 0, reps=1)
torch.cuda.synchronize()
