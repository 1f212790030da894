"""One c5a-style batch through the resident engine (jvp + vjp at K=100):
the target of ncu captures of k_engine.

    python tools/engine_probe.py [--config c5a] [--batch 4096] [--iters 100]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5a")
ap.add_argument("--batch", type=int, default=4096)
ap.add_argument("--iters", type=int, default=100)
ap.add_argument("--reps", type=int, default=1)
args = ap.parse_args()

import torch  # noqa: E402

from paper_2508_17522_b200 import QCPBatch, synth  # noqa: E402

KEYS = ("P_colptr", "P_rowidx", "P_vals", "A_colptr", "A_rowidx", "A_vals", "q", "b", "x", "y", "s")
bt = synth.generate(args.config, seed=1000, batch=args.batch) if args.config != "c5b" else synth.generate("c5b", seed=1000)
dirs = synth.directions(bt, seed=2000)
dev = {k: torch.from_numpy(np.ascontiguousarray(getattr(bt, k))).cuda() for k in KEYS}
dd = {k: torch.from_numpy(np.ascontiguousarray(getattr(dirs, k))).cuda() for k in ("dP", "dA", "dq", "db", "dx", "dy", "ds")}
kw = dict(atol=0.0, btol=0.0, max_iter=args.iters)
b = QCPBatch.from_device(bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks, dev)
for _ in range(args.reps):
    j = b.jvp_device(dd["dP"], dd["dA"], dd["dq"], dd["db"], **kw)
    v = b.vjp_device(dd["dx"], dd["dy"], dd["ds"], **kw)
torch.cuda.synchronize()
print("resident", b.resident(), "loop ms (jvp, vjp)", b.loop_time(), "layout", b.layout())
