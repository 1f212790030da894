"""Small jvp + vjp workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): every golden cone kind (SOC, PSD, exp/pow and
their duals, zero, nonneg) through BOTH loop modes (the resident engine
k_engine -- TMA bulk copies, mbarrier, warp-0 finalize overlapping the
SpMV -- and the graph loop), the c1 shape, a SELL-forced c5a mini-batch
through both, and a CTA-per-row (MODE_WIDE) problem -- i.e. every
step-kernel variant, the PSD DMMA epilogue, both finalize kernels, the
engine, preparation and assembly.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_17522_b200 as qg  # noqa: E402
from fixtures import KINDS, load, product_instance  # noqa: E402
from paper_2508_17522_b200 import QCPBatch, synth  # noqa: E402

KEYS = ("P_colptr", "P_rowidx", "P_vals", "A_colptr", "A_rowidx", "A_vals", "q", "b", "x", "y", "s")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def batch_run(bt, dirs, K):
    b = QCPBatch.from_device(bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks, {k: dev(getattr(bt, k)) for k in KEYS})
    kw = dict(atol=0.0, btol=0.0, max_iter=K)
    b.jvp_device(dev(dirs.dP), dev(dirs.dA), dev(dirs.dq), dev(dirs.db), **kw)
    b.vjp_device(dev(dirs.dx), dev(dirs.dy), dev(dirs.ds), **kw)
    b.apply_F_device(dev(np.ones(sum(bt.n) + sum(bt.m) + bt.B)), transpose=True)
    torch.cuda.synchronize()
    b.close()


def main():
    for engine in ("1", "0"):
        os.environ["QG_ENGINE"] = engine
        for kind in KINDS:
            theta, sol, pert, delta = product_instance(load(f"golden_{kind}.npz"))
            q = qg.QCP(theta, sol)
            q.jvp(pert, max_iter=30)
            q.vjp(delta, max_iter=30)
            q.kkt()
            print("golden", kind, "engine" if q.resident() else "graph", "ok", flush=True)
            q.close()
    del os.environ["QG_ENGINE"]
    bt = synth.generate("c1", seed=1)
    batch_run(bt, synth.directions(bt, seed=2), 20)
    print("c1 ok", flush=True)
    bt = synth.generate("c5a", seed=3, batch=3)
    for engine in ("1", "0"):
        os.environ["QG_ENGINE"] = engine
        os.environ["QG_SELL"] = "1"
        batch_run(bt, synth.directions(bt, seed=4), 10)
        print("c5a SELL", "engine" if engine == "1" else "graph", "ok", flush=True)
    del os.environ["QG_SELL"], os.environ["QG_ENGINE"]
    # a dense-row problem: MODE_WIDE units (rows of >= 512 entries)
    bt = synth.custom([("zero", 40, 0, 0.0), ("nonneg", 40, 0, 0.0)], n=1200, nnzA=80 * 1100, seed=5)
    batch_run(bt, synth.directions(bt, seed=6), 10)
    print("wide ok", flush=True)


if __name__ == "__main__":
    main()
