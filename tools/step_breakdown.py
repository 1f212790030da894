"""Wall-clock breakdown of one bench step (create / jvp / vjp), first call
vs repeated calls on the same handle.  Diagnostic only."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2508_17522_b200 import synth, QCPBatch
import bench

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5a"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
bt, dirs, *_ = bench.build_workload(cfg, 0, 1, B)
dev = torch.device("cuda")
blocks = bt.blocks
t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in bench.batch_bytes(bt).items()}
d = {k: torch.from_numpy(np.ascontiguousarray(getattr(dirs, k))).to(dev) for k in ("dP", "dA", "dq", "db", "dx", "dy", "ds")}
kw = dict(atol=0.0, btol=0.0, max_iter=100)
def tm(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize(); return r, 1e3 * (time.perf_counter() - t0)
for rep in range(3):
    b, tc = tm(lambda: QCPBatch.from_device(bt.n, bt.m, bt.P_nnz, bt.A_nnz, blocks, t))
    _, tj = tm(lambda: b.jvp_device(d["dP"], d["dA"], d["dq"], d["db"], **kw))
    _, tj2 = tm(lambda: b.jvp_device(d["dP"], d["dA"], d["dq"], d["db"], **kw))
    _, tv = tm(lambda: b.vjp_device(d["dx"], d["dy"], d["ds"], **kw))
    _, tv2 = tm(lambda: b.vjp_device(d["dx"], d["dy"], d["ds"], **kw))
    print(f"create {tc:8.1f} ms  jvp {tj:8.1f} / again {tj2:8.1f}  vjp {tv:8.1f} / again {tv2:8.1f}", flush=True)
    b.close()
print("F ms", b.time_kernel(0) if False else "")
