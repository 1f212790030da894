"""c4 PSD diagnostics: the F / F' step times of the c4 handle (QG_PSD_PROF
phase cycles when set) and the isolated D Pi application of the c4 cone
table (k_dpi_apply: 512 PSD(32) blocks + nonneg(10000)), event-timed.

    python tools/psd_probe.py [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2508_17522_b200 import QCPBatch, cones  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
bt, dirs, *_ = bench.build_workload("c4", 0, 1, None)
t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in bench.batch_bytes(bt).items()}
b = QCPBatch.from_device(bt.n, bt.m, bt.P_nnz, bt.A_nnz, bt.blocks, t)
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("QG_"))
for _ in range(2):
    f, ft = (b.time_kernel(w, reps=reps) for w in (0, 1))
    print(f"c4 [{env}] F {f * 1e3:.1f} us | F' {ft * 1e3:.1f} us", flush=True)

spec = cones.ConeSpec([cones.ConeBlock.nonneg(10000)] + [cones.ConeBlock.psd(32)] * 512)
m = sum(blk.dim for blk in spec.blocks)
rng = np.random.default_rng(0)
z = rng.standard_normal(m)
D = cones.ConeDerivative(spec, z, dual=True)
dz = torch.from_numpy(rng.standard_normal(m)).cuda()
for _ in range(3):
    D.matvec_device(dz)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(reps):
    e0.record()
    D.matvec_device(dz)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"isolated D Pi apply (c4 cone table): median {np.median(ts) * 1e3:.1f} us, min {min(ts) * 1e3:.1f} us",
      flush=True)
