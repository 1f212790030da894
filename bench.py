#!/usr/bin/env python
"""Benchmark: jvp+vjp evaluations per second of the QCP solution-map
derivative (BASELINE.json metric) on B200, beside the CPU reference path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5a] [--impl ours|reference]

One *step* = one evaluation of the whole workload: prepare the batch
(``QCPBatch``: CSC->CSR transposes, Pi_K*(z), D Pi preparation), then one
jvp and one vjp of every problem, LSMR at a fixed cap of K=100 iterations
(atol=btol=0) -- the matched-work protocol of BASELINE.md.  ``value`` is
evals/s with inputs resident in HBM; ``e2e`` is the same through the
host-buffer API (H2D of the problem data and directions, D2H of all
outputs inside the timed region).

Default workload (``--config c5a``): BASELINE configs[4], a batch of 4096
independent QCPs (n=1000, m=1500 = nonneg(500) + 100 x SOC(10), nnz(A) =
1.5e4 each) per rank: weak scaling, N ranks evaluate N independent batches
with no data-path collective (``--strong`` shards one batch instead).
``--config c5b`` at N > 1 splits the ONE LASSO problem by the rows of A
over the ranks (dist.py; strong scaling; one NCCL sum-allreduce of the A'
partials per operator step, inside the LSMR graphs).  The other
single-problem configs (c1..c4) run as replicas at N > 1.

Multi-GPU: launched by torch.distributed.run, one rank per GPU; device
timing max-reduced over ranks (the batch path has no data-path collective).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": "n=100, m=150, zero(30)+nonneg(120), nnz(A)~1.6e3 (recipe-conditioned, diagonal P)",
    "c2": "n=2000, m=4000, 500 x SOC(8), nnz(A)~1e5, P = I + sparse Gram",
    "c3": "n=20000, m=40002, 6667 x exp + 6667 x pow(0.5), nnz(A)~1e6, P = I + sparse Gram",
    "c4": "n=20000, m=280336, 512 x PSD(32) + nonneg(10000), nnz(A)~2e6, P = I + sparse Gram",
    "c5a": "batch of 4096 QCPs, each n=1000, m=1500 = nonneg(500) + 100 x SOC(10), nnz(A)=1.5e4, diagonal P",
    "c5b": "LASSO canonical form, n=m=20000, nnz(A)~5.0e7 (dense 10000 x 5000 features)",
}
BATCH = {"c5a": 4096}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5a", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--lsmr-iters", type=int, default=100)
    ap.add_argument("--batch", type=int, default=None, help="override the c5a batch size (per rank)")
    ap.add_argument("--strong", action="store_true", help="c5a: shard ONE batch over the ranks (strong scaling)")
    ap.add_argument("--row-shards", action="store_true",
                    help="c5b: the row-partitioned NCCL path even at N=1 (exercises it on one GPU)")
    ap.add_argument("--cpu-sample", type=int, default=None, help="problems in the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=4, help="batch configs: chunks of the host-buffer pipeline")
    return ap.parse_args()


# ------------------------------------------------------------ distributed --
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_dist(world, local, backend):
    import torch
    import torch.distributed as dist

    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            # communicator setup lines (ranks, transport, NVLS) in the log: the
            # evidence that all N ranks formed one NCCL communicator
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return dist if world > 1 else None


def max_over_ranks(dist, value, device=None):
    if dist is None:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(dist, value, device=None):
    if dist is None:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# -------------------------------------------------------------- workload --
def shard_range(total, rank, world):
    """Contiguous, balanced problem range of ``rank``."""
    return rank * total // world, (rank + 1) * total // world


def build_workload(cfg, rank, world, batch_override=None, strong=False, force_rows=False):
    """This rank's share of the workload (synthetic, seeded per rank).

    Batches of independent problems (c5a) scale WEAK by default: every rank
    evaluates its own batch of BATCH[cfg] problems (the per-GPU work of the
    N=1 line), so N ranks evaluate N times as many problems -- the tier rule
    for a path that partitions into independent objects.  ``strong`` shards
    one fixed batch over the ranks instead (``--strong``)."""
    from paper_2508_17522_b200 import synth

    if cfg in BATCH:
        per = batch_override or BATCH[cfg]
        if strong:
            lo, hi = shard_range(per, rank, world)
            bt = synth.generate(cfg, seed=1000 + rank, batch=hi - lo)
            return bt, synth.directions(bt, seed=2000 + rank), per, hi - lo, "strong"
        bt = synth.generate(cfg, seed=1000 + rank, batch=per)
        return bt, synth.directions(bt, seed=2000 + rank), per * world, per, "weak"
    if cfg in PARTITIONED and (world > 1 or force_rows):
        # one problem, rows of A split over the ranks; every
        # rank builds the same instance and keeps its rows
        full = synth.generate(cfg, seed=1000)
        bt, dirs = row_shard(full, synth.directions(full, seed=2000), rank, world)
        return bt, dirs, 1, 1, "strong"
    bt = synth.generate(cfg, seed=1000 + rank)
    return bt, synth.directions(bt, seed=2000 + rank), world, 1, "weak"


PARTITIONED = ("c5b",)   # single problems run row-partitioned at N > 1 (others: replicas)


def row_shard(full, dirs, rank, world):
    """This rank's row shard of a single-problem synth.Batch (and of its
    directions) as a synth.Batch of the local problem; ``.shard`` keeps the
    partition (dist.RowShard)."""
    from paper_2508_17522_b200 import dist, synth

    s = dist.make_shard(full, rank, world)
    a = s.arrays
    bt = synth.Batch(n=[s.n], m=[s.m], blocks=[s.blocks], P_colptr=a["P_colptr"], P_rowidx=a["P_rowidx"],
                     P_vals=a["P_vals"], A_colptr=a["A_colptr"], A_rowidx=a["A_rowidx"], A_vals=a["A_vals"],
                     q=a["q"], b=a["b"], x=a["x"], y=a["y"], s=a["s"], P_nnz=[s.P_nnz], A_nnz=[s.A_nnz])
    bt.shard = s
    d = synth.Directions(dP=dirs.dP, dA=dirs.dA[s.global_positions], dq=dirs.dq, db=dirs.db[s.lo:s.hi],
                         dx=dirs.dx, dy=dirs.dy[s.lo:s.hi], ds=dirs.ds[s.lo:s.hi])
    return bt, d


def batch_bytes(bt):
    keys = ("P_colptr", "P_rowidx", "P_vals", "A_colptr", "A_rowidx", "A_vals", "q", "b", "x", "y", "s")
    return {k: getattr(bt, k) for k in keys}


def alg_bytes(bt):
    """Algorithmic bytes per launch of the two fused operator kernels
    (DESIGN.md 'Roofline'): every stored entry read once (8 B value + 4 B
    index), row pointers once, each vector stream once, D Pi parameters
    twice in the F' step."""
    NX, NY = sum(bt.n), sum(bt.m)
    nnzP, nnzA = int(bt.P_vals.size), int(bt.A_vals.size)
    mats = 12 * (nnzP + 2 * nnzA) + 4 * (2 * NX + NY)
    vec = 40 * (NX + NY)
    nsoc = ntri = 0
    psd = 0
    for blocks in bt.blocks:
        for (k, d, o, a) in blocks:
            if k == "soc":
                nsoc += 1
            elif k == "psd":
                psd += 16 * o * o
            elif k in ("exp", "dexp", "pow", "dpow"):
                ntri += 1
    s_dpi = 8 * NY + 12 * nsoc + 76 * ntri + psd
    # PSD D Pi apply = V'WV, Hadamard with B, V S V': 4 dense d x d x d products
    # (2 d^3 flops each); the F' step applies it twice per block
    psd_flops = sum(2 * 4 * 2 * o ** 3 for blocks in bt.blocks for (k, d, o, a) in blocks if k == "psd")
    return {"F": mats + vec, "FT": mats + vec + 8 * NY + 2 * s_dpi, "FT_psd_flops": psd_flops}


# ---------------------------------------------------------------- clocks --
class Clocks:
    def __init__(self, device_index):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{device_index}.csv")
        self.idx = device_index

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait(timeout=5)
            self.f.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def flush_l2(buf):
    buf.add_(1.0)


# ------------------------------------------------------------- our arm ----
def run_ours(args):
    import torch

    rank, world, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    torch.cuda.set_device(local)
    dist = init_dist(world, local, "nccl")
    dev = torch.device("cuda", local)
    from paper_2508_17522_b200 import _native as N
    from paper_2508_17522_b200 import QCPBatch

    bt, dirs, units_total, units_here, scaling = build_workload(args.config, rank, world, args.batch, args.strong,
                                                                args.row_shards)
    K = args.lsmr_iters
    kw = dict(atol=0.0, btol=0.0, max_iter=K)
    blocks = bt.blocks  # (kind, dim, order, alpha) per block; shared list objects convert once
    host = batch_bytes(bt)
    dev_in = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in host.items()}
    ddir = {k: torch.from_numpy(np.ascontiguousarray(getattr(dirs, k))).to(dev)
            for k in ("dP", "dA", "dq", "db", "dx", "dy", "ds")}
    sizes = (bt.n, bt.m, bt.P_nnz, bt.A_nnz, blocks)
    flush = torch.empty(256 * 2 ** 20 // 8, dtype=torch.float64, device=dev)
    comm = None
    if getattr(bt, "shard", None) is not None:
        import torch.distributed as tdist

        from paper_2508_17522_b200 import dist as qdist

        if not tdist.is_initialized():  # --row-shards at N=1: a one-rank NCCL group
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            tdist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        comm = qdist.Comm.nccl()   # the row-partitioned exchange (NCCL inside the LSMR graphs)

    last_diags = {}

    def step_device():
        b = QCPBatch.from_device(*sizes, dev_in, comm=comm)
        last_diags["jvp"] = b.jvp_device(ddir["dP"], ddir["dA"], ddir["dq"], ddir["db"], **kw)[-1]
        last_diags["vjp"] = b.vjp_device(ddir["dx"], ddir["dy"], ddir["ds"], **kw)[-1]
        return b

    def timed(fn, steps):
        total = 0.0
        for _ in range(steps):
            flush_l2(flush)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            total += e0.elapsed_time(e1)
        return total

    for _ in range(args.warmup):
        step_device()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = N.kernel_launches()
    with Clocks(local) as clk:
        ms = timed(step_device, args.steps)
    launches = (N.kernel_launches() - l0) // max(args.steps, 1)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = max_over_ranks(dist, ms, dev)
    ms_per_step = ms / args.steps
    value = units_total / (ms_per_step / 1e3)
    # the fixed cap must really run K iterations for every problem (with
    # atol=btol=0 the machine-precision stop tests can still end a solve
    # early, which would inflate evals/s): checked on the last timed step
    its = {k: [int(d.iterations) for d in v] for k, v in last_diags.items()}
    its_summary = {k: {"min": min(v), "mean": round(sum(v) / len(v), 2), "max": max(v)} for k, v in its.items()}
    if any(i != K for v in its.values() for i in v):
        print(f"bench.py: WARNING: not every LSMR solve ran K={K} iterations: {its_summary}", file=sys.stderr)

    # end to end through the host-buffer API: H2D of data + directions, D2H of outputs
    e2e = None
    if not args.no_e2e:
        pin = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in host.items()}
        pdir = {k: torch.from_numpy(np.ascontiguousarray(getattr(dirs, k))).pin_memory()
                for k in ("dP", "dA", "dq", "db", "dx", "dy", "ds")}
        outs = {}

        # host buffers in, host results out: the batch in `e2e_chunks` chunks
        # through pipeline.evaluate_host (chunk k+1's upload and chunk k-1's
        # download overlap chunk k's kernels) or, at 1 chunk / row shards, the
        # whole-batch from_host + jvp_host + vjp_host path
        from paper_2508_17522_b200.pipeline import evaluate_host

        chunks = args.e2e_chunks if (args.config in BATCH and comm is None) else 1
        pout = {}

        def step_host():
            if chunks > 1:
                pout["o"] = evaluate_host(*sizes, pin, pdir, chunks=chunks, out=pout.get("o", (None,))[0], **kw)
                return
            outs.clear()  # release last step's pinned result buffers back to torch's host cache
            b = QCPBatch.from_host(*sizes, pin, comm=comm)
            outs["j"] = b.jvp_host(pdir["dP"], pdir["dA"], pdir["dq"], pdir["db"], **kw)
            outs["v"] = b.vjp_host(pdir["dx"], pdir["dy"], pdir["ds"], **kw)
            b.close()

        step_host()
        if dist:
            dist.barrier()
        ems = max_over_ranks(dist, timed(step_host, max(1, min(args.steps, 3))), dev) / max(1, min(args.steps, 3))
        h2d = sum(v.numel() * v.element_size() for v in pin.values()) + sum(
            v.numel() * v.element_size() for v in pdir.values())
        d2h = 8 * (sum(bt.n) * 2 + sum(bt.m) * 3 + bt.P_vals.size + bt.A_vals.size)
        e2e = {"value": units_total / (ems / 1e3), "unit": "evals/s", "h2d_bytes_per_step": int(h2d * world),
               "d2h_bytes_per_step": int(d2h * world), "ms_per_step": ems,
               "api": (f"pipeline.evaluate_host, {chunks} chunks (pinned host buffers; copies overlap kernels)"
                       if chunks > 1 else "QCPBatch.from_host + jvp_host + vjp_host (pinned host buffers)")}

    # roofline of the fused kernels (CUDA events inside the library, same stream)
    b = step_device()
    ab = alg_bytes(bt)
    t_ft = b.time_kernel(1, reps=20)
    t_f = b.time_kernel(0, reps=20)
    peaks = _peaks()
    ach = ab["FT"] / (t_ft / 1e3) / 1e9
    sx, sy = b.layout()
    spmv = "SELL-32" if sx and sy else ("SELL-32/CSR" if sx or sy else "CSR per-unit lanes / CTA-per-row")
    steps_roof = {"kernel": f"k_step<FT> ({spmv} SpMV A,A',P + D Pi x2 epilogue)", "bound": "hbm",
                  "achieved": round(ach, 1), "peak": peaks[0], "peak_source": peaks[1], "unit": "GB/s",
                  "frac": round(ach / peaks[0], 4),
                  **_traffic_fields(_traffic(args.config, ab["FT"], "k_step", args.batch)
                                    if world == 1 and not b.resident() else None),
                  "alg_bytes_per_launch": ab["FT"], "launch_ms": round(t_ft, 4),
                  "f_step": {"achieved": round(ab["F"] / (t_f / 1e3) / 1e9, 1), "launch_ms": round(t_f, 4),
                             "alg_bytes_per_launch": ab["F"]}}
    if b.resident():
        # the LSMR loop runs as ONE problem-resident kernel per solve (k_engine):
        # its algorithmic bytes are the same per-iteration figure (B_F + B_F'),
        # times the iterations run, over the loop's device time (CUDA events in
        # the library on the call's stream, the timed steps' last jvp / vjp)
        lj, lv = b.loop_time()
        iters = {k: sum(v) for k, v in its.items()}
        alg = (ab["F"] + ab["FT"]) * (iters["jvp"] + iters["vjp"]) // max(1, len(its["jvp"]))
        ach_e = alg / ((lj + lv) / 1e3) / 1e9
        roof = {"kernel": "k_engine (problem-resident LSMR loop: SELL-32 SpMV A,A',P from HBM/L2, vectors in "
                          "shared memory, D Pi epilogues, in-CTA finalize)", "bound": "hbm",
                "achieved": round(ach_e, 1), "peak": peaks[0], "peak_source": peaks[1], "unit": "GB/s",
                "frac": round(ach_e / peaks[0], 4),
                **_traffic_fields(_traffic(args.config, alg // 2, "k_engine", args.batch) if world == 1 else None),
                "alg_bytes_per_launch": alg // 2, "launch_ms": round((lj + lv) / 2, 4),
                "loop_ms": {"jvp": round(lj, 3), "vjp": round(lv, 3)},
                "note": "one launch per solve; algorithmic bytes = (B_F + B_F') x iterations of all problems "
                        "(matrix entries re-read every iteration); achieved > HBM peak is possible: the "
                        "matrices stay L2-resident across iterations",
                "graph_path_step_kernels": steps_roof}
    else:
        roof = steps_roof
    if ab["FT_psd_flops"]:
        # the PSD share of F' is FP64-compute-shaped: its flops over the whole
        # F' launch time, against cuBLAS DGEMM measured here (a lower bound on
        # the PSD kernels' own rate, since the launch also streams the SpMVs)
        fp64 = _dgemm_tflops(dev)
        t_psd = b.time_kernel(3, reps=20)  # k_step_psd alone: the PSD units' own time
        ach_f = ab["FT_psd_flops"] / (t_psd / 1e3) / 1e12
        roof["psd_fp64"] = {"kernel": "k_step_psd (PSD units of the F' step: SpMV pass + 2 D Pi applications "
                                      "of 4 dense products each, timed alone)",
                            "achieved": round(ach_f, 3), "peak": round(fp64, 2), "unit": "TFLOP/s",
                            "peak_source": "cuBLAS DGEMM 8192^3 fp64, measured in this run",
                            "frac": round(ach_f / fp64, 4), "flops_per_launch": ab["FT_psd_flops"],
                            "launch_ms": round(t_psd, 4), "products": "mma.sync m8n8k4 f64 (DMMA)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # contract: N=1 only
        cpu = cpu_baseline(bt, dirs, K, args, scaling)
    if rank == 0:
        line = {
            "metric": "jvp+vjp evals/s", "value": round(value, 3), "unit": "evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (KKT-reverse instances, SURVEY §8(d) recipe; random directions)",
            "config": {"workload": f"{args.config}: {CONFIGS[args.config]}", "evals_per_step": units_total,
                       "per_rank_problems": units_here,
                       "lsmr": f"fixed cap K={K} (atol=btol=0) for jvp and vjp; step includes batch preparation",
                       "l2": "256 MiB L2 flush between timed steps (excluded from timing)",
                       "parallelism": (f"row shards of one problem x{world} (NCCL allreduce of the A' partials)" if comm
                                       else f"one shard of a fixed batch per rank x{world}" if scaling == "strong"
                                       else f"an independent batch of {units_here} per rank x{world}"
                                       if args.config in BATCH else f"replicas x{world}")},
            "e2e": e2e, "gpu_launches": int(launches), "roofline": roof, "cpu_baseline": cpu,
            "clocks": clk.summary(), "lsmr_iterations_per_s": round(value * 2 * K, 1),
            "lsmr_iterations": its_summary,
        }
        print(json.dumps(line))
    if comm is not None:
        comm.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    else:
        import torch.distributed as tdist

        if tdist.is_initialized():  # the --row-shards one-rank group
            tdist.destroy_process_group()


def _blk(b):
    from paper_2508_17522_b200.cones import ConeBlock

    k, d, o, a = b
    if k == "psd":
        return ConeBlock(k, order=o)
    if k in ("pow", "dpow"):
        return ConeBlock(k, alpha=a)
    if k in ("exp", "dexp"):
        return ConeBlock(k)
    return ConeBlock(k, dim=d)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def _dgemm_tflops(dev, n=8192, reps=5):
    """Measured fp64 GEMM rate (cuBLAS DGEMM, CUDA events, best of reps):
    the FP64 tensor-core roofline the PSD products are compared with."""
    import torch
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2 * n ** 3 / (best / 1e3) / 1e12


def _traffic_fields(t):
    """roofline keys: "traffic" = DRAM bytes per launch (the contract's
    number), "traffic_detail" = read / write split and where it came from."""
    return {"traffic": t["bytes"] if t else None, "traffic_detail": t}


def _has_psd(cfg):
    return cfg == "c4"


def _traffic(cfg, alg, kernel="k_step", batch=None):
    """DRAM bytes (read + write) per launch of the dominant kernel, captured
    IN THIS RUN: tools/traffic_probe.py rebuilds this workload and runs the
    hot path once under `ncu --metrics dram__bytes_read.sum,
    dram__bytes_write.sum` filtered to that kernel (one launch).  Falls back
    to the committed capture (profiles/traffic.json) when ncu is missing or
    fails, saying so."""
    import shutil

    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else None)
    if ncu and not os.environ.get("QG_NO_NCU"):
        # an F' step of a batch with PSD blocks is two kernels (k_step over the
        # other units, k_step_psd beside it): both launches of one step
        nk = 2 if (kernel != "k_engine" and _has_psd(cfg)) else 1
        filt = ["-k", "regex:^k_engine$"] if kernel == "k_engine" else \
            ["--kernel-name-base", "mangled", "-k", "regex:k_stepILi1|k_step_psd"]
        cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum", *filt,
               "-c", str(nk), "--csv", sys.executable, os.path.join(ROOT, "tools", "traffic_probe.py"),
               "--config", cfg, "--which", "engine" if kernel == "k_engine" else "ft"]
        if batch:
            cmd += ["--batch", str(batch)]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
            vals = {}
            for line in r.stdout.splitlines():
                parts = [p.strip('"') for p in line.split('","')]
                if len(parts) > 3 and parts[-3] in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                                                     "gpu__time_duration.sum"):
                    unit, v = parts[-2], float(parts[-1].replace(",", ""))
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
                             "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1,
                             "s": 1}.get(unit, 1)
                    vals[parts[-3]] = vals.get(parts[-3], 0.0) + v * scale  # summed over the step's kernels
            if "dram__bytes_read.sum" in vals:
                return {"bytes": int(vals["dram__bytes_read.sum"] + vals.get("dram__bytes_write.sum", 0)),
                        "read": int(vals["dram__bytes_read.sum"]), "write": int(vals.get("dram__bytes_write.sum", 0)),
                        "ncu_duration_ms": round(vals.get("gpu__time_duration.sum", 0) * 1e3, 4),
                        "source": f"ncu in this run ({'k_step + k_step_psd, one F' + chr(39) + ' step' if nk == 2 else kernel + ', one launch'}, cold L2, serialised)"}
        except (OSError, subprocess.SubprocessError, ValueError):
            pass
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            v = json.load(f).get(cfg)
        return None if v is None else {"bytes": v, "source": "profiles/traffic.json (committed capture)"}
    except (OSError, ValueError):
        return None


# --------------------------------------------------------- CPU reference --
def cpu_sample_size(args, scaling, cores, bt=None, dirs=None, K=None, target_s=None, impl=None):
    """Problems in the CPU sample: ``--cpu-sample`` if given, else one per
    core, grown (in whole rounds over the cores, up to the batch) until the
    sample is about ``target_s`` seconds of CPU work."""
    if args.cpu_sample:
        return args.cpu_sample
    batched = args.config in BATCH   # many independent problems: one per host core
    base = cores if batched else 1
    if target_s is None or bt is None or not batched:
        return base
    if impl is None:
        impl = cpu_impl()[0]
    base = min(base, bt.B)
    secs = impl.time_sample(bt, dirs, K, range(base), min(cores, base))
    rounds = max(1, int(target_s / max(secs, 1e-3)))
    return min(bt.B, base * rounds)


EXTRAPOLATE = {"c3": 4, "c4": 6, "c5b": 3}   # single-problem configs whose K=100 CPU eval takes minutes


def cpu_impl():
    """The CPU implementation timed beside the GPU: the unmodified reference
    installed in baseline/_ref (conegrad, compiled backend; kind "reference")
    when it imports, else the oracle port (kind "port")."""
    from baseline import ref_cpu

    ok, why = ref_cpu.available()
    if ok:
        return ref_cpu, "reference", f"conegrad 0.1.0 from baseline/_ref ({why} SpMV backend), check=False"
    from oracle import cpu_bench

    return cpu_bench, "port", f"oracle port (reference unavailable: {why})"


def cpu_baseline(bt, dirs, K, args, scaling):
    """The reference's CPU path on the host cores (rank 0, N=1)."""
    from oracle import cpu_bench

    impl, kind, desc = cpu_impl()
    cores = cpu_bench.host_cores()
    nprob = bt.B
    if args.config in EXTRAPOLATE:
        ks = EXTRAPOLATE[args.config]
        est, t0, per_iter = impl.extrapolated_eval_seconds(bt, dirs, 0, K, ks)
        return {"value": round(1.0 / est, 6), "unit": "evals/s", "cores": 1, "kind": kind,
                "sample": f"1 problem, jvp+vjp timed at caps 0 and {ks} (setup {t0:.2f} s, "
                          f"{per_iter:.3f} s per LSMR iteration of jvp+vjp) extrapolated to K={K}; "
                          f"1 process x 1 thread ({cpu_bench.cpu_model()}); {desc}",
                "seconds": round(est, 2)}
    sample = min(cpu_sample_size(args, scaling, cores, bt, dirs, K, target_s=12.0), nprob)
    workers = min(cores, sample)
    secs = impl.time_sample(bt, dirs, K, range(sample), workers)
    return {"value": round(sample / secs, 4), "unit": "evals/s", "cores": workers, "kind": kind,
            "sample": f"{sample} of {nprob} problems of this rank's workload, jvp+vjp at K={K}, "
                      f"{workers} processes x 1 thread ({cpu_bench.cpu_model()}); {desc}",
            "seconds": round(secs, 2)}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return  # rank 0 alone times the CPU reference
    from oracle import cpu_bench

    impl, kind, desc = cpu_impl()
    bt, dirs, units_total, units_here, scaling = build_workload(args.config, 0, 1, args.batch)
    K = args.lsmr_iters
    cores = cpu_bench.host_cores()
    sample = min(cpu_sample_size(args, scaling, cores, bt, dirs, K, target_s=6.0, impl=impl), bt.B)
    workers = min(cores, sample)
    for _ in range(args.warmup):
        impl.time_sample(bt, dirs, K, range(sample), workers)
    its = []
    secs = [impl.time_sample(bt, dirs, K, range(sample), workers, its) if kind == "reference" else
            impl.time_sample(bt, dirs, K, range(sample), workers) for _ in range(args.steps)]
    value = sample / (sum(secs) / len(secs))
    flat = [i for pair in its for i in pair]
    line = {
        "impl": "reference", "metric": "jvp+vjp evals/s", "value": round(value, 4), "unit": "evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * sum(secs) / len(secs), 3), "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (same generator and seeds as the GPU arm)",
        "config": {"workload": f"{args.config}: {CONFIGS[args.config]}",
                   "lsmr": f"fixed cap K={K} (atol=btol=0)", "sample_problems_per_step": sample},
        "cpu_baseline": {"value": round(value, 4), "unit": "evals/s", "cores": workers, "kind": kind,
                         "sample": f"{sample} problems per step, {workers} processes x 1 thread "
                                   f"({cpu_bench.cpu_model()}); {desc}"},
        "e2e": {"value": round(value, 4), "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if flat:
        line["lsmr_iterations"] = {"min": min(flat), "mean": round(sum(flat) / len(flat), 2), "max": max(flat)}
    print(json.dumps(line))


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
