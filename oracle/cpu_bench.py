"""CPU timing of the oracle (the reference algorithm restated) on synthetic
batches -- TEST / BASELINE INFRASTRUCTURE ONLY.  Used by bench.py's
``cpu_baseline`` leg and ``--impl reference`` arm, never by the product.

One eval = jvp + vjp of one problem at a fixed LSMR cap K (atol=btol=0),
exactly the work the GPU arm does per problem (reference solution_map.py:
325-385 with check=False).
"""

import os
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

from oracle import cones as C  # noqa: E402
from oracle import qcp as Q  # noqa: E402


def problem(batch, dirs, p):
    """Problem p of a synth Batch as oracle tuples (theta, sol, dtheta, delta)."""
    n, m = batch.n[p], batch.m[p]
    xo, yo = sum(batch.n[:p]), sum(batch.m[:p])
    po, ao = sum(batch.P_nnz[:p]), sum(batch.A_nnz[:p])
    cpo = xo + p
    P = Q.Csc(n, n, batch.P_colptr[cpo:cpo + n + 1], batch.P_rowidx[po:po + batch.P_nnz[p]],
              batch.P_vals[po:po + batch.P_nnz[p]])
    A = Q.Csc(m, n, batch.A_colptr[cpo:cpo + n + 1], batch.A_rowidx[ao:ao + batch.A_nnz[p]],
              batch.A_vals[ao:ao + batch.A_nnz[p]])
    blocks = [C.block(k, dim=d, order=o, alpha=a) for (k, d, o, a) in batch.blocks[p]]
    th = Q.Problem(P, A, batch.q[xo:xo + n], batch.b[yo:yo + m], blocks)
    sol = Q.Sol(batch.x[xo:xo + n], batch.y[yo:yo + m], batch.s[yo:yo + m])
    pert = Q.Pert(Q.Csc(n, n, P.col_ptr, P.row_idx, dirs.dP[po:po + batch.P_nnz[p]]),
                  Q.Csc(m, n, A.col_ptr, A.row_idx, dirs.dA[ao:ao + batch.A_nnz[p]]),
                  dirs.dq[xo:xo + n], dirs.db[yo:yo + m])
    de = Q.Delta(dirs.dx[xo:xo + n], dirs.dy[yo:yo + m], dirs.ds[yo:yo + m])
    return th, sol, pert, de


def eval_one(th, sol, pert, de, K):
    Q.jvp(th, sol, pert, atol=0.0, btol=0.0, max_iter=K)
    Q.vjp(th, sol, de, atol=0.0, btol=0.0, max_iter=K)


_G = {}


def _one_thread():
    """Context limiting BLAS / OpenMP pools to one thread (numpy may have been
    imported before the environment variables above took effect)."""
    try:
        from threadpoolctl import threadpool_limits

        return threadpool_limits(1)
    except ImportError:
        import contextlib

        return contextlib.nullcontext()


def _init(batch, dirs, K):
    _G.update(batch=batch, dirs=dirs, K=K)
    try:  # one BLAS thread per worker process (numpy may be loaded before the env vars)
        from threadpoolctl import threadpool_limits

        _G["limits"] = threadpool_limits(1)
    except ImportError:
        pass


def _work(p):
    eval_one(*problem(_G["batch"], _G["dirs"], p), _G["K"])
    return p


def time_sample(batch, dirs, K, problems, workers):
    """Wall seconds to run jvp+vjp on ``problems`` over ``workers`` processes."""
    if workers <= 1:
        with _one_thread():
            t = time.perf_counter()
            for p in problems:
                eval_one(*problem(batch, dirs, p), K)
            return time.perf_counter() - t
    import multiprocessing as mp

    ctx = mp.get_context("fork")
    with ctx.Pool(workers, initializer=_init, initargs=(batch, dirs, K)) as pool:
        pool.map(_work, list(problems)[:workers])  # warm the workers (first calls are cold)
        t = time.perf_counter()
        pool.map(_work, list(problems), chunksize=1)
        return time.perf_counter() - t


def extrapolated_eval_seconds(batch, dirs, p, K, k_small):
    """Seconds of one jvp+vjp at cap K for problem p, estimated from runs at
    caps 0 (setup only) and k_small: t(K) = t0 + K (t_k - t0) / k_small.
    Used for configurations whose full-K CPU eval takes minutes.  One BLAS
    thread (the reported ``cores`` is 1)."""
    prob = problem(batch, dirs, p)
    with _one_thread():
        t = time.perf_counter()
        eval_one(*prob, 0)
        t0 = time.perf_counter() - t
        t = time.perf_counter()
        eval_one(*prob, k_small)
        tk = time.perf_counter() - t
    per_iter = max(tk - t0, 0.0) / k_small
    return t0 + K * per_iter, t0, per_iter


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
