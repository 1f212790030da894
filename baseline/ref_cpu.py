"""CPU timing of the UNMODIFIED reference (conegrad 0.1.0, installed into
baseline/_ref by baseline/install_ref.sh) on this repo's synthetic batches --
BASELINE INFRASTRUCTURE ONLY, used by bench.py's ``cpu_baseline`` leg and
its ``--impl reference`` arm.  Nothing in the product imports it.

One eval = ``conegrad.jvp`` + ``conegrad.vjp`` of one problem through the
reference's own public API and stock code path (compiled Cython SpMV
backend), with ``atol=btol=0, max_iter=K, check=False`` -- the fixed-cap
protocol the GPU arm runs (reference solution_map.py:325-385).
"""

import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.path.join(HERE, "_ref")


def available():
    """(True, backend) if the installed reference imports, else (False, why)."""
    if not os.path.isdir(os.path.join(REF, "conegrad")):
        return False, "baseline/_ref not installed (run baseline/install_ref.sh)"
    try:
        cg = _cg()
        from conegrad import _kernels
        return True, _kernels.active_backend()
    except Exception as e:  # noqa: BLE001 - report, the caller falls back
        return False, f"conegrad import failed: {e}"


def _cg():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import conegrad
    return conegrad


def problem(batch, dirs, p):
    """Problem p of a synth Batch as conegrad objects (theta, sol, dtheta, delta)."""
    cg = _cg()
    n, m = batch.n[p], batch.m[p]
    xo, yo = sum(batch.n[:p]), sum(batch.m[:p])
    po, ao = sum(batch.P_nnz[:p]), sum(batch.A_nnz[:p])
    cpo = xo + p
    pcp, pri = batch.P_colptr[cpo:cpo + n + 1], batch.P_rowidx[po:po + batch.P_nnz[p]]
    acp, ari = batch.A_colptr[cpo:cpo + n + 1], batch.A_rowidx[ao:ao + batch.A_nnz[p]]
    P = cg.CscMatrix(n, n, pcp, pri, batch.P_vals[po:po + batch.P_nnz[p]])
    A = cg.CscMatrix(m, n, acp, ari, batch.A_vals[ao:ao + batch.A_nnz[p]])
    blocks = []
    for (k, d, o, a) in batch.blocks[p]:
        blocks.append(cg.ConeBlock(k, order=o) if k == "psd" else
                      cg.ConeBlock(k, alpha=a) if k in ("pow", "dpow") else
                      cg.ConeBlock(k) if k in ("exp", "dexp") else cg.ConeBlock(k, dim=d))
    th = cg.ProblemData(P, A, batch.q[xo:xo + n], batch.b[yo:yo + m], cg.ConeSpec(blocks))
    sol = cg.Solution(batch.x[xo:xo + n], batch.y[yo:yo + m], batch.s[yo:yo + m])
    pert = cg.DataPerturbation(cg.CscMatrix(n, n, pcp, pri, dirs.dP[po:po + batch.P_nnz[p]]),
                               cg.CscMatrix(m, n, acp, ari, dirs.dA[ao:ao + batch.A_nnz[p]]),
                               dirs.dq[xo:xo + n], dirs.db[yo:yo + m])
    de = cg.SolutionDelta(dirs.dx[xo:xo + n], dirs.dy[yo:yo + m], dirs.ds[yo:yo + m])
    return th, sol, pert, de


def eval_one(th, sol, pert, de, K):
    """jvp + vjp through the reference's public API; returns the two LSMR
    iteration counts (a fixed cap with atol=btol=0 should run exactly K)."""
    cg = _cg()
    _, dj = cg.jvp(th, sol, pert, atol=0.0, btol=0.0, max_iter=K, check=False)
    _, dv = cg.vjp(th, sol, de, atol=0.0, btol=0.0, max_iter=K, check=False)
    return dj.iterations, dv.iterations


_G = {}


def _one_thread():
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(1)
    except ImportError:
        import contextlib
        return contextlib.nullcontext()


def _init(batch, dirs, K):
    _G.update(batch=batch, dirs=dirs, K=K)
    try:
        from threadpoolctl import threadpool_limits
        _G["limits"] = threadpool_limits(1)
    except ImportError:
        pass


def _work(p):
    return eval_one(*problem(_G["batch"], _G["dirs"], p), _G["K"])


def time_sample(batch, dirs, K, problems, workers, its=None):
    """Wall seconds of jvp+vjp on ``problems`` over ``workers`` processes
    (one BLAS thread each); ``its`` (a list) collects the iteration counts."""
    problems = list(problems)
    if workers <= 1:
        with _one_thread():
            t = time.perf_counter()
            res = [eval_one(*problem(batch, dirs, p), K) for p in problems]
            dt = time.perf_counter() - t
    else:
        import multiprocessing as mp
        ctx = mp.get_context("fork")
        with ctx.Pool(workers, initializer=_init, initargs=(batch, dirs, K)) as pool:
            pool.map(_work, problems[:workers])  # warm the workers (first calls are cold)
            t = time.perf_counter()
            res = pool.map(_work, problems, chunksize=1)
            dt = time.perf_counter() - t
    if its is not None:
        its.extend(res)
    return dt


def extrapolated_eval_seconds(batch, dirs, p, K, k_small):
    """Seconds of one jvp+vjp at cap K for problem p from runs at caps 0
    (setup only) and k_small: t(K) = t0 + K (t_k - t0) / k_small.  For
    configurations whose full-K CPU eval takes minutes."""
    prob = problem(batch, dirs, p)
    with _one_thread():
        eval_one(*prob, 0)  # warm (first calls are cold)
        t = time.perf_counter()
        eval_one(*prob, 0)
        t0 = time.perf_counter() - t
        t = time.perf_counter()
        eval_one(*prob, k_small)
        tk = time.perf_counter() - t
    per_iter = max(tk - t0, 0.0) / k_small
    return t0 + K * per_iter, t0, per_iter
