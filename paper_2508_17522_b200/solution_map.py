"""Derivatives of the QCP solution map on the GPU -- the drop-in boundary.

Mirrors the reference's public surface (solution_map.py:50-385): ``jvp`` /
``vjp`` with the same keyword arguments, defaults, pre-check behaviour,
return types and ``Diagnostics``.  Underneath, everything runs through the
C ABI of libqcpgrad.so:

* ``QCP`` -- the prepared "QCP object" of the north star: problem data and a
  primal-dual solution uploaded once, the projection derivative prepared
  once, then any number of ``jvp``/``vjp`` calls;
* ``QCPBatch`` -- a batch of independent problems solved together (one
  kernel sequence for the whole batch, per-problem LSMR scalars and stop
  flags).

Host arrays (NumPy) in, host arrays out, exactly like the reference; the
``*_device`` methods take and return CUDA tensors for on-device pipelines.
"""

from dataclasses import dataclass
from typing import Optional

import numpy as np

from paper_2508_17522_b200 import _native as N
from paper_2508_17522_b200 import cones
from paper_2508_17522_b200.embedding import DataPerturbation, ProblemData
from paper_2508_17522_b200.errors import DomainError, ValidationError
from paper_2508_17522_b200.sparse import same_pattern


def _vector(name, v, length=None):
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.ndim != 1 or (length is not None and v.shape != (length,)):
        raise ValidationError(f"{name} must be a vector of length {length}, got {v.shape}")
    if not np.all(np.isfinite(v)):
        raise ValidationError(f"{name} contains non-finite entries")
    return v


class Solution:
    """A primal-dual solution ``(x, y, s)``."""

    __slots__ = ("x", "y", "s")

    def __init__(self, x, y, s):
        self.x = _vector("x", x)
        self.y = _vector("y", y)
        self.s = _vector("s", s, len(self.y))

    n = property(lambda self: len(self.x))
    m = property(lambda self: len(self.y))

    def __repr__(self):
        return f"Solution(n={self.n}, m={self.m})"


class SolutionDelta:
    """A direction ``(dx, dy, ds)`` in solution space."""

    __slots__ = ("dx", "dy", "ds")

    def __init__(self, dx, dy, ds):
        self.dx = _vector("dx", dx)
        self.dy = _vector("dy", dy)
        self.ds = _vector("ds", ds, len(self.dy))

    def dot(self, other):
        return float(self.dx @ other.dx + self.dy @ other.dy + self.ds @ other.ds)

    def norm(self):
        return float(np.sqrt(self.dot(self)))

    def __repr__(self):
        return f"SolutionDelta(n={len(self.dx)}, m={len(self.dy)}, norm={self.norm():.3e})"


@dataclass
class KktReport:
    """Optimality residuals of a candidate solution (solution_map.py:99-136)."""

    primal: float
    stationarity: float
    gap: float
    primal_cone_distance: float
    dual_cone_distance: float
    tol: float
    ok: bool

    def max_violation(self):
        return max(self.primal, self.stationarity, self.gap, self.primal_cone_distance,
                   self.dual_cone_distance)

    def as_dict(self):
        return {"primal": self.primal, "stationarity": self.stationarity, "gap": self.gap,
                "primal_cone_distance": self.primal_cone_distance,
                "dual_cone_distance": self.dual_cone_distance, "tol": self.tol, "ok": self.ok}


@dataclass
class Diagnostics:
    """What happened inside a jvp / vjp (solution_map.py:139-167)."""

    iterations: int
    converged: bool
    residual_norm: float
    rhs_norm: float
    derivative_unreliable: bool
    kkt: Optional[KktReport]

    def as_dict(self):
        return {"iterations": self.iterations, "converged": self.converged,
                "residual_norm": self.residual_norm, "rhs_norm": self.rhs_norm,
                "derivative_unreliable": self.derivative_unreliable,
                "kkt": None if self.kkt is None else self.kkt.as_dict()}


def _diag(d, kkt=None):
    return Diagnostics(int(d.iterations), bool(d.converged), float(d.residual_norm), float(d.rhs_norm),
                       bool(d.derivative_unreliable), kkt)


def _opts(atol, btol, max_iter):
    o = N.LsmrOpts()
    o.atol, o.btol = float(atol), float(btol)
    # C ABI: 0 -> default cap 10*(in+out); < 0 -> an explicit cap of zero
    o.max_iter = 0 if max_iter is None else (int(max_iter) if int(max_iter) > 0 else -1)
    return o


# ---------------------------------------------------------------------------
# prepared handles
# ---------------------------------------------------------------------------

class QCPBatch:
    """A batch of independent QCPs prepared on the GPU.

    ``thetas``/``sols`` are sequences of ``ProblemData``/``Solution``.  All
    kernels run once per LSMR iteration for the whole batch; converged
    problems drop out via per-problem flags.
    """

    def __init__(self, thetas, sols):
        import torch

        thetas, sols = list(thetas), list(sols)
        if len(thetas) != len(sols) or not thetas:
            raise ValidationError("need equally many problems and solutions (at least one)")
        for th, so in zip(thetas, sols):
            if not isinstance(th, ProblemData):
                raise ValidationError(f"theta must be a ProblemData, got {type(th).__name__}")
            if not isinstance(so, Solution):
                raise ValidationError(f"sol must be a Solution, got {type(so).__name__}")
            if (so.n, so.m) != (th.n, th.m):
                raise ValidationError(f"solution dimensions ({so.n}, {so.m}) do not match "
                                      f"problem dimensions ({th.n}, {th.m})")
        self.thetas, self.sols = thetas, sols
        cat = lambda xs, dt=np.float64: np.concatenate([np.asarray(v, dtype=dt) for v in xs]) if xs else np.zeros(0, dt)
        f64, i64 = torch.float64, torch.int64
        dev = dict(
            P_colptr=N.to_dev(cat([t.P.col_ptr for t in thetas], np.int64), i64),
            P_rowidx=N.to_dev(cat([t.P.row_idx for t in thetas], np.int64), i64),
            P_vals=N.to_dev(cat([t.P.values for t in thetas]), f64),
            A_colptr=N.to_dev(cat([t.A.col_ptr for t in thetas], np.int64), i64),
            A_rowidx=N.to_dev(cat([t.A.row_idx for t in thetas], np.int64), i64),
            A_vals=N.to_dev(cat([t.A.values for t in thetas]), f64),
            q=N.to_dev(cat([t.q for t in thetas]), f64), b=N.to_dev(cat([t.b for t in thetas]), f64),
            x=N.to_dev(cat([s.x for s in sols]), f64), y=N.to_dev(cat([s.y for s in sols]), f64),
            s=N.to_dev(cat([s.s for s in sols]), f64))
        self._create([t.n for t in thetas], [t.m for t in thetas], [t.P.nnz for t in thetas],
                     [t.A.nnz for t in thetas], [list(t.cone.blocks) for t in thetas], dev)
        self._sol_dev = (dev["x"], dev["y"], dev["s"])

    @classmethod
    def from_device(cls, n, m, P_nnz, A_nnz, blocks, tensors, comm=None):
        """Create from concatenated CUDA tensors (keys as in ``qg_batch_desc``).
        With ``comm`` (``dist.Comm``) the tensors are this rank's row shard of
        a row-partitioned batch (``dist.py``)."""
        self = cls.__new__(cls)
        self.thetas = self.sols = None
        self._create(n, m, P_nnz, A_nnz, blocks, tensors, comm)
        self._sol_dev = (tensors["x"], tensors["y"], tensors["s"])
        return self

    @classmethod
    def from_host(cls, n, m, P_nnz, A_nnz, blocks, arrays, comm=None):
        """Create from concatenated HOST arrays (NumPy or pinned torch CPU
        tensors, keys as in ``qg_batch_desc``): the host-buffer boundary."""
        import torch

        f64, i64 = torch.float64, torch.int64
        t = {k: N.to_dev(v, i64 if k.endswith(("colptr", "rowidx")) else f64) for k, v in arrays.items()}
        return cls.from_device(n, m, P_nnz, A_nnz, blocks, t, comm=comm)

    def jvp_host(self, dP, dA, dq, db, **kw):
        """jvp from concatenated host arrays on the patterns of P / A; returns
        host (dx, dy, ds) and per-problem Diagnostics."""
        import torch

        d = [N.to_dev(a, torch.float64) for a in (dP, dA, dq, db)]
        dx, dy, ds, diags = self.jvp_device(*d, **kw)
        return N.to_host(dx), N.to_host(dy), N.to_host(ds), [_diag(g) for g in diags]

    def vjp_host(self, dx, dy, ds, **kw):
        import torch

        d = [N.to_dev(a, torch.float64) for a in (dx, dy, ds)]
        dP, dA, dq, db, diags = self.vjp_device(*d, **kw)
        return (N.to_host(dP), N.to_host(dA), N.to_host(dq), N.to_host(db),
                [_diag(g) for g in diags])

    def layout(self):
        """(SELL-32 slices on the X side, on the Y side); 0 = CSR path."""
        sx, sy = N.ctypes.c_int64(), N.ctypes.c_int64()
        N.check(N.lib().qg_handle_layout(self._h, N.ctypes.byref(sx), N.ctypes.byref(sy)))
        return int(sx.value), int(sy.value)

    def resident(self):
        """True when this batch's LSMR solves run problem-resident (one
        persistent kernel, a CTA per problem, vectors in shared memory)."""
        r = N.ctypes.c_int32()
        N.check(N.lib().qg_handle_engine(self._h, N.ctypes.byref(r)))
        return bool(r.value)

    def loop_time(self):
        """(jvp ms, vjp ms): device time of the last LSMR loops on this batch
        (CUDA events on the call's stream, after the init phases)."""
        j, v = N.ctypes.c_double(), N.ctypes.c_double()
        N.check(N.lib().qg_loop_time(self._h, N.ctypes.byref(j), N.ctypes.byref(v)))
        return float(j.value), float(v.value)

    def time_kernel(self, which, reps=20):
        """Mean device ms per launch of a hot kernel (0: F step, 1: F' step,
        2: LSMR update, 3: the F' step's PSD units alone), CUDA events on the
        current stream."""
        ms = N.c_dbl()
        N.check(N.lib().qg_time_kernel(self._h, int(which), int(reps), N.ctypes.byref(ms), N.stream_ptr()))
        return float(ms.value)

    def _create(self, n, m, P_nnz, A_nnz, blocks, t, comm=None):
        lib = N.lib()
        self.B = len(n)
        self.n, self.m = [int(v) for v in n], [int(v) for v in m]
        self.P_nnz, self.A_nnz = [int(v) for v in P_nnz], [int(v) for v in A_nnz]
        self.blocks = blocks
        self.NX, self.NY = sum(self.n), sum(self.m)
        self.xoff = np.concatenate([[0], np.cumsum(self.n)]).astype(np.int64)
        self.yoff = np.concatenate([[0], np.cumsum(self.m)]).astype(np.int64)
        self.poff = np.concatenate([[0], np.cumsum(self.P_nnz)]).astype(np.int64)
        self.aoff = np.concatenate([[0], np.cumsum(self.A_nnz)]).astype(np.int64)
        table, counts = N.cone_table(blocks)
        keep = dict(n=np.asarray(self.n, dtype=np.int64), m=np.asarray(self.m, dtype=np.int64),
                    pn=np.asarray(self.P_nnz, dtype=np.int64), an=np.asarray(self.A_nnz, dtype=np.int64),
                    nb=counts, blk=table)
        d = N.BatchDesc()
        d.nprob = self.B
        d.n, d.m = N.as_i64_ptr(keep["n"]), N.as_i64_ptr(keep["m"])
        d.P_nnz, d.A_nnz, d.nblocks = N.as_i64_ptr(keep["pn"]), N.as_i64_ptr(keep["an"]), N.as_i64_ptr(keep["nb"])
        d.blocks = table.ctypes.data_as(N.ctypes.POINTER(N.ConeBlockC))
        for k in ("P_colptr", "P_rowidx", "P_vals", "A_colptr", "A_rowidx", "A_vals", "q", "b", "x", "y", "s"):
            setattr(d, k, t[k].data_ptr())
        h = N.c_vp()
        if comm is None:
            N.check(lib.qg_create_batch(N.ctypes.byref(h), N.ctypes.byref(d), N.stream_ptr()))
        else:
            N.check(lib.qg_create_batch_dist(N.ctypes.byref(h), N.ctypes.byref(d), comm.ptr, N.stream_ptr()))
        self._h, self._lib, self._comm = h, lib, comm  # the handle keeps the communicator alive

    def close(self):
        if getattr(self, "_h", None):
            self._lib.qg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- device-level entry points ------------------------------------------
    def jvp_device(self, dP_vals, dA_vals, dq, db, *, atol=1e-10, btol=1e-10, max_iter=None,
                   dP_struct=None, dA_struct=None):
        """jvp with CUDA inputs.  ``d*_vals`` on the patterns of P / A unless
        ``dP_struct``/``dA_struct`` = (colptr, rowidx, nnz list) give others."""
        lib = N.lib()
        pc = N.PerturbationC()
        keep = []
        if dP_struct is None and dA_struct is None:
            pc.same_pattern = 1
            pc.dP_nnz, pc.dA_nnz = N.i64_array(self.P_nnz), N.i64_array(self.A_nnz)
            keep += [pc.dP_nnz, pc.dA_nnz]
        else:
            pc.same_pattern = 0
            (pcp, pri, pnz), (acp, ari, anz) = dP_struct, dA_struct
            pc.dP_nnz, pc.dA_nnz = N.i64_array(pnz), N.i64_array(anz)
            pc.dP_colptr, pc.dP_rowidx = pcp.data_ptr(), pri.data_ptr()
            pc.dA_colptr, pc.dA_rowidx = acp.data_ptr(), ari.data_ptr()
            keep += [pc.dP_nnz, pc.dA_nnz]
        pc.dP_vals, pc.dA_vals = dP_vals.data_ptr(), dA_vals.data_ptr()
        pc.dq, pc.db = dq.data_ptr(), db.data_ptr()
        dx, dy, ds = N.empty(self.NX), N.empty(self.NY), N.empty(self.NY)
        diags = (N.DiagC * self.B)()
        o = _opts(atol, btol, max_iter)
        N.check(lib.qg_jvp(self._h, N.ctypes.byref(pc), N.ctypes.byref(o), N.ptr(dx), N.ptr(dy), N.ptr(ds),
                           diags, N.stream_ptr()))
        return dx[:self.NX], dy[:self.NY], ds[:self.NY], list(diags)

    def vjp_device(self, dx, dy, ds, *, atol=1e-10, btol=1e-10, max_iter=None):
        lib = N.lib()
        dP, dA = N.empty(self.poff[-1]), N.empty(self.aoff[-1])
        dq, db = N.empty(self.NX), N.empty(self.NY)
        diags = (N.DiagC * self.B)()
        o = _opts(atol, btol, max_iter)
        N.check(lib.qg_vjp(self._h, N.ptr(dx), N.ptr(dy), N.ptr(ds), N.ctypes.byref(o), N.ptr(dP), N.ptr(dA),
                           N.ptr(dq), N.ptr(db), diags, N.stream_ptr()))
        return dP[:self.poff[-1]], dA[:self.aoff[-1]], dq[:self.NX], db[:self.NY], list(diags)

    def apply_F_device(self, w, transpose=False):
        out = N.empty(self.NX + self.NY + self.B)
        N.check(N.lib().qg_apply_F(self._h, 1 if transpose else 0, N.ptr(w), N.ptr(out), N.stream_ptr()))
        return out

    def embedding_point_device(self):
        out = N.empty(self.NX + self.NY + self.B)
        N.check(N.lib().qg_embedding_point(self._h, N.ptr(out), N.stream_ptr()))
        return out

    # -- re-solving oracle (testkit.refine / fd_jvp) --------------------------
    def set_point_device(self, z, want_deriv=True):
        """Move the handle to the embedding point ``z`` (CUDA, [X | Y | T])."""
        N.check(N.lib().qg_set_point(self._h, N.ptr(z.contiguous()), 1 if want_deriv else 0, N.stream_ptr()))

    def residual_device(self):
        """Normalized residual N(z) at the handle's point (CUDA, [X | Y | T])."""
        out = N.empty(self.NX + self.NY + self.B)
        N.check(N.lib().qg_residual(self._h, N.ptr(out), N.stream_ptr()))
        return out[:self.NX + self.NY + self.B]

    def lsmr_jacobian_device(self, rhs, rank1=None, *, atol=1e-10, btol=1e-10, max_iter=None):
        """LSMR on J = F - rank1 e_N' (F alone for rank1=None) at the handle's
        point; returns (solution, diags)."""
        sol = N.empty(self.NX + self.NY + self.B)
        diags = (N.DiagC * self.B)()
        o = _opts(atol, btol, max_iter)
        N.check(N.lib().qg_lsmr_jacobian(self._h, N.ptr(rhs.contiguous()),
                                         N.ptr(rank1.contiguous()) if rank1 is not None else None,
                                         N.ctypes.byref(o), N.ptr(sol), diags, N.stream_ptr()))
        return sol[:self.NX + self.NY + self.B], list(diags)

    def kkt_device(self, x=None, y=None, s=None):
        x0, y0, s0 = self._sol_dev
        rep = (N.c_dbl * (5 * self.B))()
        N.check(N.lib().qg_check(self._h, N.ptr(x if x is not None else x0), N.ptr(y if y is not None else y0),
                                 N.ptr(s if s is not None else s0), rep, N.stream_ptr()))
        return np.array(rep[:]).reshape(self.B, 5)

    # -- host-level batch helpers --------------------------------------------
    def _split(self, arr, off):
        return [arr[off[i]:off[i + 1]] for i in range(self.B)]

    def jvp_all(self, dthetas, **kw):
        import torch

        same = all(same_pattern(d.dP, t.P) and same_pattern(d.dA, t.A) for d, t in zip(dthetas, self.thetas))
        cat = lambda xs: N.to_dev(np.concatenate(xs) if xs else np.zeros(0), torch.float64)
        args = dict(dP_vals=cat([d.dP.values for d in dthetas]), dA_vals=cat([d.dA.values for d in dthetas]),
                    dq=cat([d.dq for d in dthetas]), db=cat([d.db for d in dthetas]))
        if not same:
            i64 = lambda xs: N.to_dev(np.concatenate(xs), torch.int64)
            args["dP_struct"] = (i64([d.dP.col_ptr for d in dthetas]), i64([d.dP.row_idx for d in dthetas]),
                                 [d.dP.nnz for d in dthetas])
            args["dA_struct"] = (i64([d.dA.col_ptr for d in dthetas]), i64([d.dA.row_idx for d in dthetas]),
                                 [d.dA.nnz for d in dthetas])
        dx, dy, ds, diags = self.jvp_device(**args, **kw)
        dx, dy, ds = N.to_host(dx), N.to_host(dy), N.to_host(ds)
        out = []
        for i in range(self.B):
            xs, ys = slice(self.xoff[i], self.xoff[i + 1]), slice(self.yoff[i], self.yoff[i + 1])
            out.append((SolutionDelta(dx[xs], dy[ys], ds[ys]), _diag(diags[i])))
        return out

    def vjp_all(self, deltas, **kw):
        import torch

        cat = lambda xs: N.to_dev(np.concatenate(xs) if xs else np.zeros(0), torch.float64)
        dP, dA, dq, db, diags = self.vjp_device(cat([d.dx for d in deltas]), cat([d.dy for d in deltas]),
                                                cat([d.ds for d in deltas]), **kw)
        dP, dA, dq, db = (N.to_host(t) for t in (dP, dA, dq, db))
        out = []
        for i, th in enumerate(self.thetas):
            g = DataPerturbation(th.P.with_values(dP[self.poff[i]:self.poff[i + 1]]),
                                 th.A.with_values(dA[self.aoff[i]:self.aoff[i + 1]]),
                                 dq[self.xoff[i]:self.xoff[i + 1]], db[self.yoff[i]:self.yoff[i + 1]],
                                 _trusted=True)
            out.append((g, _diag(diags[i])))
        return out


class QCP(QCPBatch):
    """Prepared derivative of one QCP's solution map at ``sol``."""

    def __init__(self, theta, sol):
        super().__init__([theta], [sol])
        self.theta, self.sol = theta, sol

    def jvp(self, dtheta, *, atol=1e-10, btol=1e-10, max_iter=None):
        _check_dtheta(self.theta, dtheta)
        (delta, diag), = self.jvp_all([dtheta], atol=atol, btol=btol, max_iter=max_iter)
        return delta, diag

    def vjp(self, delta, *, atol=1e-10, btol=1e-10, max_iter=None):
        _check_delta(self.theta, delta)
        (grad, diag), = self.vjp_all([delta], atol=atol, btol=btol, max_iter=max_iter)
        return grad, diag

    def apply_F(self, w, transpose=False):
        """``F w`` / ``F' w`` (embedding.py:420-425), host vectors."""
        import torch

        w = _vector("w", w, self.theta.embedding_dim)
        return self.apply_F_device(N.to_dev(w, torch.float64), transpose)[:w.size].cpu().numpy()

    def embedding_point(self):
        return self.embedding_point_device()[:self.theta.embedding_dim].cpu().numpy()

    def kkt(self, tol=None):
        r = self.kkt_device()[0]
        tol = float(1e-6 * (1.0 + self.theta.norm()) if tol is None else tol)
        return KktReport(*(float(v) for v in r), tol, bool(max(r) <= tol))


# ---------------------------------------------------------------------------
# reference-compatible functions
# ---------------------------------------------------------------------------

def _check_dtheta(theta, dtheta):
    if not isinstance(dtheta, DataPerturbation):
        raise ValidationError(f"dtheta must be a DataPerturbation, got {type(dtheta).__name__}")
    if (dtheta.n, dtheta.m) != (theta.n, theta.m):
        raise ValidationError(f"perturbation dimensions ({dtheta.n}, {dtheta.m}) do not match "
                              f"problem dimensions ({theta.n}, {theta.m})")


def _check_delta(theta, delta):
    if not isinstance(delta, SolutionDelta):
        raise ValidationError(f"delta must be a SolutionDelta, got {type(delta).__name__}")
    if (len(delta.dx), len(delta.dy)) != (theta.n, theta.m):
        raise ValidationError(f"delta dimensions ({len(delta.dx)}, {len(delta.dy)}) do not match "
                              f"problem dimensions ({theta.n}, {theta.m})")


def _check_sol(theta, sol):
    if not isinstance(sol, Solution):
        raise ValidationError(f"sol must be a Solution, got {type(sol).__name__}")
    if (sol.n, sol.m) != (theta.n, theta.m):
        raise ValidationError(f"solution dimensions ({sol.n}, {sol.m}) do not match "
                              f"problem dimensions ({theta.n}, {theta.m})")


def embed(sol):
    """``z = (x, y - s, 1)`` (solution_map.py:170-179)."""
    return np.concatenate([sol.x, sol.y - sol.s, [1.0]])


def phi(theta, z):
    """Decode an embedding point (solution_map.py:182-194); projection on GPU."""
    z = _vector("z", z, theta.embedding_dim)
    zN = z[-1]
    if zN <= 0.0:
        raise DomainError(f"decoding needs z_N > 0, got {zN}")
    mid = z[theta.n:-1]
    proj = cones.project_dual(theta.cone, mid)
    return Solution(z[:theta.n] / zN, proj / zN, (proj - mid) / zN)


def check_solution(theta, sol, tol=None):
    """KKT residuals of ``sol`` (solution_map.py:263-288), on the GPU."""
    _check_sol(theta, sol)
    return QCP(theta, sol).kkt(tol)


def _prepare(theta, sol, check, check_tol):
    _check_sol(theta, sol)
    q = QCP(theta, sol)
    report = None
    if check:
        try:
            report = q.kkt(check_tol)
        except BaseException:
            q.close()
            raise
        if not report.ok:
            q.close()  # release the handle's device buffers now, not at garbage collection
            exc = ValidationError("solution fails the optimality pre-check: "
                                  f"max violation {report.max_violation():.3e} > tolerance {report.tol:.3e} "
                                  "(pass check=False to differentiate anyway)")
            exc.kkt = report
            raise exc
    return q, report


def jvp(theta, sol, dtheta, *, atol=1e-10, btol=1e-10, max_iter=None, check=True, check_tol=None):
    """Directional derivative of the solution map (solution_map.py:325-355)."""
    q, report = _prepare(theta, sol, check, check_tol)
    try:
        delta, diag = q.jvp(dtheta, atol=atol, btol=btol, max_iter=max_iter)
    finally:
        q.close()
    diag.kkt = report
    return delta, diag


def vjp(theta, sol, delta, *, atol=1e-10, btol=1e-10, max_iter=None, check=True, check_tol=None):
    """Adjoint of the solution-map derivative (solution_map.py:358-385)."""
    q, report = _prepare(theta, sol, check, check_tol)
    try:
        grad, diag = q.vjp(delta, atol=atol, btol=btol, max_iter=max_iter)
    finally:
        q.close()
    diag.kkt = report
    return grad, diag
