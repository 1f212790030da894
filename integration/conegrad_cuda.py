"""The reference-side binding of INTEGRATION.md, made real: routes the
unmodified reference's (``conegrad`` 0.1.0) ``jvp`` / ``vjp`` /
``check_solution`` through libqcpgrad's C ABI.

    import conegrad_cuda          # integration/ on sys.path
    conegrad_cuda.install()       # conegrad.jvp / vjp now run on the B200

This is what a maintainer would add to the reference as
``conegrad/_kernels/cuda.py``.  It converts the reference's
value types to this repo's client (``paper_2508_17522_b200``, whose every
compute call goes through ``include/qcpgrad.h``), calls the GPU path, and
converts results, diagnostics and exceptions back, so callers -- including
the reference's own test suite -- cannot tell the difference except in
rounding:

* ``jvp(theta, sol, dtheta, *, atol, btol, max_iter, check, check_tol)``
  replaces ``solution_map.jvp`` (reference solution_map.py:325-355);
* ``vjp(...)`` replaces ``solution_map.vjp`` (solution_map.py:358-385);
* ``check_solution(theta, sol, tol)`` replaces solution_map.py:263-288
  (the five KKT residuals on the device, ``qg_check``).

Exceptions are re-raised as the reference's own classes (errors.py:13-38)
with the same messages; a failed pre-check carries ``.kkt`` as a reference
``KktReport``.  ``install()`` rebinds the names everywhere the reference
imported them by value (``conegrad``, ``conegrad.solution_map``,
``conegrad.cli``), so it must run before callers bind them (the pytest
plugin ``integration/conegrad_plugin.py`` does it at start-up).
"""

import contextlib

import numpy as np

import conegrad
from conegrad import errors as ref_errors
from conegrad import solution_map as ref_sm

import paper_2508_17522_b200 as qg
from paper_2508_17522_b200 import errors as qg_errors

_REF_JVP, _REF_VJP, _REF_CHECK = ref_sm.jvp, ref_sm.vjp, ref_sm.check_solution


# ------------------------------------------------------------ conversions --
def _csc(M):
    if isinstance(M, conegrad.CscMatrix):
        r, c = M.shape
        return qg.CscMatrix(r, c, M.col_ptr, M.row_idx, M.values, _trusted=True)
    return M  # not a reference matrix: the client's validation reports it


def _cone(spec):
    if not isinstance(spec, conegrad.ConeSpec):
        return spec
    out = []
    for b in spec.blocks:
        if b.kind == "psd":
            out.append(qg.ConeBlock("psd", order=b.order))
        elif b.kind in ("pow", "dpow"):
            out.append(qg.ConeBlock(b.kind, alpha=b.alpha))
        elif b.kind in ("exp", "dexp"):
            out.append(qg.ConeBlock(b.kind))
        else:
            out.append(qg.ConeBlock(b.kind, dim=b.dim))
    return qg.ConeSpec(out)


def _theta(theta):
    if not isinstance(theta, conegrad.ProblemData):
        return theta
    # the reference already validated it (symmetric P, shapes, finiteness)
    return qg.ProblemData(_csc(theta.P), _csc(theta.A), theta.q, theta.b, _cone(theta.cone), _trusted=True)


def _sol(sol):
    return qg.Solution(sol.x, sol.y, sol.s) if isinstance(sol, conegrad.Solution) else sol


def _dtheta(d):
    if not isinstance(d, conegrad.DataPerturbation):
        return d
    return qg.DataPerturbation(_csc(d.dP), _csc(d.dA), d.dq, d.db, _trusted=True)


def _delta(d):
    return qg.SolutionDelta(d.dx, d.dy, d.ds) if isinstance(d, conegrad.SolutionDelta) else d


def _kkt(r):
    if r is None:
        return None
    return ref_sm.KktReport(r.primal, r.stationarity, r.gap, r.primal_cone_distance, r.dual_cone_distance,
                            r.tol, r.ok)


def _diag(d):
    return ref_sm.Diagnostics(d.iterations, d.converged, d.residual_norm, d.rhs_norm, d.derivative_unreliable,
                              _kkt(d.kkt))


_ERRORS = (
    (qg_errors.NotDifferentiableError, ref_errors.NotDifferentiableError),
    (qg_errors.NumericalError, ref_errors.NumericalError),
    (qg_errors.DomainError, ref_errors.DomainError),
    (qg_errors.ValidationError, ref_errors.ValidationError),
)


@contextlib.contextmanager
def _reference_errors():
    """Re-raise the client's exceptions as the reference's classes."""
    try:
        yield
    except qg_errors.DeviceError:
        raise  # a device failure has no reference counterpart: surface it as is
    except qg_errors.ConegradError as e:
        for mine, theirs in _ERRORS:
            if isinstance(e, mine):
                if theirs in (ref_errors.NumericalError, ref_errors.NotDifferentiableError):
                    err = theirs(str(e), getattr(e, "iteration", None))
                else:
                    err = theirs(str(e))
                if hasattr(e, "kkt"):
                    err.kkt = _kkt(e.kkt)
                raise err from None
        raise ref_errors.ConegradError(str(e)) from None


# ---------------------------------------------------------- entry points --
def jvp(theta, sol, dtheta, *, atol=1e-10, btol=1e-10, max_iter=None, check=True, check_tol=None):
    """``conegrad.jvp`` on the GPU (reference solution_map.py:325-355)."""
    with _reference_errors():
        d, diag = qg.jvp(_theta(theta), _sol(sol), _dtheta(dtheta), atol=atol, btol=btol, max_iter=max_iter,
                         check=check, check_tol=check_tol)
    return ref_sm.SolutionDelta(d.dx, d.dy, d.ds), _diag(diag)


def vjp(theta, sol, delta, *, atol=1e-10, btol=1e-10, max_iter=None, check=True, check_tol=None):
    """``conegrad.vjp`` on the GPU (reference solution_map.py:358-385); dP /
    dA come back on the patterns (and CSC storage order) of P / A."""
    with _reference_errors():
        g, diag = qg.vjp(_theta(theta), _sol(sol), _delta(delta), atol=atol, btol=btol, max_iter=max_iter,
                         check=check, check_tol=check_tol)
    dP = theta.P.with_values(np.asarray(g.dP.values))
    dA = theta.A.with_values(np.asarray(g.dA.values))
    return conegrad.DataPerturbation(dP, dA, g.dq, g.db), _diag(diag)


def check_solution(theta, sol, tol=None):
    """``conegrad.check_solution`` with the residuals computed on the GPU."""
    with _reference_errors():
        r = qg.check_solution(_theta(theta), _sol(sol), tol)
    return _kkt(r)


def install(check=True):
    """Rebind the reference's jvp / vjp (and, with ``check``,
    check_solution) to the GPU path wherever the reference bound them."""
    import conegrad.cli as ref_cli

    for mod in (conegrad, ref_sm, ref_cli):
        if hasattr(mod, "jvp"):
            mod.jvp = jvp
        if hasattr(mod, "vjp"):
            mod.vjp = vjp
        if check and hasattr(mod, "check_solution"):
            mod.check_solution = check_solution


def uninstall():
    import conegrad.cli as ref_cli

    for mod in (conegrad, ref_sm, ref_cli):
        for name, fn in (("jvp", _REF_JVP), ("vjp", _REF_VJP), ("check_solution", _REF_CHECK)):
            if hasattr(mod, name):
                setattr(mod, name, fn)
