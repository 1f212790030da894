"""Product cones and the GPU cone calculus.

Block kinds, canonical order and svec storage follow the reference
(cones.py:36-202).  ``project``/``project_dual``/``dprojection(_dual)`` run
the library's cone kernels (projection, root finding, batched Jacobi eigh)
on the device: a ``ConeDerivative`` is a prepared device object whose
``matvec`` is one blockwise kernel launch.
"""

import math

import numpy as np

from paper_2508_17522_b200 import _native as N
from paper_2508_17522_b200.errors import ValidationError

ZERO, NONNEG, SOC, PSD, EXP, DEXP, POW, DPOW = ("zero", "nonneg", "soc", "psd", "exp", "dexp", "pow", "dpow")
KINDS = (ZERO, NONNEG, SOC, PSD, EXP, DEXP, POW, DPOW)
_RANK = {k: i for i, k in enumerate(KINDS)}


class ConeBlock:
    """One block of a product cone (kind, dim, order for psd, alpha for pow)."""

    __slots__ = ("kind", "dim", "order", "alpha")

    def __init__(self, kind, dim=None, order=None, alpha=None):
        if kind not in KINDS:
            raise ValidationError(f"unknown cone kind {kind!r}")
        self.kind, self.order, self.alpha = kind, None, None
        if kind in (ZERO, NONNEG, SOC):
            if dim is None or int(dim) < 1:
                raise ValidationError(f"{kind} block needs dimension >= 1")
            self.dim = int(dim)
        elif kind == PSD:
            if order is None or int(order) < 1:
                raise ValidationError("psd block needs matrix order >= 1")
            self.order = int(order)
            self.dim = self.order * (self.order + 1) // 2
        elif kind in (EXP, DEXP):
            if dim not in (None, 3):
                raise ValidationError(f"{kind} block has fixed dimension 3")
            self.dim = 3
        else:
            a = None if alpha is None else float(alpha)
            if a is None or not 0.0 < a < 1.0:
                raise ValidationError(f"{kind} block needs exponent strictly inside (0, 1)")
            self.alpha, self.dim = a, 3

    zero = classmethod(lambda cls, dim: cls(ZERO, dim=dim))
    nonneg = classmethod(lambda cls, dim: cls(NONNEG, dim=dim))
    soc = classmethod(lambda cls, dim: cls(SOC, dim=dim))
    psd = classmethod(lambda cls, order: cls(PSD, order=order))
    exp = classmethod(lambda cls: cls(EXP))
    dual_exp = classmethod(lambda cls: cls(DEXP))
    power = classmethod(lambda cls, alpha: cls(POW, alpha=alpha))
    dual_power = classmethod(lambda cls, alpha: cls(DPOW, alpha=alpha))

    def __repr__(self):
        if self.kind == PSD:
            return f"ConeBlock(psd, order={self.order})"
        if self.kind in (POW, DPOW):
            return f"ConeBlock({self.kind}, alpha={self.alpha})"
        return f"ConeBlock({self.kind}, dim={self.dim})"


class ConeSpec:
    """Ordered product of blocks in canonical kind order (cones.py:132-166)."""

    __slots__ = ("blocks", "dim", "_slices", "_dev")

    def __init__(self, blocks):
        blocks = tuple(blocks)
        last = -1
        for i, b in enumerate(blocks):
            if not isinstance(b, ConeBlock):
                raise ValidationError(f"blocks[{i}] is not a ConeBlock")
            r = _RANK[b.kind]
            if r < last:
                raise ValidationError(f"cone blocks out of canonical order: {b.kind} after {blocks[i - 1].kind}")
            if r == last and b.kind in (ZERO, NONNEG):
                raise ValidationError(f"at most one {b.kind} block is allowed")
            last = r
        self.blocks = blocks
        off = np.cumsum([0] + [b.dim for b in blocks])
        self.dim = int(off[-1])
        self._slices = tuple((b, int(off[i]), int(off[i + 1])) for i, b in enumerate(blocks))
        self._dev = None

    def slices(self):
        return self._slices

    def __repr__(self):
        return f"ConeSpec({list(self.blocks)!r})"

    def _handle(self):
        """Device cone table for this spec (created once)."""
        if self._dev is None:
            self._dev = _DeviceCones(self)
        return self._dev


class _DeviceCones:
    def __init__(self, spec):
        lib = N.lib()
        h = N.c_vp()
        arr = N.cone_array(spec.blocks)
        N.check(lib.qg_cones_create(N.ctypes.byref(h), arr, len(spec.blocks), N.stream_ptr()))
        self.h, self.dim, self._lib = h, spec.dim, lib

    def __del__(self):
        try:
            if self.h:
                self._lib.qg_cones_destroy(self.h)
        except Exception:
            pass


# svec layout: lower triangle, column major, off-diagonals times sqrt(2)
def _tri(order):
    cols, rows = np.triu_indices(order)
    return rows, cols, np.where(rows == cols, 1.0, math.sqrt(2.0))


def svec(Z):
    Z = np.asarray(Z, dtype=np.float64)
    r, c, s = _tri(Z.shape[0])
    return Z[r, c] * s


def smat(v, order):
    r, c, s = _tri(order)
    vals = np.asarray(v, dtype=np.float64) / s
    Z = np.zeros((order, order))
    Z[r, c] = vals
    Z[c, r] = vals
    return Z


def _point(spec, z):
    z = np.ascontiguousarray(z, dtype=np.float64)
    if z.shape != (spec.dim,):
        raise ValidationError(f"point must have length {spec.dim}, got {z.shape}")
    if not np.all(np.isfinite(z)):
        raise ValidationError("point contains non-finite entries")
    return z


def _project(spec, z, dual):
    import torch

    z = _point(spec, z)
    if spec.dim == 0:
        return np.zeros(0)
    h = spec._handle()
    zd = N.to_dev(z, torch.float64)
    out = N.empty(spec.dim)
    N.check(N.lib().qg_cones_project(h.h, 1 if dual else 0, N.ptr(zd), N.ptr(out), N.stream_ptr()))
    return out[:spec.dim].cpu().numpy()


def project(spec, z):
    """Euclidean projection onto the product cone (GPU)."""
    return _project(spec, z, False)


def project_dual(spec, z):
    """Euclidean projection onto the dual cone (GPU)."""
    return _project(spec, z, True)


class ConeDerivative:
    """Prepared projection derivative at a point (self-adjoint); matvec on GPU."""

    __slots__ = ("dim", "_h", "_z")

    def __init__(self, spec, z, dual):
        import torch

        z = _point(spec, z)
        self.dim = spec.dim
        # a private device table so several prepared derivatives can coexist
        self._h = _DeviceCones(spec) if spec.dim else None
        if self._h is not None:
            self._z = N.to_dev(z, torch.float64)
            N.check(N.lib().qg_cones_prepare(self._h.h, 1 if dual else 0, N.ptr(self._z), N.stream_ptr()))

    def matvec_device(self, dz):
        out = N.empty(self.dim)
        N.check(N.lib().qg_cones_apply(self._h.h, N.ptr(dz), N.ptr(out), N.stream_ptr()))
        return out[:self.dim]

    def matvec(self, dz):
        import torch

        dz = np.ascontiguousarray(dz, dtype=np.float64)
        if dz.shape != (self.dim,):
            raise ValidationError(f"direction must have length {self.dim}, got {dz.shape}")
        if self.dim == 0:
            return np.zeros(0)
        return self.matvec_device(N.to_dev(dz, torch.float64)).cpu().numpy()


def dprojection(spec, z):
    return ConeDerivative(spec, z, dual=False)


def dprojection_dual(spec, z):
    return ConeDerivative(spec, z, dual=True)


def dproject(spec, z, dz):
    return dprojection(spec, z).matvec(dz)


def dproject_dual(spec, z, dz):
    return dprojection_dual(spec, z).matvec(dz)
