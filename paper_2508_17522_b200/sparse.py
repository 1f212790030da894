"""Host-side CSC containers with the reference's validation contract.

``CscMatrix`` keeps the reference layout -- int64 ``col_ptr``/``row_idx``,
float64 ``values``, strictly increasing rows per column, finite values
(reference sparse.py:19-133) -- because that is the wire format callers
already hold.  Validation is host bookkeeping; every product runs on the
GPU (``matvec``/``rmatvec`` call the library's SpMV, there is no NumPy
product path).
"""

import numpy as np

from paper_2508_17522_b200 import _native as N
from paper_2508_17522_b200.errors import ValidationError


def _as(name, a, dtype):
    try:
        return np.ascontiguousarray(a, dtype=dtype)
    except (TypeError, ValueError) as exc:
        raise ValidationError(f"{name} is not numeric: {exc}") from None


class CscMatrix:
    """Immutable compressed-sparse-column matrix (validated at construction)."""

    __slots__ = ("nrows", "ncols", "col_ptr", "row_idx", "values", "_cols", "_dev")

    def __init__(self, nrows, ncols, col_ptr, row_idx, values, _trusted=False):
        nrows, ncols = int(nrows), int(ncols)
        col_ptr = _as("col_ptr", col_ptr, np.int64)
        row_idx = _as("row_idx", row_idx, np.int64)
        values = _as("matrix values", values, np.float64)
        if not _trusted:
            _validate(nrows, ncols, col_ptr, row_idx, values)
        self.nrows, self.ncols = nrows, ncols
        self.col_ptr, self.row_idx, self.values = col_ptr, row_idx, values
        self._cols = None
        self._dev = None

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    @property
    def nnz(self):
        return int(self.values.shape[0])

    def __repr__(self):
        return f"CscMatrix(shape={self.shape}, nnz={self.nnz})"

    @classmethod
    def zeros(cls, nrows, ncols):
        return cls(nrows, ncols, np.zeros(ncols + 1, np.int64), np.zeros(0, np.int64), np.zeros(0))

    @classmethod
    def from_dense(cls, arr):
        arr = np.asarray(arr, dtype=np.float64)
        if arr.ndim != 2:
            raise ValidationError("from_dense expects a 2-d array")
        cols, rows = np.nonzero(arr.T)
        cp = np.zeros(arr.shape[1] + 1, dtype=np.int64)
        np.cumsum(np.bincount(cols, minlength=arr.shape[1]), out=cp[1:])
        return cls(arr.shape[0], arr.shape[1], cp, rows.astype(np.int64), arr[rows, cols])

    def to_dense(self):
        out = np.zeros(self.shape)
        out[self.row_idx, self.entry_cols()] = self.values
        return out

    def entry_cols(self):
        if self._cols is None:
            self._cols = np.repeat(np.arange(self.ncols, dtype=np.int64), np.diff(self.col_ptr))
        return self._cols

    def with_values(self, values):
        values = _as("matrix values", values, np.float64)
        if values.shape != (self.nnz,):
            raise ValidationError(f"expected {self.nnz} values, got {values.shape}")
        if not np.all(np.isfinite(values)):
            raise ValidationError("matrix values must be finite")
        return CscMatrix(self.nrows, self.ncols, self.col_ptr, self.row_idx, values, _trusted=True)

    def device_arrays(self):
        """Cached CUDA copies (col_ptr, row_idx, values)."""
        import torch

        if self._dev is None:
            self._dev = (N.to_dev(self.col_ptr, torch.int64), N.to_dev(self.row_idx, torch.int64),
                         N.to_dev(self.values, torch.float64))
        return self._dev

    def _spmv(self, v, adjoint):
        import torch

        lib = N.lib()
        cp, ri, va = self.device_arrays()
        n_in, n_out = (self.nrows, self.ncols) if adjoint else (self.ncols, self.nrows)
        v = np.ascontiguousarray(v, dtype=np.float64)
        if v.shape != (n_in,):
            what = "rmatvec" if adjoint else "matvec"
            raise ValidationError(f"{what} expects a vector of length {n_in}, got {v.shape}")
        x = N.to_dev(v, torch.float64) if n_in else N.empty(1)
        out = N.empty(n_out)
        N.check(lib.qg_spmv_csc(self.nrows, self.ncols, N.ptr(cp), N.ptr(ri), N.ptr(va), self.nnz,
                                1 if adjoint else 0, N.ptr(x), N.ptr(out), N.stream_ptr()))
        return out[:n_out].cpu().numpy()

    def matvec(self, x):
        """``A @ x`` on the GPU."""
        return self._spmv(x, False)

    def rmatvec(self, y):
        """``A.T @ y`` on the GPU."""
        return self._spmv(y, True)


def _validate(nrows, ncols, col_ptr, row_idx, values):
    """Structure checks of the reference CscMatrix (sparse.py:34-73)."""
    if nrows < 0 or ncols < 0:
        raise ValidationError("matrix dimensions must be nonnegative")
    if col_ptr.ndim != 1 or col_ptr.shape[0] != ncols + 1:
        raise ValidationError(f"col_ptr must have length ncols + 1 = {ncols + 1}")
    if row_idx.ndim != 1 or values.ndim != 1 or row_idx.shape[0] != values.shape[0]:
        raise ValidationError("row_idx and values must be 1-d arrays of equal length")
    if col_ptr[0] != 0 or col_ptr[-1] != row_idx.shape[0]:
        raise ValidationError("col_ptr must start at 0 and end at nnz")
    if np.any(np.diff(col_ptr) < 0):
        raise ValidationError("col_ptr must be nondecreasing")
    nnz = row_idx.shape[0]
    if nnz:
        if row_idx.min() < 0 or row_idx.max() >= nrows:
            raise ValidationError("row index out of range")
        step = np.diff(row_idx)
        last_in_col = col_ptr[1:-1] - 1
        last_in_col = last_in_col[(last_in_col >= 0) & (last_in_col < nnz - 1)]
        inside = np.ones(nnz - 1, dtype=bool)
        inside[last_in_col] = False
        if np.any(step[inside] <= 0):
            raise ValidationError("row indices must be strictly increasing within each column")
    if not np.all(np.isfinite(values)):
        raise ValidationError("matrix values must be finite")


def add_scaled(a, b, alpha=1.0):
    """``a + alpha * b`` on the union pattern, entries of a column in row
    order, cancellations kept as explicit entries (reference sparse.py:142-170;
    host-side construction of shifted problem data for fd_jvp)."""
    if a.shape != b.shape:
        raise ValidationError(f"cannot add matrices of shapes {a.shape} and {b.shape}")
    stride = np.int64(max(a.nrows, 1))
    keys = np.concatenate([a.entry_cols() * stride + a.row_idx, b.entry_cols() * stride + b.row_idx])
    uniq, inv = np.unique(keys, return_inverse=True)
    # per union entry: 0 + a_ij (+ alpha b_ij), in operand order
    vals = np.bincount(inv, weights=np.concatenate([a.values, alpha * b.values]), minlength=uniq.size)
    cols, rows = uniq // stride, uniq % stride
    cp = np.zeros(a.ncols + 1, dtype=np.int64)
    np.cumsum(np.bincount(cols, minlength=a.ncols), out=cp[1:])
    return CscMatrix(a.nrows, a.ncols, cp, rows.astype(np.int64), vals)


def same_pattern(a, b):
    return (a.shape == b.shape and (a.col_ptr is b.col_ptr or np.array_equal(a.col_ptr, b.col_ptr))
            and (a.row_idx is b.row_idx or np.array_equal(a.row_idx, b.row_idx)))


def check_symmetric(mat, tol=1e-12):
    """Pattern symmetric and values within ``tol * max|v|`` (sparse.py:173-194)."""
    if mat.nrows != mat.ncols:
        raise ValidationError(f"matrix of shape {mat.shape} cannot be symmetric")
    if mat.nnz == 0:
        return
    n = np.int64(mat.nrows)
    r, c = mat.row_idx, mat.entry_cols()
    k1, k2 = c * n + r, r * n + c
    o1, o2 = np.argsort(k1, kind="stable"), np.argsort(k2, kind="stable")
    if not np.array_equal(k1[o1], k2[o2]):
        raise ValidationError("sparsity pattern is not symmetric")
    if np.any(np.abs(mat.values[o1] - mat.values[o2]) > tol * np.max(np.abs(mat.values))):
        raise ValidationError("matrix values are not symmetric")
