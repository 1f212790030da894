"""Problem data and data-space perturbations (reference embedding.py:59-189).

Host containers with the reference's validation; the embedding maps
themselves (D_uQ, D_theta Q, F, F') exist only as device kernels behind the
``QCP`` handle in :mod:`paper_2508_17522_b200.solution_map`.
"""

import numpy as np

from paper_2508_17522_b200.cones import ConeSpec
from paper_2508_17522_b200.errors import ValidationError
from paper_2508_17522_b200.sparse import CscMatrix, check_symmetric, same_pattern


def _vec(name, v, n):
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.shape != (n,):
        raise ValidationError(f"{name} must have shape ({n},), got {v.shape}")
    if not np.all(np.isfinite(v)):
        raise ValidationError(f"{name} contains non-finite entries")
    return v


def _mat(name, M, r, c):
    if not isinstance(M, CscMatrix):
        raise ValidationError(f"{name} must be a CscMatrix, got {type(M).__name__}")
    if M.shape != (r, c):
        raise ValidationError(f"{name} must have shape ({r}, {c}), got {M.shape}")
    return M


class ProblemData:
    """``(P, A, q, b)`` plus the cone; P square, symmetric, both triangles stored."""

    __slots__ = ("n", "m", "P", "A", "q", "b", "cone")

    def __init__(self, P, A, q, b, cone, _trusted=False):
        if not isinstance(cone, ConeSpec):
            raise ValidationError(f"cone must be a ConeSpec, got {type(cone).__name__}")
        if not isinstance(A, CscMatrix):
            raise ValidationError(f"A must be a CscMatrix, got {type(A).__name__}")
        self.m, self.n = A.shape
        self.P = _mat("P", P, self.n, self.n)
        if not _trusted:
            check_symmetric(self.P)
        self.A = A
        self.q = _vec("q", q, self.n)
        self.b = _vec("b", b, self.m)
        if cone.dim != self.m:
            raise ValidationError(f"cone dimension {cone.dim} does not match the row count {self.m} of A")
        self.cone = cone

    @property
    def embedding_dim(self):
        return self.n + self.m + 1

    def norm(self):
        P, A = self.P.values, self.A.values
        return float(np.sqrt(P @ P + A @ A + self.q @ self.q + self.b @ self.b))

    def __repr__(self):
        return (f"ProblemData(n={self.n}, m={self.m}, nnz_P={self.P.nnz}, nnz_A={self.A.nnz}, "
                f"blocks={len(self.cone.blocks)})")


class DataPerturbation:
    """A direction ``(dP, dA, dq, db)``; dP symmetric."""

    __slots__ = ("n", "m", "dP", "dA", "dq", "db")

    def __init__(self, dP, dA, dq, db, _trusted=False):
        if not isinstance(dA, CscMatrix):
            raise ValidationError(f"dA must be a CscMatrix, got {type(dA).__name__}")
        self.m, self.n = dA.shape
        self.dP = _mat("dP", dP, self.n, self.n)
        if not _trusted:
            check_symmetric(self.dP)
        self.dA = dA
        self.dq = _vec("dq", dq, self.n)
        self.db = _vec("db", db, self.m)

    @classmethod
    def zeros_like(cls, theta):
        return cls(theta.P.with_values(np.zeros(theta.P.nnz)), theta.A.with_values(np.zeros(theta.A.nnz)),
                   np.zeros(theta.n), np.zeros(theta.m))

    def scaled(self, alpha):
        a = float(alpha)
        return DataPerturbation(self.dP.with_values(a * self.dP.values), self.dA.with_values(a * self.dA.values),
                                a * self.dq, a * self.db, _trusted=True)

    def dot(self, other):
        if not (same_pattern(self.dP, other.dP) and same_pattern(self.dA, other.dA)):
            raise ValidationError("perturbations must share sparsity patterns")
        return float(self.dP.values @ other.dP.values + self.dA.values @ other.dA.values
                     + self.dq @ other.dq + self.db @ other.db)

    def norm(self):
        return float(np.sqrt(self.dot(self)))

    def __repr__(self):
        return f"DataPerturbation(n={self.n}, m={self.m}, norm={self.norm():.3e})"
