"""Binary ingest beside the reference's JSON.

The reference's wire format is JSON (``jsonio.py``): at C5b's 5e7 stored
entries that is ~1.5 GB of decimal text.  These helpers store the same
objects -- with the same field names as the JSON files (jsonio.py:21-33) --
as ``.npz`` archives of raw little-endian arrays (bit-exact, no decimal
round trip), and the concatenated batch layout of ``qg_batch_desc`` for
feeding ``QCPBatch.from_host`` / ``from_device`` directly.  Any DLPack
producer (CuPy, JAX, ...) enters through ``from_dlpack``.

Validation is the product types' own (``CscMatrix``, ``ProblemData``, ...),
so a corrupt archive fails exactly like a bad JSON file.
"""

import numpy as np

from paper_2508_17522_b200.cones import ConeBlock, ConeSpec
from paper_2508_17522_b200.embedding import DataPerturbation, ProblemData
from paper_2508_17522_b200.errors import ValidationError
from paper_2508_17522_b200.solution_map import Solution, SolutionDelta
from paper_2508_17522_b200.sparse import CscMatrix

_KINDS = ("zero", "nonneg", "soc", "psd", "exp", "dexp", "pow", "dpow")
_CONE = np.dtype([("kind", "<i4"), ("dim", "<i8"), ("order", "<i8"), ("alpha", "<f8")])


def _csc_arrays(prefix, mat):
    return {f"{prefix}.shape": np.asarray(mat.shape, dtype="<i8"), f"{prefix}.col_ptr": mat.col_ptr,
            f"{prefix}.row_idx": mat.row_idx, f"{prefix}.values": mat.values}


def _csc(z, prefix):
    try:
        r, c = (int(v) for v in z[f"{prefix}.shape"])
        return CscMatrix(r, c, z[f"{prefix}.col_ptr"], z[f"{prefix}.row_idx"], z[f"{prefix}.values"])
    except KeyError as e:
        raise ValidationError(f"missing array {e.args[0]!r}") from None


def cone_table(spec):
    """ConeSpec -> structured array (kind, dim, order, alpha)."""
    out = np.zeros(len(spec.blocks), dtype=_CONE)
    for i, b in enumerate(spec.blocks):
        out[i] = (_KINDS.index(b.kind), b.dim, b.order or 0, b.alpha or 0.0)
    return out


def cone_spec(table):
    blocks = []
    for k, d, o, a in np.asarray(table, dtype=_CONE).tolist():
        if not 0 <= k < len(_KINDS):
            raise ValidationError(f"unknown cone kind code {k}")
        kind = _KINDS[k]
        blocks.append(ConeBlock(kind, dim=d) if kind in ("zero", "nonneg", "soc") else
                      ConeBlock(kind, order=o) if kind == "psd" else
                      ConeBlock(kind, alpha=a) if kind in ("pow", "dpow") else ConeBlock(kind))
    return ConeSpec(blocks)


def _check_keys(z, allowed, what):
    extra = sorted(set(z.files) - set(allowed))
    if extra:  # jsonio rejects unknown keys everywhere (jsonio.py:35-36)
        raise ValidationError(f"{what}: unknown keys {extra}")
    missing = sorted(set(allowed) - set(z.files))
    if missing:
        raise ValidationError(f"{what}: missing keys {missing}")


# ----------------------------------------------------------------- objects --
def save_problem(path, theta):
    np.savez(path, n=np.int64(theta.n), m=np.int64(theta.m), cones=cone_table(theta.cone),
             q=theta.q, b=theta.b, **_csc_arrays("P", theta.P), **_csc_arrays("A", theta.A))


def load_problem(path):
    with np.load(path, allow_pickle=False) as z:
        _check_keys(z, {"n", "m", "cones", "q", "b"} | {f"{p}.{k}" for p in "PA"
                                                       for k in ("shape", "col_ptr", "row_idx", "values")},
                    "problem")
        theta = ProblemData(_csc(z, "P"), _csc(z, "A"), z["q"], z["b"], cone_spec(z["cones"]))
        if (theta.n, theta.m) != (int(z["n"]), int(z["m"])):
            raise ValidationError("problem: n / m do not match the matrices")
        return theta


def save_solution(path, sol):
    np.savez(path, x=sol.x, y=sol.y, s=sol.s)


def load_solution(path):
    with np.load(path, allow_pickle=False) as z:
        _check_keys(z, {"x", "y", "s"}, "solution")
        return Solution(z["x"], z["y"], z["s"])


def save_perturbation(path, dtheta):
    np.savez(path, dq=dtheta.dq, db=dtheta.db, **_csc_arrays("dP", dtheta.dP), **_csc_arrays("dA", dtheta.dA))


def load_perturbation(path):
    with np.load(path, allow_pickle=False) as z:
        _check_keys(z, {"dq", "db"} | {f"{p}.{k}" for p in ("dP", "dA")
                                       for k in ("shape", "col_ptr", "row_idx", "values")}, "perturbation")
        return DataPerturbation(_csc(z, "dP"), _csc(z, "dA"), z["dq"], z["db"])


def save_delta(path, delta):
    np.savez(path, dx=delta.dx, dy=delta.dy, ds=delta.ds)


def load_delta(path):
    with np.load(path, allow_pickle=False) as z:
        _check_keys(z, {"dx", "dy", "ds"}, "delta")
        return SolutionDelta(z["dx"], z["dy"], z["ds"])


# ------------------------------------------------------- batch (C ABI) ---
_BATCH_ARRAYS = ("P_colptr", "P_rowidx", "P_vals", "A_colptr", "A_rowidx", "A_vals", "q", "b", "x", "y", "s")


def save_batch(path, n, m, P_nnz, A_nnz, blocks, arrays):
    """A batch in the ``qg_batch_desc`` layout: per-problem sizes, one cone
    table per problem (concatenated with counts) and the concatenated arrays."""
    tables = [np.asarray([(_KINDS.index(k), d, o or 0, a or 0.0) for (k, d, o, a) in bl], dtype=_CONE)
              for bl in blocks]
    np.savez(path, n=np.asarray(n, "<i8"), m=np.asarray(m, "<i8"), P_nnz=np.asarray(P_nnz, "<i8"),
             A_nnz=np.asarray(A_nnz, "<i8"), nblocks=np.asarray([len(t) for t in tables], "<i8"),
             blocks=np.concatenate(tables) if tables else np.zeros(0, _CONE),
             **{k: np.asarray(arrays[k]) for k in _BATCH_ARRAYS})


def load_batch(path):
    """-> (n, m, P_nnz, A_nnz, blocks, arrays) ready for QCPBatch.from_host."""
    with np.load(path, allow_pickle=False) as z:
        _check_keys(z, {"n", "m", "P_nnz", "A_nnz", "nblocks", "blocks"} | set(_BATCH_ARRAYS), "batch")
        n, m = z["n"].tolist(), z["m"].tolist()
        cnt, tab = z["nblocks"], z["blocks"]
        if not (len(n) == len(m) == len(cnt) == len(z["P_nnz"]) == len(z["A_nnz"])):
            raise ValidationError("batch: per-problem size arrays differ in length")
        if int(cnt.sum()) != len(tab):
            raise ValidationError("batch: block counts do not match the block table")
        off = np.concatenate([[0], np.cumsum(cnt)])
        rows = tab.tolist()
        blocks = [[(_KINDS[k], d, o, a) for (k, d, o, a) in rows[off[i]:off[i + 1]]] for i in range(len(n))]
        arrays = {k: np.array(z[k]) for k in _BATCH_ARRAYS}
        return n, m, z["P_nnz"].tolist(), z["A_nnz"].tolist(), blocks, arrays


def from_dlpack(arrays):
    """Device tensors from any DLPack producer (keys as ``qg_batch_desc``),
    zero-copy where the producer allows, for ``QCPBatch.from_device``."""
    import torch

    out = {}
    for k, v in arrays.items():
        t = torch.from_dlpack(v)
        if not t.is_cuda:
            raise ValidationError(f"{k}: DLPack tensor is not on a CUDA device")
        want = torch.int64 if k.endswith(("colptr", "rowidx")) else torch.float64
        out[k] = t.to(want).contiguous()
    return out
