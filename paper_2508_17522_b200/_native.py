"""ctypes binding of libqcpgrad.so (the C ABI in include/qcpgrad.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
compute entry point raises ``DeviceError``.  Device memory and streams come
from PyTorch (plumbing only); the kernels are the library's own.
"""

import ctypes
import os
import re

import numpy as np

from paper_2508_17522_b200.errors import (
    ConegradError,
    DeviceError,
    DomainError,
    NotDifferentiableError,
    NumericalError,
    ValidationError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QG_LIB_PATH") or os.path.join(HERE, "_lib", "libqcpgrad.so")  # override: A/B builds
HEADER = os.path.join(os.path.dirname(HERE), "include", "qcpgrad.h")

c_i32, c_i64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
P_i64 = ctypes.POINTER(c_i64)

KIND_CODE = {"zero": 0, "nonneg": 1, "soc": 2, "psd": 3, "exp": 4, "dexp": 5, "pow": 6, "dpow": 7}

QG_OK, QG_ERR_VALIDATION, QG_ERR_DOMAIN, QG_ERR_NUMERICAL = 0, 1, 2, 3
QG_ERR_NOT_DIFFERENTIABLE, QG_ERR_CUDA, QG_ERR_UNSUPPORTED = 4, 5, 6


class ConeBlockC(ctypes.Structure):
    _fields_ = [("kind", c_i32), ("dim", c_i32), ("order", c_i32), ("alpha", c_dbl)]


class BatchDesc(ctypes.Structure):
    _fields_ = [("nprob", c_i64), ("n", P_i64), ("m", P_i64), ("P_nnz", P_i64), ("A_nnz", P_i64),
                ("nblocks", P_i64), ("blocks", ctypes.POINTER(ConeBlockC)),
                ("P_colptr", c_vp), ("P_rowidx", c_vp), ("P_vals", c_vp),
                ("A_colptr", c_vp), ("A_rowidx", c_vp), ("A_vals", c_vp),
                ("q", c_vp), ("b", c_vp), ("x", c_vp), ("y", c_vp), ("s", c_vp)]


class PerturbationC(ctypes.Structure):
    _fields_ = [("dP_nnz", P_i64), ("dA_nnz", P_i64),
                ("dP_colptr", c_vp), ("dP_rowidx", c_vp), ("dP_vals", c_vp),
                ("dA_colptr", c_vp), ("dA_rowidx", c_vp), ("dA_vals", c_vp),
                ("dq", c_vp), ("db", c_vp), ("same_pattern", c_i32)]


class LsmrOpts(ctypes.Structure):
    _fields_ = [("atol", c_dbl), ("btol", c_dbl), ("max_iter", c_i64)]


class DiagC(ctypes.Structure):
    _fields_ = [("iterations", c_i64), ("converged", c_i32), ("derivative_unreliable", c_i32),
                ("residual_norm", c_dbl), ("atr_norm", c_dbl), ("rhs_norm", c_dbl)]


_SIGS = {
    "qg_last_error": (ctypes.c_char_p, []),
    "qg_version": (ctypes.c_char_p, []),
    "qg_kernel_launches": (c_i64, []),
    "qg_create_batch": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.POINTER(BatchDesc), c_vp]),
    "qg_destroy": (ctypes.c_int, [c_vp]),
    "qg_handle_sizes": (ctypes.c_int, [c_vp, P_i64, P_i64, P_i64]),
    "qg_handle_layout": (ctypes.c_int, [c_vp, P_i64, P_i64]),
    "qg_handle_engine": (ctypes.c_int, [c_vp, ctypes.POINTER(ctypes.c_int32)]),
    "qg_loop_time": (ctypes.c_int, [c_vp, ctypes.POINTER(c_dbl), ctypes.POINTER(c_dbl)]),
    "qg_jvp": (ctypes.c_int, [c_vp, ctypes.POINTER(PerturbationC), ctypes.POINTER(LsmrOpts),
                              c_vp, c_vp, c_vp, ctypes.POINTER(DiagC), c_vp]),
    "qg_vjp": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(LsmrOpts),
                              c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(DiagC), c_vp]),
    "qg_apply_F": (ctypes.c_int, [c_vp, ctypes.c_int, c_vp, c_vp, c_vp]),
    "qg_embedding_point": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "qg_check": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(c_dbl), c_vp]),
    "qg_cones_create": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.POINTER(ConeBlockC), c_i64, c_vp]),
    "qg_cones_destroy": (ctypes.c_int, [c_vp]),
    "qg_cones_project": (ctypes.c_int, [c_vp, ctypes.c_int, c_vp, c_vp, c_vp]),
    "qg_cones_prepare": (ctypes.c_int, [c_vp, ctypes.c_int, c_vp, c_vp]),
    "qg_cones_apply": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "qg_time_kernel": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(c_dbl), c_vp]),
    "qg_spmv_csc": (ctypes.c_int, [c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, ctypes.c_int, c_vp, c_vp, c_vp]),
    "qg_set_point": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int, c_vp]),
    "qg_residual": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "qg_lsmr_jacobian": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.POINTER(LsmrOpts), c_vp,
                                        ctypes.POINTER(DiagC), c_vp]),
    "qg_comm_nccl_id":(ctypes.c_int, [ctypes.POINTER(ctypes.c_ubyte)]),
    "qg_comm_create_nccl": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.POINTER(ctypes.c_ubyte), ctypes.c_int,
                                           ctypes.c_int]),
    "qg_comm_create_local": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.c_int]),
    "qg_comm_destroy": (ctypes.c_int, [c_vp]),
    "qg_comm_rank": (ctypes.c_int, [c_vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    "qg_comm_allreduce": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp]),
    "qg_create_batch_dist": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.POINTER(BatchDesc), c_vp, c_vp]),
}

_lib = None


def header_symbols():
    """Function names declared by include/qcpgrad.h."""
    with open(HEADER, encoding="utf-8") as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(qg_[a-z_]+)\s*\(", text)))


def load_library():
    """Load libqcpgrad.so and bind every entry point (no device needed)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"native library missing: {LIB_PATH} (run paper_2508_17522_b200.build)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name, None)
            if fn is None and os.environ.get("QG_LIB_PATH"):
                continue  # an older A/B build; tests/test_abi.py checks the shipped library exports all
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def lib():
    """The library, after checking that a CUDA device is usable."""
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the derivative path runs only on the GPU (no CPU fallback)")
    return load_library()


def check(status):
    if status == QG_OK:
        return
    msg = load_library().qg_last_error().decode("utf-8", "replace")
    if status == QG_ERR_VALIDATION:
        raise ValidationError(msg)
    if status == QG_ERR_DOMAIN:
        raise DomainError(msg)
    if status == QG_ERR_NOT_DIFFERENTIABLE:
        raise NotDifferentiableError(msg)
    if status == QG_ERR_NUMERICAL:
        m = re.search(r"iteration (\d+)", msg)
        raise NumericalError(msg, iteration=int(m.group(1)) if m else None)
    if status == QG_ERR_UNSUPPORTED:
        raise DeviceError(f"unsupported: {msg}")
    raise DeviceError(msg)


# ---------------------------------------------------------------- device --

def device():
    import torch

    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def to_dev(a, dtype):
    """numpy / torch -> contiguous CUDA tensor of ``dtype`` (torch dtype)."""
    import torch

    if isinstance(a, torch.Tensor):
        # pinned sources DMA asynchronously, ordered on the current stream
        return a.to(device=device(), dtype=dtype, non_blocking=a.is_pinned()).contiguous()
    arr = np.ascontiguousarray(a)
    t = torch.from_numpy(arr)
    return t.to(device=device(), dtype=dtype, non_blocking=False).contiguous()


def to_host(t):
    """CUDA tensor -> NumPy array through a pinned staging buffer (torch's
    caching host allocator reuses it across calls; DMA instead of a pageable
    copy)."""
    import torch

    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return out.numpy()


def empty(n, dtype=None):
    import torch

    return torch.empty(max(int(n), 1), dtype=dtype or torch.float64, device=device())


def ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def cone_array(blocks):
    arr = (ConeBlockC * max(len(blocks), 1))()
    for i, b in enumerate(blocks):
        arr[i].kind = KIND_CODE[b.kind]
        arr[i].dim = int(b.dim)
        arr[i].order = int(b.order or 0)
        arr[i].alpha = float(b.alpha or 0.0)
    return arr


CONE_DTYPE = np.dtype([("kind", np.int32), ("dim", np.int32), ("order", np.int32), ("_pad", np.int32),
                       ("alpha", np.float64)])


def cone_struct(blocks):
    """Structured array in qg_cone_block layout from ConeBlock objects or
    (kind, dim, order, alpha) tuples."""
    out = np.zeros(len(blocks), dtype=CONE_DTYPE)
    for i, b in enumerate(blocks):
        if isinstance(b, tuple):
            k, d, o, a = b
        else:
            k, d, o, a = b.kind, b.dim, b.order, b.alpha
        out[i] = (KIND_CODE[k], int(d), int(o or 0), 0, float(a or 0.0))
    return out


def cone_table(per_problem):
    """Concatenated cone table for a batch; lists shared between problems
    (the same list object) are converted once."""
    if per_problem and all(bl is per_problem[0] for bl in per_problem):
        # one shared block list (a homogeneous batch): tile it
        one = cone_struct(per_problem[0])
        return (np.ascontiguousarray(np.tile(one, len(per_problem))),
                np.full(len(per_problem), len(one), dtype=np.int64))
    cache, parts = {}, []
    for bl in per_problem:
        arr = cache.get(id(bl))
        if arr is None:
            arr = cache[id(bl)] = cone_struct(bl)
        parts.append(arr)
    flat = np.concatenate(parts) if parts else np.zeros(0, dtype=CONE_DTYPE)
    return np.ascontiguousarray(flat), np.array([len(b) for b in per_problem], dtype=np.int64)


def as_i64_ptr(arr):
    return arr.ctypes.data_as(P_i64)


def i64_array(values):
    arr = (c_i64 * max(len(values), 1))()
    for i, v in enumerate(values):
        arr[i] = int(v)
    return arr


def kernel_launches():
    return int(load_library().qg_kernel_launches())


def version():
    return load_library().qg_version().decode()


__all__ = ["ConegradError", "load_library", "lib", "check", "header_symbols"]
