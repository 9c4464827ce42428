"""ctypes binding of the C ABI in ``include/bidomain_b200.h``.

The shared library is built in-tree (``paper_1711_08708_b200/libbidomain_b200.so``)
by ``__graft_entry__.build()`` / ``make -C paper_1711_08708_b200/csrc``.  There is
no CPU fallback: if the library or a GPU is missing, every product entry point
raises :class:`NativeUnavailableError`.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import (BidomainError, NonConvergenceError, NumericalBreakdownError,
                     PreconditionerError)

LIB_NAME = "libbidomain_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

BD_OK, BD_EINVAL, BD_EPRECOND, BD_ENOCONV, BD_EBREAKDOWN, BD_ECUDA, BD_ENOMEM = range(7)
INNER_KIND = {"exact": 0, "ic0": 1, "jacobi": 2}

_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_dbl = C.c_double
_pp = C.POINTER(C.c_void_p)


class NativeUnavailableError(BidomainError):
    """The sm_100a library or a CUDA device is not available."""


class BdStats(C.Structure):
    _fields_ = [
        ("iterations", _i64), ("mv_count", _i64), ("p1_count", _i64), ("pk_count", _i64),
        ("converged", _i32), ("status", _i32), ("wall_ms", _dbl), ("device_ms", _dbl),
        ("final_residual", _dbl), ("curvature", _dbl),
    ]


# (name, restype, argtypes) — every symbol declared in include/bidomain_b200.h
SIGNATURES = [
    ("bd_version", C.c_char_p, []),
    ("bd_ctx_create", _i32, [C.c_int, _vp, _pp]),
    ("bd_ctx_destroy", _i32, [_vp]),
    ("bd_ctx_set_stream", _i32, [_vp, _vp]),
    ("bd_ctx_synchronize", _i32, [_vp]),
    ("bd_last_error", C.c_char_p, [_vp]),
    ("bd_csr_create", _i32, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _pp]),
    ("bd_csr_destroy", _i32, [_vp]),
    ("bd_spmv", _i32, [_vp, _vp, _vp, _dbl, _dbl]),
    ("bd_spmv_split", _i32, [_vp, _vp, _i64, _vp, _vp, _dbl, _dbl]),
    ("bd_dot", _i32, [_vp, _i64, _vp, _vp, C.POINTER(_dbl)]),
    ("bd_mean", _i32, [_vp, _i64, _vp, C.POINTER(_dbl)]),
    ("bd_system_create", _i32, [_vp, _vp, _vp, _vp, _vp, _dbl, _pp]),
    ("bd_system_destroy", _i32, [_vp]),
    ("bd_system_apply", _i32, [_vp, _vp, _vp]),
    ("bd_system_normalize", _i32, [_vp, _vp, _vp]),
    ("bd_system_weighted_mean_u", _i32, [_vp, _vp, C.POINTER(_dbl)]),
    ("bd_inner_create", _i32, [_vp, C.c_int, _i64, _vp, _vp, _vp, C.c_int, _pp,
                               C.POINTER(C.c_int)]),
    ("bd_inner_create_ex", _i32, [_vp, C.c_int, _i64, _vp, _vp, _vp, C.c_int, _vp, C.c_int, _pp,
                                  C.POINTER(C.c_int)]),
    ("bd_inner_destroy", _i32, [_vp]),
    ("bd_inner_apply", _i32, [_vp, _vp, _vp]),
    ("bd_inner_factor_info", _i32, [_vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)]),
    ("bd_inner_export_factor", _i32, [_vp, _vp, _vp, _vp, _vp]),
    ("bd_blocklu_create", _i32, [_vp, _vp, _vp, _dbl, _pp]),
    ("bd_blocklu_destroy", _i32, [_vp]),
    ("bd_blocklu_apply", _i32, [_vp, _vp, _vp]),
    ("bd_blocklu_bulk_inverse", _i32, [_vp, _vp, _vp]),
    ("bd_blocklu_schur_inverse", _i32, [_vp, _vp, _vp]),
    ("bd_blocklu_counters", _i32, [_vp, C.POINTER(_i64)]),
    ("bd_blocklu_reset_counters", _i32, [_vp]),
    ("bd_pcg_solve", _i32, [_vp, _vp, _vp, _vp, _dbl, _i64, _vp, C.POINTER(BdStats), _vp,
                            C.POINTER(_i64), _vp, C.POINTER(_i64)]),
    ("bd_profile_enable", _i32, [_vp, C.c_int]),
    ("bd_profile_read", _i32, [_vp, _vp, _vp, C.c_int]),
    ("bd_launch_count", _i64, [_vp]),
    ("bd_membrane_rhs", _i32, [_vp, _vp, _vp, _vp, C.c_uint64, _dbl, _dbl, _dbl, _dbl, _dbl,
                               _dbl, _dbl, _vp, _vp]),
    ("bd_membrane_rhs_raw", _i32, [_vp, _i64, _i64, _vp, _dbl, _vp, _vp, _vp, C.c_uint64, _dbl,
                                   _dbl, _dbl, _dbl, _dbl, _dbl, _dbl, _vp, _vp]),
    ("bd_membrane_gate", _i32, [_vp, _i64, _vp, _vp, _dbl, _dbl, _dbl, _dbl, _dbl, _dbl, _vp]),
    ("bd_assemble_p1", _i32, [_vp, C.c_int, _i64, _vp, _i64, _vp, _vp, _vp, _pp, C.POINTER(_i64)]),
    ("bd_assemble_export", _i32, [_vp, _vp, _vp, _vp, _vp]),
    ("bd_tensors_transmural", _i32, [_vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp, C.c_int, _vp, _vp]),
    ("bd_assemble_destroy", _i32, [_vp]),
    ("bd_step_track", _i32, [_vp, _vp, _vp, _vp, _dbl, _dbl, _dbl, _dbl, _dbl, _vp, C.POINTER(_dbl)]),
    ("bd_shard_create", _i32, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _dbl, _vp, _vp, _dbl,
                               _i64, _vp, _vp, _vp, _pp]),
    ("bd_shard_destroy", _i32, [_vp]),
    ("bd_shard_vectors", _i32, [_vp, _pp]),
    ("bd_shard_begin", _i32, [_vp, _dbl, _i64, _vp]),
    ("bd_shard_lambda", _i32, [_vp, _vp, _vp, _vp, C.c_int]),
    ("bd_shard_init", _i32, [_vp, _vp, C.c_int]),
    ("bd_shard_check", _i32, [_vp, C.c_int]),
    ("bd_shard_update", _i32, [_vp]),
    ("bd_shard_pinv1", _i32, [_vp]),
    ("bd_shard_pinv2", _i32, [_vp, _vp]),
    ("bd_shard_pinv3", _i32, [_vp, _vp]),
    ("bd_shard_pinv4", _i32, [_vp]),
    ("bd_shard_finish", _i32, [_vp, C.c_int]),
    ("bd_shard_wmean", _i32, [_vp]),
    ("bd_shard_normalize", _i32, [_vp, _vp]),
    ("bd_shard_done", _i32, [_vp, C.POINTER(C.c_int)]),
    ("bd_shard_read", _i32, [_vp, C.POINTER(_i64), C.POINTER(_dbl), _vp, _vp, _i64]),
    ("bd_gather", _i32, [_vp, _i64, _vp, _vp, _vp]),
]

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load the shared library and declare every symbol (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise NativeUnavailableError(
                    f"{LIB_NAME} not built at {path}; run __graft_entry__.build()")
            lib = C.CDLL(path)
            for name, res, args in SIGNATURES:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def lib():
    return load_library()


def check(status: int, ctx=None, stats=None):
    """Map a bd_status onto the reference exception types (bd/errors.py)."""
    if status == BD_OK:
        return
    msg = lib().bd_last_error(ctx).decode() if ctx else f"status {status}"
    if status == BD_EINVAL:
        raise ValueError(msg)
    if status == BD_EPRECOND:
        raise PreconditionerError(msg)
    if status == BD_ENOCONV:
        raise NonConvergenceError(msg, stats=stats)
    if status == BD_EBREAKDOWN:
        raise NumericalBreakdownError(msg, stats=stats)
    raise BidomainError(f"CUDA failure: {msg}")


class Context:
    """One device + stream; owns the native bd_ctx handle."""

    _default = None

    def __init__(self, device: int = 0):
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailableError("no CUDA device: the bidomain path has no CPU fallback")
        self.device = torch.device("cuda", device)
        torch.cuda.init()
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device).cuda_stream
        h = C.c_void_p()
        check(lib().bd_ctx_create(device, C.c_void_p(stream), C.byref(h)))
        self.handle = h

    @classmethod
    def default(cls) -> "Context":
        if cls._default is None:
            cls._default = Context(0)
        return cls._default

    def sync_stream(self):
        """Point the native context at torch's current stream."""
        import torch

        stream = torch.cuda.current_stream(self.device).cuda_stream
        lib().bd_ctx_set_stream(self.handle, C.c_void_p(stream))

    def launches(self) -> int:
        return int(lib().bd_launch_count(self.handle))

    def synchronize(self):
        check(lib().bd_ctx_synchronize(self.handle), self.handle)

    def __del__(self):
        try:
            if getattr(self, "handle", None) and _lib is not None:
                _lib.bd_ctx_destroy(self.handle)
        except Exception:
            pass


def ptr(t) -> C.c_void_p:
    """Device pointer of a contiguous fp64 CUDA tensor."""
    if t is None:
        return C.c_void_p(None)
    return C.c_void_p(t.data_ptr())
