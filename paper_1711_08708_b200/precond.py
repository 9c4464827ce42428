"""Block-LU preconditioner with the monodomain Schur surrogate (drop-in for
bd/precond.py:31-312).

Host side (scipy, setup only): β = mean diag S_1, the grounded S_1 + β e₀e₀ᵀ
and K_m = S_m + γ diag(M_H) are formed exactly as the reference does
(including the CSR additions that drop stored zeros), then handed to the
sm_100a library, which factors them on the host in C++ (IC(0) bit-exact with
`_try_factor`, or a nested-dissection sparse Cholesky for "exact") and runs
every application on the GPU: sync-free level-ordered triangular solves,
S_i SpMVs and the mean projections fused into their producers.
"""
from __future__ import annotations

import ctypes as C
from concurrent.futures import ThreadPoolExecutor
from abc import ABC, abstractmethod
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .assembly import Space, assemble_stiffness, lumped_mass_diagonal
from .conductivity import ConductivityParams, TensorField
from .errors import PreconditionerError
from .mesh import Mesh
from .system import BidomainSystem, BlockVector, _as_block, _torch, as_device, csr_arrays

INNER_NAMES = ("exact", "ic0", "jacobi")


def build_monodomain_matrix(mesh: Mesh, params: ConductivityParams, gamma: float,
                            fibers=None, assembly: str = "host") -> sp.csr_matrix:
    """K_m = S(harmonic-mean tensor) + γ diag(M_H) (bd/precond.py:34-47);
    assembly="device" assembles the stiffness on the GPU."""
    if gamma <= 0:
        raise ValueError("gamma must be strictly positive")
    if assembly == "device":
        from .assembly import device_assembler
        da = device_assembler(mesh, params, fibers)
        stiff, mass = da.stiffness("mono"), da.lumped_mass(Space.HEART_ONLY)
    elif assembly == "host":
        stiff = assemble_stiffness(mesh, TensorField(params, mesh.dim, "mono", fibers),
                                   Space.HEART_ONLY)
        mass = lumped_mass_diagonal(mesh, Space.HEART_ONLY)
    else:
        raise ValueError(f"unknown assembly mode {assembly!r}")
    out = (stiff + gamma * sp.diags(mass)).tocsr()
    out.sum_duplicates()
    out.sort_indices()
    return out


@dataclass
class RegularizedStiffness:
    """S_1 + (β/n) 𝟙𝟙ᵀ, solved through the grounded matrix plus mean
    projections (bd/precond.py:50-76)."""

    base: sp.csr_matrix
    beta: float

    @property
    def n(self) -> int:
        return self.base.shape[0]

    def matvec(self, x):
        x = np.asarray(x, dtype=float)
        return self.base @ x + self.beta * x.mean()

    def grounded(self) -> sp.csr_matrix:
        bump = sp.csr_matrix(([self.beta], ([0], [0])), shape=self.base.shape)
        out = (self.base + bump).tocsr()
        out.sort_indices()
        return out


def regularize_stiffness(stiff: sp.csr_matrix) -> RegularizedStiffness:
    return RegularizedStiffness(sp.csr_matrix(stiff), float(stiff.diagonal().mean()))


class InnerPreconditioner(ABC):
    """setup(SPD sparse) then a linear, symmetric, positive apply_inverse."""

    @abstractmethod
    def setup(self, matrix) -> None:
        ...

    @abstractmethod
    def apply_inverse(self, y):
        ...


class NativeInner(InnerPreconditioner):
    """Inner preconditioner living in the sm_100a library."""

    kind = None
    max_restarts = 0

    def __init__(self):
        self.handle = None
        self.ctx = None
        self.n = 0
        self.restarts_used = 0

    def setup(self, matrix, coords=None) -> None:
        """Factor on the host (C++) and upload.  ``coords`` (n×dim vertex
        coordinates, optional) only steer the row partition of the tiled
        triangular-solve schedule; the factor does not depend on them."""
        a = sp.csr_matrix(matrix, dtype=float)
        a.sum_duplicates()
        a.sort_indices()
        if a.shape[0] != a.shape[1]:
            raise ValueError("inner preconditioner needs a square matrix")
        self.release()
        ctx = _lib.Context.default()
        ip, ix, dv = csr_arrays(a)
        h = C.c_void_p()
        used = C.c_int(0)
        xyz, dim = None, 0
        if coords is not None:
            xyz = np.ascontiguousarray(coords, dtype=np.float64)
            if xyz.ndim != 2 or xyz.shape[0] != a.shape[0]:
                raise ValueError("coords must be (n, dim)")
            dim = xyz.shape[1]
        _lib.check(_lib.lib().bd_inner_create_ex(
            ctx.handle, _lib.INNER_KIND[self.kind], a.shape[0], ip.ctypes.data_as(C.c_void_p),
            ix.ctypes.data_as(C.c_void_p), dv.ctypes.data_as(C.c_void_p), int(self.max_restarts),
            xyz.ctypes.data_as(C.c_void_p) if xyz is not None else None, dim, C.byref(h),
            C.byref(used)), ctx.handle)
        self.handle, self.ctx, self.n = h, ctx, a.shape[0]
        self.restarts_used = int(used.value)

    def apply_inverse(self, y):
        """z = P⁻¹ y on the device; returns a CUDA tensor (numpy in → numpy out)."""
        if self.handle is None:
            raise PreconditionerError("inner preconditioner used before setup")
        is_np = not isinstance(y, _torch().Tensor)
        yd = as_device(y, self.ctx)
        if tuple(yd.shape) != (self.n,):
            raise ValueError(f"vector length {tuple(yd.shape)} does not match {self.n}")
        z = _torch().empty_like(yd)
        _lib.check(_lib.lib().bd_inner_apply(self.handle, _lib.ptr(yd), _lib.ptr(z)),
                   self.ctx.handle)
        return z.cpu().numpy() if is_np else z

    def factor_info(self):
        n, nnz, lv = C.c_int64(), C.c_int64(), C.c_int64()
        _lib.check(_lib.lib().bd_inner_factor_info(self.handle, C.byref(n), C.byref(nnz),
                                                   C.byref(lv)), self.ctx.handle)
        return {"n": n.value, "nnz": nnz.value, "levels": lv.value}

    def _export(self):
        info = self.factor_info()
        n, nnz = info["n"], info["nnz"]
        ip = np.empty(n + 1, dtype=np.int64)
        ix = np.empty(nnz, dtype=np.int32)
        dv = np.empty(nnz, dtype=np.float64)
        perm = np.empty(n, dtype=np.int32)
        _lib.check(_lib.lib().bd_inner_export_factor(
            self.handle, ip.ctypes.data_as(C.c_void_p), ix.ctypes.data_as(C.c_void_p),
            dv.ctypes.data_as(C.c_void_p), perm.ctypes.data_as(C.c_void_p)), self.ctx.handle)
        return sp.csr_matrix((dv, ix, ip), shape=(n, n)), perm

    def release(self):
        if self.handle is not None and _lib._lib is not None:
            _lib._lib.bd_inner_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class ExactFactorization(NativeInner):
    """Sparse Cholesky LLᵀ with a nested-dissection ordering (stands in for
    CHOLMOD, bd/precond.py:96-120); solves to machine precision."""

    kind = "exact"

    @property
    def factor(self):
        return self._export()


class IncompleteCholesky0(NativeInner):
    """Zero-fill IC on the matrix pattern with (1+1e-3)^k diagonal restarts;
    the factor is bit-identical to the reference's (bd/precond.py:123-198)."""

    kind = "ic0"

    def __init__(self, max_restarts: int = 20):
        super().__init__()
        self.max_restarts = max_restarts

    @property
    def lower_factor(self) -> sp.csr_matrix:
        return self._export()[0]


class Jacobi(NativeInner):
    """Diagonal preconditioner (bd/precond.py:219-232)."""

    kind = "jacobi"


def make_inner(name: str) -> InnerPreconditioner:
    if name == "exact":
        return ExactFactorization()
    if name == "ic0":
        return IncompleteCholesky0()
    if name == "jacobi":
        return Jacobi()
    raise ValueError(f"unknown inner preconditioner {name!r}; choose one of {INNER_NAMES}")


def _coords(system):
    """Vertex coordinates for the solve-schedule partition, when known."""
    pts = getattr(system, "coords", None)
    if pts is None and getattr(system, "mesh", None) is not None:
        pts = system.mesh.vertices
    if pts is None or len(pts) != system.n:
        return None
    return np.asarray(pts, dtype=float)


class BlockLUPreconditioner:
    """P_Λ = L_P U_P with the monodomain K_m in the Schur slot
    (bd/precond.py:246-312).  One application = two bulk inverses, one K_m
    inverse and two S_i products, all on the device."""

    def __init__(self, system: BidomainSystem, inner: str = "exact",
                 monodomain_matrix: sp.csr_matrix | None = None):
        if inner not in INNER_NAMES:
            raise ValueError(f"unknown inner preconditioner {inner!r}; choose one of {INNER_NAMES}")
        self.system = system
        self.inner_name = inner
        self.regularized = regularize_stiffness(system.stiff_total)
        coords = _coords(system)
        # the two inner factorisations are independent host work (the C setup
        # releases the GIL): the bulk one runs on a worker thread while the
        # Schur block is built and factored here; a bulk error still wins
        self.inner_bulk = make_inner(inner)
        grounded = self.regularized.grounded()
        _lib.Context.default()  # one shared context, created here before the worker starts
        with ThreadPoolExecutor(max_workers=1) as pool:
            bulk = pool.submit(self.inner_bulk.setup, grounded, coords=coords)
            schur_err = None
            try:
                if monodomain_matrix is None:
                    if system.mesh is None or system.params is None:
                        raise PreconditionerError(
                            "system carries no mesh/params; pass monodomain_matrix")
                    monodomain_matrix = build_monodomain_matrix(
                        system.mesh, system.params, system.gamma, getattr(system, "fibers", None))
                self.inner_schur = make_inner(inner)
                self.inner_schur.setup(monodomain_matrix,
                                       coords=None if coords is None else coords[: system.n_heart])
            except Exception as exc:  # reported after the bulk result
                schur_err = exc
            bulk.result()
            if schur_err is not None:
                raise schur_err
        self.monodomain_matrix = monodomain_matrix
        nat = system.native
        h = C.c_void_p()
        _lib.check(_lib.lib().bd_blocklu_create(nat.handle, self.inner_bulk.handle,
                                                self.inner_schur.handle, self.regularized.beta,
                                                C.byref(h)), nat.ctx.handle)
        self.handle = h
        self.ctx = nat.ctx

    # -- counters (bd/precond.py:272-279) ----------------------------------------
    # The device counts applications inside the captured PCG loop; the
    # reference's counters are plain assignable attributes, so an assignment
    # is kept as a host-side offset on top of the device count.
    def _counters(self):
        buf = (C.c_int64 * 3)()
        _lib.check(_lib.lib().bd_blocklu_counters(self.handle, buf), self.ctx.handle)
        off = self.__dict__.get("_count_off", (0, 0, 0))
        return [int(b) + o for b, o in zip(buf, off)]

    def _set_counter(self, i: int, value: int) -> None:
        cur = self._counters()
        off = list(self.__dict__.get("_count_off", (0, 0, 0)))
        off[i] += int(value) - cur[i]
        self._count_off = tuple(off)

    @property
    def p1_count(self) -> int:
        return self._counters()[0]

    @p1_count.setter
    def p1_count(self, value: int) -> None:
        self._set_counter(0, value)

    @property
    def pk_count(self) -> int:
        return self._counters()[1]

    @pk_count.setter
    def pk_count(self, value: int) -> None:
        self._set_counter(1, value)

    @property
    def si_count(self) -> int:
        return self._counters()[2]

    @si_count.setter
    def si_count(self, value: int) -> None:
        self._set_counter(2, value)

    def reset_counters(self) -> None:
        _lib.check(_lib.lib().bd_blocklu_reset_counters(self.handle), self.ctx.handle)
        self._count_off = (0, 0, 0)

    # -- applications ----------------------------------------------------------------
    def _bulk_inverse(self, y):
        is_np = not isinstance(y, _torch().Tensor)
        yd = as_device(y, self.ctx)
        if tuple(yd.shape) != (self.system.n,):
            raise ValueError("vector does not match the bulk size")
        z = _torch().empty_like(yd)
        _lib.check(_lib.lib().bd_blocklu_bulk_inverse(self.handle, _lib.ptr(yd), _lib.ptr(z)),
                   self.ctx.handle)
        return z.cpu().numpy() if is_np else z

    def _schur_inverse(self, y):
        is_np = not isinstance(y, _torch().Tensor)
        yd = as_device(y, self.ctx)
        if tuple(yd.shape) != (self.system.n_heart,):
            raise ValueError("vector does not match the heart size")
        z = _torch().empty_like(yd)
        _lib.check(_lib.lib().bd_blocklu_schur_inverse(self.handle, _lib.ptr(yd), _lib.ptr(z)),
                   self.ctx.handle)
        return z.cpu().numpy() if is_np else z

    def apply_inverse(self, rhs) -> BlockVector:
        rhs = _as_block(rhs)
        if rhs.n != self.system.n or rhs.m != self.system.n_heart:
            raise ValueError("block vector does not match system sizes")
        out = _torch().empty_like(rhs.buf)
        _lib.check(_lib.lib().bd_blocklu_apply(self.handle, _lib.ptr(rhs.buf), _lib.ptr(out)),
                   self.ctx.handle)
        return BlockVector.from_buffer(out, rhs.n)

    def __del__(self):
        try:
            if _lib._lib is not None and getattr(self, "handle", None):
                _lib._lib.bd_blocklu_destroy(self.handle)
        except Exception:
            pass
