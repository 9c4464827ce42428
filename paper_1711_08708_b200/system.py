"""The coupled 2×2 block operator Λ on the device (drop-in for bd/system.py).

``BidomainSystem`` keeps the reference's constructor and attributes (host scipy
CSR blocks, mass diagonals, γ, optional mesh/params) and lazily uploads S_1 and
S_i to the sm_100a library; ``apply`` / ``normalize`` / ``weighted_mean_u``
run there.  ``BlockVector`` is one contiguous fp64 CUDA buffer [u | v] with
``u`` / ``v`` views, so every PCG kernel streams a single array.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.sparse as sp

from . import _lib
from .assembly import Space, assemble_stiffness, lumped_mass_diagonal
from .conductivity import ConductivityParams, TensorField
from .mesh import Mesh


def gamma(chi: float, c_m: float, dt: float) -> float:
    """γ = χ c_m / dt (bd/system.py:22-26)."""
    if chi <= 0 or c_m <= 0 or dt <= 0:
        raise ValueError("chi, c_m and dt must be strictly positive")
    return chi * c_m / dt


def _torch():
    import torch

    return torch


def as_device(a, ctx: "_lib.Context | None" = None):
    """fp64 contiguous CUDA tensor view/copy of a numpy array or tensor."""
    torch = _torch()
    ctx = ctx or _lib.Context.default()
    if isinstance(a, torch.Tensor):
        t = a.to(device=ctx.device, dtype=torch.float64)
        return t.contiguous()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(ctx.device)


class BlockVector:
    """(u ∈ Rⁿ, v ∈ Rᵐ) stored as one device buffer (bd/system.py:29-47)."""

    __slots__ = ("buf", "n", "m")

    def __init__(self, u, v):
        torch = _torch()
        ud, vd = as_device(u), as_device(v)
        if ud.dim() != 1 or vd.dim() != 1:
            raise ValueError("block vector components must be 1-D")
        self.n, self.m = int(ud.shape[0]), int(vd.shape[0])
        self.buf = torch.cat([ud, vd])

    @classmethod
    def from_buffer(cls, buf, n: int) -> "BlockVector":
        out = cls.__new__(cls)
        out.buf = buf
        out.n = n
        out.m = int(buf.shape[0]) - n
        return out

    @classmethod
    def zeros(cls, n: int, n_heart: int) -> "BlockVector":
        torch = _torch()
        buf = torch.zeros(n + n_heart, dtype=torch.float64, device=_lib.Context.default().device)
        return cls.from_buffer(buf, n)

    @property
    def u(self):
        return self.buf[: self.n]

    @u.setter
    def u(self, value):
        self.buf[: self.n] = as_device(value)

    @property
    def v(self):
        return self.buf[self.n:]

    @v.setter
    def v(self, value):
        self.buf[self.n:] = as_device(value)

    def copy(self) -> "BlockVector":
        return BlockVector.from_buffer(self.buf.clone(), self.n)

    def dot(self, other: "BlockVector") -> float:
        """u·u' + v·v' as one fixed-order device reduction."""
        ctx = _lib.Context.default()
        out = C.c_double()
        _lib.check(_lib.lib().bd_dot(ctx.handle, self.buf.numel(), _lib.ptr(self.buf),
                                     _lib.ptr(other.buf), C.byref(out)), ctx.handle)
        return float(out.value)

    def norm(self) -> float:
        return float(np.sqrt(self.dot(self)))

    def numpy(self):
        b = self.buf.cpu().numpy()
        return b[: self.n].copy(), b[self.n:].copy()


class BidomainSystem:
    """Assembled blocks of the per-step operator (bd/system.py:50-150)."""

    def __init__(self, stiff_total, stiff_intra, stiff_extra, mass_diag, heart_mass_diag,
                 gamma, mesh: Mesh | None = None, params: ConductivityParams | None = None,
                 fibers=None):
        self.stiff_total = sp.csr_matrix(stiff_total)
        self.stiff_intra = sp.csr_matrix(stiff_intra)
        self.stiff_extra = sp.csr_matrix(stiff_extra) if stiff_extra is not None else None
        self.mass_diag = np.asarray(mass_diag, dtype=float)
        self.heart_mass_diag = np.asarray(heart_mass_diag, dtype=float)
        self.gamma = float(gamma)
        self.mesh = mesh
        self.params = params
        self.fibers = fibers
        self.coords = None  # optional vertex coordinates (partition hint) when mesh is None
        self._native = None

    # -- reference properties -------------------------------------------------
    @property
    def n(self) -> int:
        return self.stiff_total.shape[0]

    @property
    def n_heart(self) -> int:
        return self.stiff_intra.shape[0]

    @property
    def dof(self) -> int:
        return self.n + self.n_heart

    @classmethod
    def build(cls, mesh: Mesh, params: ConductivityParams, dt: float, fibers=None,
              with_extra: bool = True, assembly: str = "host") -> "BidomainSystem":
        """Assemble all blocks for time step dt (bd/system.py:82-97).
        assembly="device" runs the P1 assembly on the GPU (DeviceAssembler)."""
        d = mesh.dim
        if assembly == "device":
            from .assembly import device_assembler
            da = device_assembler(mesh, params, fibers)
            return cls(stiff_total=da.stiffness("bar1"), stiff_intra=da.stiffness("intra"),
                       stiff_extra=da.stiffness("bar_e") if with_extra else None,
                       mass_diag=da.lumped_mass(Space.FULL),
                       heart_mass_diag=da.lumped_mass(Space.HEART_ONLY),
                       gamma=gamma(params.chi, params.c_m, dt), mesh=mesh, params=params,
                       fibers=fibers)
        if assembly != "host":
            raise ValueError(f"unknown assembly mode {assembly!r}")
        return cls(
            stiff_total=assemble_stiffness(mesh, TensorField(params, d, "bar1", fibers)),
            stiff_intra=assemble_stiffness(mesh, TensorField(params, d, "intra", fibers),
                                           Space.HEART_ONLY),
            stiff_extra=(assemble_stiffness(mesh, TensorField(params, d, "bar_e", fibers))
                         if with_extra else None),
            mass_diag=lumped_mass_diagonal(mesh),
            heart_mass_diag=lumped_mass_diagonal(mesh, Space.HEART_ONLY),
            gamma=gamma(params.chi, params.c_m, dt),
            mesh=mesh, params=params, fibers=fibers,
        )

    # -- native handles ----------------------------------------------------------
    @property
    def native(self):
        if self._native is None:
            self._native = _NativeSystem(self)
        return self._native

    def _check(self, x: BlockVector) -> None:
        if x.n != self.n or x.m != self.n_heart:
            raise ValueError(f"block vector shapes ({x.n},)/({x.m},) do not match "
                             f"system sizes {self.n}/{self.n_heart}")

    def apply(self, x: BlockVector) -> BlockVector:
        """q = Λ x on the device (bd/system.py:106-116)."""
        x = _as_block(x)
        self._check(x)
        nat = self.native
        out = _torch().empty_like(x.buf)
        _lib.check(_lib.lib().bd_system_apply(nat.handle, _lib.ptr(x.buf), _lib.ptr(out)),
                   nat.ctx.handle)
        return BlockVector.from_buffer(out, self.n)

    def build_rhs(self, v_prev, ion_current, stim_current, chi: float) -> BlockVector:
        """(0ⁿ, M_H ∘ (γ v − χ (ion − stim))) (bd/system.py:118-136)."""
        nh = self.n_heart
        vs = []
        for name, vec in (("v_prev", v_prev), ("ion_current", ion_current),
                          ("stim_current", stim_current)):
            t = as_device(vec)
            if tuple(t.shape) != (nh,):
                raise ValueError(f"{name} must have length {nh}")
            vs.append(t)
        v, ion, stim = vs
        mh = self.native.mh
        load = self.gamma * v - chi * (ion - stim)
        torch = _torch()
        buf = torch.zeros(self.dof, dtype=torch.float64, device=v.device)
        buf[self.n:] = mh * load
        return BlockVector.from_buffer(buf, self.n)

    def normalize(self, x: BlockVector) -> BlockVector:
        """u − (M·u)/ΣM, v copied (bd/system.py:138-146)."""
        x = _as_block(x)
        self._check(x)
        nat = self.native
        out = _torch().empty_like(x.buf)
        _lib.check(_lib.lib().bd_system_normalize(nat.handle, _lib.ptr(x.buf), _lib.ptr(out)),
                   nat.ctx.handle)
        return BlockVector.from_buffer(out, self.n)

    def weighted_mean_u(self, u) -> float:
        nat = self.native
        ud = as_device(u)
        out = C.c_double()
        _lib.check(_lib.lib().bd_system_weighted_mean_u(nat.handle, _lib.ptr(ud), C.byref(out)),
                   nat.ctx.handle)
        return float(out.value)


def _as_block(x) -> BlockVector:
    if isinstance(x, BlockVector):
        return x
    return BlockVector(x.u, x.v)


def csr_arrays(a: sp.csr_matrix):
    """(indptr int64, indices int32, data float64), C-contiguous, for the ABI."""
    a = sp.csr_matrix(a)
    return (np.ascontiguousarray(a.indptr, dtype=np.int64),
            np.ascontiguousarray(a.indices, dtype=np.int32),
            np.ascontiguousarray(a.data, dtype=np.float64))


class NativeCsr:
    def __init__(self, ctx: "_lib.Context", a: sp.csr_matrix):
        self.ctx = ctx
        self.shape = a.shape
        ip, ix, dv = csr_arrays(a)
        h = C.c_void_p()
        _lib.check(_lib.lib().bd_csr_create(ctx.handle, a.shape[0], a.shape[1], int(ip[-1]),
                                            ip.ctypes.data_as(C.c_void_p),
                                            ix.ctypes.data_as(C.c_void_p),
                                            dv.ctypes.data_as(C.c_void_p), C.byref(h)),
                   ctx.handle)
        self.handle = h

    def matvec(self, x, y=None, alpha=1.0, beta=0.0):
        torch = _torch()
        xd = as_device(x, self.ctx)
        if y is None:
            y = torch.zeros(self.shape[0], dtype=torch.float64, device=xd.device)
        _lib.check(_lib.lib().bd_spmv(self.handle, _lib.ptr(xd), _lib.ptr(y), alpha, beta),
                   self.ctx.handle)
        return y

    def matvec_split(self, x, nsplit: int, x_ghost, y=None, alpha=1.0, beta=0.0):
        """y = alpha * A [x[:nsplit] ; x_ghost] + beta * y (bd_spmv_split)."""
        torch = _torch()
        if y is None:
            y = torch.zeros(self.shape[0], dtype=torch.float64, device=x.device)
        _lib.check(_lib.lib().bd_spmv_split(self.handle, _lib.ptr(x), int(nsplit), _lib.ptr(x_ghost),
                                            _lib.ptr(y), alpha, beta), self.ctx.handle)
        return y

    def __del__(self):
        try:
            if _lib._lib is not None and getattr(self, "handle", None):
                _lib._lib.bd_csr_destroy(self.handle)
        except Exception:
            pass


class _NativeSystem:
    def __init__(self, system: BidomainSystem):
        ctx = _lib.Context.default()
        self.ctx = ctx
        self.S1 = NativeCsr(ctx, system.stiff_total)
        self.Si = NativeCsr(ctx, system.stiff_intra)
        mass = np.ascontiguousarray(system.mass_diag, dtype=np.float64)
        mh = np.ascontiguousarray(system.heart_mass_diag, dtype=np.float64)
        if mass.shape != (system.n,) or mh.shape != (system.n_heart,):
            raise ValueError("mass diagonals do not match the stiffness blocks")
        h = C.c_void_p()
        _lib.check(_lib.lib().bd_system_create(ctx.handle, self.S1.handle, self.Si.handle,
                                               mass.ctypes.data_as(C.c_void_p),
                                               mh.ctypes.data_as(C.c_void_p), system.gamma,
                                               C.byref(h)), ctx.handle)
        self.handle = h
        self.mh = as_device(mh, ctx)
        self.mass = as_device(mass, ctx)

    def __del__(self):
        try:
            if _lib._lib is not None and getattr(self, "handle", None):
                _lib._lib.bd_system_destroy(self.handle)
        except Exception:
            pass
