"""P1 stiffness and lumped mass (host setup, numpy/scipy).

Same discretisation as the reference (`bd/assembly.py:36-97`): per element
vol · G σ Gᵀ with σ at the centroid, local matrices symmetrised, COO → CSR
with duplicates summed and indices sorted; row-sum-lumped mass.  Elements are
processed in chunks so the 6.3M-tet (config 2) and 50M-tet (config 3) meshes
assemble in bounded memory; meshes below one chunk reproduce the reference's
arrays exactly.

`DeviceAssembler` is the same discretisation on the GPU (`bd_assemble_p1`,
csrc/bd_assembly.cuh): the element tensors are formed once
on the host, local matrices / gradients / harmonic means and the
COO -> CSR reduction (stable radix sort, sequential per-entry sums in element
order) run on the device.  Entries agree with the host path to rounding
(different summation order); entries whose contributions cancel in exact
arithmetic are stored as exactly 0.0, as the host sum gives them, so the
zero-dropping CSR adds downstream (grounding, K_m) produce the host's IC(0)
patterns.  The lumped mass is summed in the reference order.
"""
from __future__ import annotations

import math
from enum import Enum

import numpy as np
import scipy.sparse as sp

from .conductivity import TensorField
from .errors import AssemblyError
from .mesh import Mesh, Region

CHUNK = 1 << 21  # elements per assembly chunk


class Space(Enum):
    FULL = "full"
    HEART_ONLY = "heart_only"


def _select(mesh: Mesh, space: Space):
    if space == Space.HEART_ONLY:
        mask = mesh.tags == Region.HEART
        return mesh.elements[mask], mesh.tags[mask], mesh.heart_vertex_count
    return mesh.elements, mesh.tags, mesh.vertex_count


def _grads_volumes(vertices: np.ndarray, elements: np.ndarray, dim: int):
    coords = vertices[elements]
    edges = coords[:, 1:, :] - coords[:, :1, :]
    det = np.linalg.det(edges)
    if not (det > 0).all():
        raise AssemblyError("degenerate element (non-positive volume)")
    tail = np.linalg.inv(edges).transpose(0, 2, 1)
    g0 = -tail.sum(axis=1, keepdims=True)
    return np.concatenate([g0, tail], axis=1), det / math.factorial(dim)


def assemble_stiffness(mesh: Mesh, field: TensorField, space: Space = Space.FULL) -> sp.csr_matrix:
    """Symmetric PSD stiffness with the constants in its kernel."""
    elements, tags, n = _select(mesh, space)
    arity = mesh.dim + 1
    total = None
    for s in range(0, max(len(elements), 1), CHUNK):
        el = elements[s:s + CHUNK]
        if len(el) == 0:
            break
        grads, vols = _grads_volumes(mesh.vertices, el, mesh.dim)
        sigma = field.evaluate_batch(mesh.vertices[el].mean(axis=1), tags[s:s + CHUNK])
        local = np.einsum("eid,edk,ejk->eij", grads, sigma, grads)
        local = 0.5 * (local + local.transpose(0, 2, 1))
        local *= vols[:, None, None]
        rows = np.repeat(el, arity, axis=1).ravel()
        cols = np.tile(el, (1, arity)).ravel()
        part = sp.coo_matrix((local.ravel(), (rows, cols)), shape=(n, n)).tocsr()
        part.sum_duplicates()
        total = part if total is None else (total + part)
    if total is None:
        total = sp.csr_matrix((n, n))
    total = total.tocsr()
    total.sum_duplicates()
    total.sort_indices()
    return total


def lumped_mass_diagonal(mesh: Mesh, space: Space = Space.FULL) -> np.ndarray:
    """Vertex i gets Σ |element|/(d+1) over its elements (bd/assembly.py:79-97)."""
    elements, _, n = _select(mesh, space)
    diag = np.zeros(n)
    for s in range(0, len(elements), CHUNK):
        el = elements[s:s + CHUNK]
        coords = mesh.vertices[el]
        det = np.linalg.det(coords[:, 1:, :] - coords[:, :1, :])
        if not (det > 0).all():
            raise AssemblyError("degenerate element (non-positive volume)")
        share = det / math.factorial(mesh.dim) / (mesh.dim + 1)
        for k in range(mesh.dim + 1):
            np.add.at(diag, el[:, k], share)
    return diag


def assemble_lumped_mass(mesh: Mesh, space: Space = Space.FULL) -> sp.csr_matrix:
    return sp.csr_matrix(sp.diags(lumped_mass_diagonal(mesh, space)))


class DeviceAssembler:
    """All blocks of one (mesh, params, fibres) on the GPU: S_1 (bar1), S_i
    (intra, heart), S_e (bar_e), K_m stiffness (harmonic mean, heart) and the
    two lumped masses.  Heart tensors are evaluated once on the host."""

    def __init__(self, mesh: Mesh, field_params, fibers=None):
        from . import _lib

        self._lib = _lib
        self.ctx = _lib.Context.default()
        self.mesh = mesh
        d = mesh.dim
        self.heart = mesh.tags == Region.HEART
        self.verts = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
        self.el = np.ascontiguousarray(mesh.elements, dtype=np.int64)
        self.el_h = np.ascontiguousarray(self.el[self.heart])
        self.intra, self.extra = self._heart_tensors(field_params, fibers)
        self.params = field_params
        self._mass = {}

    def _heart_tensors(self, p, fibers):
        """(σ_i, σ_e) per heart element: on the device for the transmural
        rotation of configs 2/3 (`bd_tensors_transmural`), else the host
        TensorField evaluation."""
        from .conductivity import TransmuralRotation

        d = self.mesh.dim
        if isinstance(fibers, TransmuralRotation) and d == 3:
            import ctypes as C
            L = self._lib
            ne = self.el_h.shape[0]
            oi = np.empty((ne, 3, 3))
            oe = np.empty((ne, 3, 3))
            if p.orthotropic:
                gi = [p.g_i_l, p.g_i_t, p.g_i_n if p.g_i_n is not None else p.g_i_t]
                ge = [p.g_e_l, p.g_e_t, p.g_e_n if p.g_e_n is not None else p.g_e_t]
            else:
                gi, ge = [p.g_i_l, p.g_i_t, 0.0], [p.g_e_l, p.g_e_t, 0.0]
            arr = lambda v: (C.c_double * len(v))(*[float(x) for x in v])  # noqa: E731
            model = arr([fibers.z0, fibers.z1, fibers.angle0, fibers.angle1])
            L.check(L.lib().bd_tensors_transmural(
                self.ctx.handle, self.verts.shape[0], self.verts.ctypes.data, ne,
                self.el_h.ctypes.data, model, arr(gi), arr(ge), int(bool(p.orthotropic)),
                oi.ctypes.data, oe.ctypes.data), self.ctx.handle)
            return oi, oe
        tf = TensorField(p, d, "bar1", fibers)
        cent = self.verts[self.el_h].mean(axis=1)
        return tuple(np.ascontiguousarray(a, dtype=np.float64) for a in tf._heart_tensors(cent))

    def _torso(self, base: np.ndarray) -> np.ndarray:
        """Full-element tensor array: heart rows from `base`, torso c·I."""
        d = self.mesh.dim
        out = np.zeros((self.el.shape[0], d, d))
        out[self.heart] = base
        known = self.heart.copy()
        for t in (Region.TORSO_LUNG, Region.TORSO_CAVITY, Region.TORSO_OTHER):
            mask = self.mesh.tags == t
            if mask.any():
                out[mask] = self.params.torso_conductivity(t) * np.eye(d)
            known |= mask
        if not known.all():
            raise ValueError("unknown region tag in mesh")
        return out

    def _run(self, el, nv, sigma, sigma2=None, space=Space.FULL):
        L = self._lib
        C = __import__("ctypes")
        h = C.c_void_p()
        nnz = C.c_int64()
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        s2 = None if sigma2 is None else np.ascontiguousarray(sigma2, dtype=np.float64)
        st = L.lib().bd_assemble_p1(self.ctx.handle, self.mesh.dim, int(nv), self.verts.ctypes.data,
                                    int(el.shape[0]), el.ctypes.data, sigma.ctypes.data,
                                    None if s2 is None else s2.ctypes.data, C.byref(h),
                                    C.byref(nnz))
        if st == L.BD_EINVAL:
            raise AssemblyError(L.lib().bd_last_error(self.ctx.handle).decode())
        L.check(st, self.ctx.handle)
        try:
            n = int(nnz.value)
            indptr = np.empty(nv + 1, dtype=np.int64)
            indices = np.empty(n, dtype=np.int32)
            data = np.empty(n, dtype=np.float64)
            mass = np.empty(nv, dtype=np.float64)
            L.check(L.lib().bd_assemble_export(h, indptr.ctypes.data, indices.ctypes.data,
                                               data.ctypes.data, mass.ctypes.data),
                    self.ctx.handle)
        finally:
            L.lib().bd_assemble_destroy(h)
        self._mass.setdefault(space, mass)
        return sp.csr_matrix((data, indices, indptr), shape=(nv, nv)), mass

    def stiffness(self, kind: str) -> sp.csr_matrix:
        n, m = self.mesh.vertex_count, self.mesh.heart_vertex_count
        if kind == "bar1":
            return self._run(self.el, n, self._torso(self.intra + self.extra))[0]
        if kind == "bar_e":
            return self._run(self.el, n, self._torso(self.extra))[0]
        if kind == "intra":
            return self._run(self.el_h, m, self.intra, space=Space.HEART_ONLY)[0]
        if kind == "mono":
            return self._run(self.el_h, m, self.intra, self.extra, space=Space.HEART_ONLY)[0]
        raise ValueError(f"unknown tensor field kind {kind!r}")

    def lumped_mass(self, space: Space = Space.FULL) -> np.ndarray:
        if space not in self._mass:
            self.stiffness("bar1" if space == Space.FULL else "intra")
        return self._mass[space]


_DEV_CACHE: dict = {}


def device_assembler(mesh: Mesh, params, fibers=None) -> DeviceAssembler:
    """One cached DeviceAssembler per (mesh, params, fibres) (the system and
    the monodomain matrix share the heart tensors)."""
    key = (id(mesh), id(params), id(fibers))
    a = _DEV_CACHE.get("last")
    if a is None or a[0] != key:
        _DEV_CACHE["last"] = (key, DeviceAssembler(mesh, params, fibers))
    return _DEV_CACHE["last"][1]
