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
(different summation order).  Entries whose contributions cancel in exact
arithmetic (0.2% at config 2) then take the host sum's value bit for bit
(`reference_order_values`: exact zero or rounding residue), so the
zero-dropping CSR adds downstream (grounding, K_m) produce the reference's
IC(0) patterns.  The lumped mass is summed in the
reference order.
"""
from __future__ import annotations

import math
import os
from enum import Enum

import numpy as np
import scipy.sparse as sp

from .conductivity import TensorField
from .errors import AssemblyError
from .mesh import Mesh, Region

CHUNK = 1 << 21  # elements per assembly chunk
# |entry| <= REF_ZERO_REL * |row diagonal|: an exact-arithmetic cancellation
# (measured: those are <= 1e-17 of the diagonal, all others >= 1e-6)
REF_ZERO_REL = 1e-10


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


def reference_order_values(mesh: Mesh, field: TensorField, space: Space, rows: np.ndarray,
                           cols: np.ndarray) -> np.ndarray:
    """The host assembly's value of the entries (rows[k], cols[k]), bit for bit,
    without assembling the whole matrix.

    Entries whose element contributions cancel in exact arithmetic come out of
    the reference's floating-point sum either as exactly 0.0 or as a rounding
    residue (~1e-32), depending on the last bits of each contribution and on
    the summation order; the zero-dropping CSR adds downstream (grounding,
    K_m: bd/precond.py:44-46, 72-75) then remove the zeros and keep the
    residues, so the IC(0) pattern depends on it.  This recomputes such
    entries exactly as `assemble_stiffness` does: the same numpy element
    arithmetic on the elements incident to the rows, and per chunk a COO ->
    CSR sum of each row's complete entry sequence in the original element
    order (so scipy's per-row sort permutes it exactly as in the full
    matrix), chunks added in order."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if rows.size == 0:
        return np.zeros(0)
    elements, tags, n = _select(mesh, space)
    arity = mesh.dim + 1
    want = np.zeros(n, dtype=bool)
    want[np.unique(rows)] = True
    total = None
    for s in range(0, len(elements), CHUNK):
        el_all = elements[s:s + CHUNK]
        hit = want[el_all].any(axis=1)
        if not hit.any():
            continue
        el = el_all[hit]
        grads, vols = _grads_volumes(mesh.vertices, el, mesh.dim)
        sigma = field.evaluate_batch(mesh.vertices[el].mean(axis=1), tags[s:s + CHUNK][hit])
        local = np.einsum("eid,edk,ejk->eij", grads, sigma, grads)
        local = 0.5 * (local + local.transpose(0, 2, 1))
        local *= vols[:, None, None]
        r = np.repeat(el, arity, axis=1).ravel()
        c = np.tile(el, (1, arity)).ravel()
        keep = want[r]  # complete rows only, in the original entry order
        part = sp.coo_matrix((local.ravel()[keep], (r[keep], c[keep])), shape=(n, n)).tocsr()
        part.sum_duplicates()
        total = part if total is None else (total + part)
    total = total.tocsr()
    total.sum_duplicates()
    total.sort_indices()
    return np.asarray(total[rows, cols]).ravel()


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
        self.fibers = fibers
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
        """Assemble on the device.  Meshes whose (element, local pair) keys
        exceed BD_ASSEMBLY_MAX_PAIRS (default 6e8, ~25 GB of device scratch)
        are assembled in row blocks: each block's rows from the elements that
        touch them (a local mesh), the same per-entry element order as one
        pass, so the result is identical."""
        arity = self.mesh.dim + 1
        max_pairs = float(os.environ.get("BD_ASSEMBLY_MAX_PAIRS", "6e8"))
        if el.shape[0] * arity * arity > max_pairs:
            return self._run_blocks(el, nv, sigma, sigma2, space, max_pairs)
        return self._run_one(self.verts, el, nv, sigma, sigma2, space)

    def _run_blocks(self, el, nv, sigma, sigma2, space, max_pairs):
        arity = self.mesh.dim + 1
        nblk = int(np.ceil(2.0 * el.shape[0] * arity * arity / max_pairs))
        bounds = np.linspace(0, nv, nblk + 1).astype(np.int64)
        ips, ixs, dvs, masses = [np.zeros(1, dtype=np.int64)], [], [], []
        off = 0
        for r0, r1 in zip(bounds[:-1], bounds[1:]):
            if r1 <= r0:
                continue
            touch = ((el >= r0) & (el < r1)).any(axis=1)
            sub = el[touch]
            lv = np.unique(sub)
            loc = np.ascontiguousarray(np.searchsorted(lv, sub), dtype=np.int64)
            s1 = np.ascontiguousarray(sigma[touch])
            s2 = None if sigma2 is None else np.ascontiguousarray(sigma2[touch])
            a, mass = self._run_one(np.ascontiguousarray(self.verts[lv]), loc, lv.size, s1, s2,
                                    None)
            i0, i1 = np.searchsorted(lv, r0), np.searchsorted(lv, r1)
            rows = a[i0:i1]
            ips.append(rows.indptr[1:].astype(np.int64) + off)
            off += rows.nnz
            ixs.append(lv[rows.indices].astype(np.int32))
            dvs.append(rows.data)
            masses.append(mass[i0:i1])
            del a, rows, touch, sub, loc, s1, s2
        mat = sp.csr_matrix((np.concatenate(dvs), np.concatenate(ixs), np.concatenate(ips)),
                            shape=(nv, nv))
        mass = np.concatenate(masses)
        self._mass.setdefault(space, mass)
        return mat, mass

    def _run_one(self, verts, el, nv, sigma, sigma2=None, space=Space.FULL):
        L = self._lib
        C = __import__("ctypes")
        h = C.c_void_p()
        nnz = C.c_int64()
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        s2 = None if sigma2 is None else np.ascontiguousarray(sigma2, dtype=np.float64)
        st = L.lib().bd_assemble_p1(self.ctx.handle, self.mesh.dim, int(nv), verts.ctypes.data,
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
        if space is not None:
            self._mass.setdefault(space, mass)
        return sp.csr_matrix((data, indices, indptr), shape=(nv, nv)), mass

    def stiffness(self, kind: str) -> sp.csr_matrix:
        n, m = self.mesh.vertex_count, self.mesh.heart_vertex_count
        if kind == "bar1":
            mat = self._run(self.el, n, self._torso(self.intra + self.extra))[0]
            space = Space.FULL
        elif kind == "bar_e":
            mat = self._run(self.el, n, self._torso(self.extra))[0]
            space = Space.FULL
        elif kind == "intra":
            mat = self._run(self.el_h, m, self.intra, space=Space.HEART_ONLY)[0]
            space = Space.HEART_ONLY
        elif kind == "mono":
            mat = self._run(self.el_h, m, self.intra, self.extra, space=Space.HEART_ONLY)[0]
            space = Space.HEART_ONLY
        else:
            raise ValueError(f"unknown tensor field kind {kind!r}")
        return self._reference_zeros(mat, kind, space)

    def _reference_zeros(self, mat: sp.csr_matrix, kind: str, space: Space) -> sp.csr_matrix:
        """Entries whose element contributions cancel in exact arithmetic.

        The device sums them in another order than the reference, so they
        come out as different rounding residues (|s| <= 1e-17 of the row's
        diagonal; every other entry is >= 1e-6 of it, tools/hostcheck/
        zero_pattern.py).  In the reference's own sum such an entry is either
        exactly 0.0 or a residue, and its zero-dropping CSR adds (grounding,
        K_m: bd/precond.py:44-46, 72-75) keep the residues in the IC(0)
        pattern, so they change the preconditioner.  Hence (BD_ASSEMBLY_REFZEROS):
          "1" (default): they take the host assembly's value bit for bit
              (`reference_order_values`); config 2/3 meshes have 0.2% of them,
              all exact zeros in the reference; the isotropic torso of config 4
              has residues on most of its rows, so there this costs about a
              host assembly of the torso;
          "snap": set to exactly 0.0 (the exact-arithmetic value);
          "0": the raw device sums."""
        mode = os.environ.get("BD_ASSEMBLY_REFZEROS", "1")
        if mode == "0" or mat.nnz == 0:
            return mat
        rows = np.repeat(np.arange(mat.shape[0], dtype=np.int64), np.diff(mat.indptr))
        diag = np.abs(mat.diagonal())
        pos = np.flatnonzero(np.abs(mat.data) <= REF_ZERO_REL * diag[rows])
        if pos.size == 0:
            return mat
        if mode == "snap":
            mat.data[pos] = 0.0
            return mat
        field = TensorField(self.params, self.mesh.dim, kind, self.fibers)
        mat.data[pos] = reference_order_values(self.mesh, field, space, rows[pos],
                                               mat.indices[pos].astype(np.int64))
        return mat

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
