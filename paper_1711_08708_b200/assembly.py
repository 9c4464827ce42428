"""P1 stiffness and lumped mass (host setup, numpy/scipy).

Same discretisation as the reference (`bd/assembly.py:36-97`): per element
vol · G σ Gᵀ with σ at the centroid, local matrices symmetrised, COO → CSR
with duplicates summed and indices sorted; row-sum-lumped mass.  Elements are
processed in chunks so the 6.3M-tet (config 2) and 50M-tet (config 3) meshes
assemble in bounded memory; meshes below one chunk reproduce the reference's
arrays exactly.
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
