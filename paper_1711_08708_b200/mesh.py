"""Structured simplicial meshes with a heart-first vertex ordering (host setup).

Same data model as the reference (`bd/mesh.py:20-126`): a ``Mesh`` holds
vertices, simplices, region tags and the heart vertex count; heart vertices
occupy indices ``0..N_H-1`` so restriction is truncation.  The builders are
vectorised (no per-element Python loops) so the BASELINE configurations
(up to 256×256×128 cells) can be generated on the host of the GPU box:

* ``build_cube_mesh`` / ``build_square_mesh`` / ``build_heart_torso_2d``
  reproduce the reference builders (`bd/mesh.py:142-267`) vertex for vertex
  and element for element;
* ``build_box_mesh`` generalises the Kuhn cube to an nx×ny×nz box of any
  extent (config 2/3 slab), ``build_ellipse_torso_2d`` is the config-1
  elliptical heart in a [0,20]² torso, ``build_ellipsoid_torso_3d`` the
  config-4 ventricular shell.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from .errors import AssemblyError


class Region(IntEnum):
    HEART = 0
    TORSO_LUNG = 1
    TORSO_CAVITY = 2
    TORSO_OTHER = 3


@dataclass(frozen=True)
class Mesh:
    """Simplicial mesh with a tagged, vertex-contiguous cardiac submesh."""

    dim: int
    vertices: np.ndarray
    elements: np.ndarray
    tags: np.ndarray
    heart_vertex_count: int

    @property
    def vertex_count(self) -> int:
        return int(self.vertices.shape[0])

    @property
    def heart_vertex_ids(self) -> np.ndarray:
        return np.arange(self.heart_vertex_count)

    def element_volumes(self) -> np.ndarray:
        coords = self.vertices[self.elements]
        edges = coords[:, 1:, :] - coords[:, :1, :]
        return np.linalg.det(edges) / math.factorial(self.dim)

    def element_centroids(self) -> np.ndarray:
        return self.vertices[self.elements].mean(axis=1)

    def heart_volume(self) -> float:
        return float(self.element_volumes()[self.tags == Region.HEART].sum())

    def restriction(self) -> "RestrictionMap":
        return RestrictionMap(self.vertex_count, self.heart_vertex_count)

    def validate(self) -> None:
        """Structural invariants (bd/mesh.py:70-86); AssemblyError on violation."""
        if self.dim not in (2, 3):
            raise AssemblyError(f"unsupported dimension {self.dim}")
        if self.elements.shape[1] != self.dim + 1:
            raise AssemblyError("element arity does not match dimension")
        srt = np.sort(self.elements, axis=1)
        if (np.diff(srt, axis=1) == 0).any():
            raise AssemblyError("element with repeated vertices")
        if not (self.element_volumes() > 0).all():
            raise AssemblyError("non-positive element volume")
        heart_el = self.elements[self.tags == Region.HEART]
        if heart_el.size and heart_el.max() >= self.heart_vertex_count:
            raise AssemblyError("heart element touches a non-heart vertex index")
        if np.unique(heart_el).size != self.heart_vertex_count:
            raise AssemblyError("heart vertex block is not contiguous")


@dataclass(frozen=True)
class RestrictionMap:
    """Truncation to the heart block and its transpose (zero padding)."""

    n: int
    n_heart: int

    def apply(self, full_vector):
        return restrict(self, full_vector)

    def transpose_apply(self, heart_vector):
        return transpose_restrict(self, heart_vector)


def restrict(rmap: RestrictionMap, full_vector):
    full_vector = np.asarray(full_vector)
    if full_vector.shape != (rmap.n,):
        raise ValueError(f"expected vector of length {rmap.n}, got {full_vector.shape}")
    return full_vector[: rmap.n_heart].copy()


def transpose_restrict(rmap: RestrictionMap, heart_vector):
    heart_vector = np.asarray(heart_vector)
    if heart_vector.shape != (rmap.n_heart,):
        raise ValueError(f"expected vector of length {rmap.n_heart}, got {heart_vector.shape}")
    out = np.zeros(rmap.n, dtype=heart_vector.dtype)
    out[: rmap.n_heart] = heart_vector
    return out


# Corner offsets of the six Kuhn tetrahedra of a cube (all walk (0,0,0) ->
# (1,1,1) along one axis order), in the reference's order (bd/mesh.py:132-139).
KUHN_PATHS = np.array([
    [(0, 0, 0), (1, 0, 0), (1, 1, 0), (1, 1, 1)],
    [(0, 0, 0), (1, 0, 0), (1, 0, 1), (1, 1, 1)],
    [(0, 0, 0), (0, 1, 0), (1, 1, 0), (1, 1, 1)],
    [(0, 0, 0), (0, 1, 0), (0, 1, 1), (1, 1, 1)],
    [(0, 0, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1)],
    [(0, 0, 0), (0, 0, 1), (0, 1, 1), (1, 1, 1)],
], dtype=np.int64)


def _kuhn_flip() -> np.ndarray:
    """Which Kuhn paths have negative orientation (swap the last two corners)."""
    p = KUHN_PATHS.astype(float)
    return np.linalg.det(p[:, 1:, :] - p[:, :1, :]) < 0


def box_grid(cells, lengths=(1.0, 1.0, 1.0)):
    """Vertices and Kuhn tets of an nx×ny×nz box, vid=(i*(ny+1)+j)*(nz+1)+k."""
    nx, ny, nz = (int(c) for c in cells)
    hx, hy, hz = (float(L) / c for L, c in zip(lengths, (nx, ny, nz)))
    ii, jj, kk = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1),
                             indexing="ij")
    vertices = np.column_stack([ii.ravel() * hx, jj.ravel() * hy, kk.ravel() * hz]).astype(float)
    ci, cj, ck = (a.ravel() for a in np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz),
                                                 indexing="ij"))
    sj, sk = (nz + 1), (ny + 1) * (nz + 1)
    base = ci * sk + cj * sj + ck  # vid of the cell's (0,0,0) corner
    off = KUHN_PATHS[..., 0] * sk + KUHN_PATHS[..., 1] * sj + KUHN_PATHS[..., 2]  # (6,4)
    elements = (base[:, None, None] + off[None, :, :]).reshape(-1, 4)
    flip = np.tile(_kuhn_flip(), base.size)
    elements[flip, 2], elements[flip, 3] = elements[flip, 3].copy(), elements[flip, 2].copy()
    cell_ijk = np.repeat(np.column_stack([ci, cj, ck]), 6, axis=0)
    return vertices, elements, cell_ijk


def rect_grid(cells, lengths=(1.0, 1.0)):
    """Vertices and two triangles per cell of an nx×ny grid, vid = j*(nx+1)+i
    (bd/mesh.py:188-209 layout)."""
    nx, ny = (int(c) for c in cells)
    hx, hy = (float(L) / c for L, c in zip(lengths, (nx, ny)))
    jj, ii = np.meshgrid(np.arange(ny + 1), np.arange(nx + 1), indexing="ij")
    vertices = np.column_stack([ii.ravel() * hx, jj.ravel() * hy]).astype(float)
    cj, ci = (a.ravel() for a in np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij"))
    v00 = cj * (nx + 1) + ci
    v10, v01, v11 = v00 + 1, v00 + (nx + 1), v00 + (nx + 2)
    elements = np.stack([np.column_stack([v00, v10, v11]), np.column_stack([v00, v11, v01])],
                        axis=1).reshape(-1, 3).astype(np.int64)
    cell_ij = np.repeat(np.column_stack([ci, cj]), 2, axis=0)
    return vertices, elements, cell_ij


def heart_first(dim, vertices, elements, tags) -> Mesh:
    """Permute vertices so the heart block comes first, preserving relative
    order (bd/mesh.py:252-263)."""
    mask = np.zeros(vertices.shape[0], dtype=bool)
    mask[np.unique(elements[tags == Region.HEART])] = True
    nh = int(mask.sum())
    new = np.empty(vertices.shape[0], dtype=np.int64)
    new[mask] = np.arange(nh)
    new[~mask] = nh + np.arange(vertices.shape[0] - nh)
    reordered = np.empty_like(vertices)
    reordered[new] = vertices
    return Mesh(dim, reordered, new[elements], np.asarray(tags, dtype=np.int64), nh)


def build_box_mesh(cells, lengths=(1.0, 1.0, 1.0), validate: bool = True) -> Mesh:
    """Kuhn-split box, all heart (isolated-heart slab, configs 2/3)."""
    if min(cells) < 1:
        raise ValueError("cells must be positive")
    vertices, elements, _ = box_grid(cells, lengths)
    tags = np.full(len(elements), int(Region.HEART), dtype=np.int64)
    mesh = Mesh(3, vertices, elements, tags, vertices.shape[0])
    if validate:
        mesh.validate()
    return mesh


def build_cube_mesh(cells_per_side: int) -> Mesh:
    """Unit cube, Kuhn 6-tet split, all heart (bd/mesh.py:142-185)."""
    m = int(cells_per_side)
    if m < 2:
        raise ValueError("cells_per_side must be at least 2")
    return build_box_mesh((m, m, m))


def build_rect_mesh(cells, lengths=(1.0, 1.0)) -> Mesh:
    vertices, elements, _ = rect_grid(cells, lengths)
    tags = np.full(len(elements), int(Region.HEART), dtype=np.int64)
    mesh = Mesh(2, vertices, elements, tags, vertices.shape[0])
    mesh.validate()
    return mesh


def build_square_mesh(cells_per_side: int) -> Mesh:
    """Unit square, two triangles per cell, all heart (bd/mesh.py:212-220)."""
    if cells_per_side < 2:
        raise ValueError("cells_per_side must be at least 2")
    return build_rect_mesh((cells_per_side, cells_per_side))


def build_heart_torso_2d(cells_per_side: int) -> Mesh:
    """Block heart [0.25,0.75]² in a lung / cavity / tissue torso (bd/mesh.py:223-267)."""
    m = int(cells_per_side)
    if m < 4 or m % 4 != 0:
        raise ValueError("cells_per_side must be a positive multiple of 4")
    vertices, elements, cell = rect_grid((m, m))
    q = m // 4
    i, j = cell[:, 0], cell[:, 1]
    band = (q <= j) & (j < 3 * q)
    tags = np.full(len(elements), int(Region.TORSO_OTHER), dtype=np.int64)
    tags[band & (i >= 3 * q)] = Region.TORSO_CAVITY
    tags[band & (i < q)] = Region.TORSO_LUNG
    tags[band & (q <= i) & (i < 3 * q)] = Region.HEART
    mesh = heart_first(2, vertices, elements, tags)
    mesh.validate()
    return mesh


def build_ellipse_torso_2d(cells_per_side: int = 512, length: float = 20.0,
                           center=(10.0, 10.0), outer=(4.0, 3.0), inner=(2.5, 1.8)) -> Mesh:
    """Config 1: elliptical myocardial annulus (outer semi-axes 4×3 cm minus a
    concentric 2.5×1.8 cm cavity) in a [0,L]² torso.  Elements are tagged by
    centroid: annulus → HEART, cavity → TORSO_CAVITY (blood), rest →
    TORSO_OTHER; vertices are permuted heart-first."""
    m = int(cells_per_side)
    vertices, elements, _ = rect_grid((m, m), (length, length))
    cen = vertices[elements].mean(axis=1)
    dx, dy = cen[:, 0] - center[0], cen[:, 1] - center[1]
    r_out = (dx / outer[0]) ** 2 + (dy / outer[1]) ** 2
    r_in = (dx / inner[0]) ** 2 + (dy / inner[1]) ** 2
    tags = np.full(len(elements), int(Region.TORSO_OTHER), dtype=np.int64)
    tags[r_in < 1.0] = Region.TORSO_CAVITY
    tags[(r_out < 1.0) & (r_in >= 1.0)] = Region.HEART
    mesh = heart_first(2, vertices, elements, tags)
    mesh.validate()
    return mesh


def build_ellipsoid_torso_3d(cells_per_side: int = 384, length: float = 20.0,
                             outer=(5.0, 4.0, 4.0), wall: float = 1.0,
                             validate: bool = False) -> Mesh:
    """Config 4: ellipsoidal ventricular shell (outer semi-axes 5×4×4 cm, wall
    1 cm, centred) in a Kuhn-split [0,L]³ torso box; cavity = blood."""
    m = int(cells_per_side)
    vertices, elements, _ = box_grid((m, m, m), (length, length, length))
    c = length / 2.0
    cen = vertices[elements].mean(axis=1) - c
    inner = tuple(a - wall for a in outer)
    r_out = sum((cen[:, k] / outer[k]) ** 2 for k in range(3))
    r_in = sum((cen[:, k] / inner[k]) ** 2 for k in range(3))
    tags = np.full(len(elements), int(Region.TORSO_OTHER), dtype=np.int64)
    tags[r_in < 1.0] = Region.TORSO_CAVITY
    tags[(r_out < 1.0) & (r_in >= 1.0)] = Region.HEART
    mesh = heart_first(3, vertices, elements, tags)
    if validate:
        mesh.validate()
    return mesh
