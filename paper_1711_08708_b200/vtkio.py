"""Legacy-ASCII VTK unstructured grids (drop-in for bd/vtkio.py:1-140).

Same file layout as the reference so files interchange both ways: POINTS
padded to 3 components, CELLS with the arity prefix, CELL_TYPES (5 triangle,
10 tetrahedron), region tags as the first CELL_DATA scalar, and for field
snapshots POINT_DATA `u` (all vertices) and `v` (heart vertices, NaN
elsewhere).  Floats carry 17 significant digits so coordinates round-trip
bit for bit.  Sections are written as whole numpy blocks (np.savetxt), and
field arguments may be device tensors (copied once).
"""
from __future__ import annotations

import io

import numpy as np

from .errors import BidomainError
from .mesh import Mesh, Region

VTK_TRIANGLE, VTK_TETRA = 5, 10
_CELL = {2: VTK_TRIANGLE, 3: VTK_TETRA}
_DIM = {VTK_TRIANGLE: 2, VTK_TETRA: 3}


def _host(x) -> np.ndarray:
    if hasattr(x, "detach"):  # torch tensor (possibly on the GPU)
        x = x.detach().cpu().numpy()
    return np.asarray(x, dtype=float)


def _block(handle, arr, fmt):
    buf = io.StringIO()
    np.savetxt(buf, arr, fmt=fmt)
    handle.write(buf.getvalue())


def _geometry(handle, mesh: Mesh, title: str) -> None:
    n, ne, a = mesh.vertex_count, mesh.elements.shape[0], mesh.dim + 1
    handle.write(f"# vtk DataFile Version 3.0\n{title}\nASCII\nDATASET UNSTRUCTURED_GRID\n")
    pts = np.zeros((n, 3))
    pts[:, : mesh.dim] = mesh.vertices
    handle.write(f"POINTS {n} double\n")
    _block(handle, pts, "%.17g")
    handle.write(f"CELLS {ne} {ne * (a + 1)}\n")
    cells = np.empty((ne, a + 1), dtype=np.int64)
    cells[:, 0] = a
    cells[:, 1:] = mesh.elements
    _block(handle, cells, "%d")
    handle.write(f"CELL_TYPES {ne}\n")
    _block(handle, np.full(ne, _CELL[mesh.dim], dtype=np.int64), "%d")
    handle.write(f"CELL_DATA {ne}\nSCALARS region int 1\nLOOKUP_TABLE default\n")
    _block(handle, np.asarray(mesh.tags, dtype=np.int64), "%d")


def write_mesh_vtk(mesh: Mesh, path, title: str = "bidomain mesh") -> None:
    """Mesh with region tags as CELL_DATA (bd/vtkio.py:45-53)."""
    with open(path, "w") as fh:
        _geometry(fh, mesh, title)


def write_fields_vtk(mesh: Mesh, path, u, v, title: str = "bidomain fields") -> None:
    """Snapshot: u on every vertex, v on the heart (NaN outside) (bd/vtkio.py:56-76)."""
    u = _host(u)
    v_full = np.full(mesh.vertex_count, np.nan)
    v_full[: mesh.heart_vertex_count] = _host(v)
    with open(path, "w") as fh:
        _geometry(fh, mesh, title)
        fh.write(f"POINT_DATA {mesh.vertex_count}\nSCALARS u double 1\nLOOKUP_TABLE default\n")
        _block(fh, u, "%.17g")
        fh.write("SCALARS v double 1\nLOOKUP_TABLE default\n")
        _block(fh, v_full, "%.17g")


def read_mesh_vtk(path) -> Mesh:
    """Read back what the writers above (or the reference's) produce
    (bd/vtkio.py:79-118): geometry, tags, heart-first vertex count."""
    with open(path) as fh:
        tok = fh.read().split()

    def at(word):
        try:
            return tok.index(word)
        except ValueError as exc:
            raise BidomainError(f"VTK file lacks {word} section") from exc

    p = at("POINTS")
    n = int(tok[p + 1])
    xyz = np.asarray(tok[p + 3: p + 3 + 3 * n], dtype=float).reshape(n, 3)
    p = at("CELLS")
    ne, total = int(tok[p + 1]), int(tok[p + 2])
    raw = np.asarray(tok[p + 3: p + 3 + total], dtype=np.int64)
    arity = int(raw[0]) if raw.size else 0
    if ne and total != ne * (arity + 1):
        raise BidomainError("CELLS section has mixed arities")
    cells = raw.reshape(ne, arity + 1)[:, 1:]
    p = at("CELL_TYPES")
    ctype = int(tok[p + 2])
    if ctype not in _DIM:
        raise BidomainError(f"unsupported VTK cell type {ctype}")
    dim = _DIM[ctype]
    if arity != dim + 1:
        raise BidomainError("cell arity inconsistent with cell type")
    p = at("SCALARS")
    if tok[p + 1] != "region":
        raise BidomainError("expected region scalars as first CELL_DATA")
    tags = np.asarray(tok[p + 6: p + 6 + ne], dtype=np.int64)
    heart = cells[tags == Region.HEART]
    mesh = Mesh(dim, xyz[:, :dim].copy(), cells, tags, int(heart.max()) + 1 if heart.size else 0)
    mesh.validate()
    return mesh


def write_activation_csv(mesh: Mesh, phi, path) -> None:
    """activation.csv of the `simulate` command (bd/cli.py:111-120): one row per
    heart vertex, vertex_id, x, y, z (17 digits), phi_ms (10 digits, nan if
    never activated)."""
    phi = _host(phi)
    m = mesh.heart_vertex_count
    xyz = np.zeros((m, 3))
    xyz[:, : mesh.dim] = mesh.vertices[:m]
    with open(path, "w", newline="") as fh:
        fh.write("vertex_id,x,y,z,phi_ms\r\n")
        for vid in range(m):
            fh.write(f"{vid},{xyz[vid, 0]:.17g},{xyz[vid, 1]:.17g},{xyz[vid, 2]:.17g},"
                     f"{phi[vid]:.10g}\r\n")
