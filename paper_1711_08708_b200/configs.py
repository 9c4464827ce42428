"""The BASELINE.json workloads as deterministic synthetic inputs (host setup).

No dataset is involved: every configuration is a structured mesh plus
conductivity/fibre/stimulus choices.  Choices the BASELINE text leaves open
are fixed here and stated in DESIGN.md:

* stimulus amplitude "1" (dimensionless MS units) = 140 µA/cm² (×c_m·v_span),
  duration 2 ms, half-open window;
* chi = 200 /cm everywhere (config 0 states it; 1–4 do not);
* config 1: point stimulus = ball r 0.3 cm at (6.5, 10) on the heart's left
  edge; the "Dirichlet ground" is kept as the reference's mass-weighted
  normalisation (bd/system.py:138-146);
* configs 2/3: fibre angle −60° (z=0) → +60° (top), sheet in-plane ⊥, normal
  e_z; corner stimulus = ball r 0.1 cm at the origin;
* config 4: apex stimulus = ball r 0.3 cm at the ellipsoid's −x apex
  mid-wall.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .conductivity import (CircumferentialFibers, ConductivityParams, EllipsoidHelical,
                           TransmuralRotation, UniformFibers)
from .ionic import IonicParams, StimulusBox, StimulusProtocol, StimulusSite
from .mesh import (Mesh, build_box_mesh, build_ellipse_torso_2d, build_ellipsoid_torso_3d,
                   build_rect_mesh)

AMPLITUDE = 140.0   # = 1 in Mitchell–Schaeffer units (c_m · v_span)
DURATION = 2.0      # ms


@dataclass
class Workload:
    name: str
    mesh: Mesh
    params: ConductivityParams
    fibers: object
    protocol: StimulusProtocol
    dt: float = 0.05
    steps: int = 100
    tol: float = 1e-10
    inner: str = "ic0"
    ionic: IonicParams = field(default_factory=IonicParams)
    probes: np.ndarray = None
    description: str = ""

    @property
    def n(self) -> int:
        return self.mesh.vertex_count

    @property
    def n_heart(self) -> int:
        return self.mesh.heart_vertex_count

    @property
    def dof(self) -> int:
        return self.n + self.n_heart


def _probes(mesh: Mesh, points) -> np.ndarray:
    hv = mesh.vertices[: mesh.heart_vertex_count]
    return np.array([int(np.argmin(((hv - np.asarray(p)) ** 2).sum(axis=1))) for p in points],
                    dtype=np.int64)


def params_2d(**kw) -> ConductivityParams:
    base = dict(g_i_l=3.0, g_i_t=1.0, g_e_l=2.0, g_e_t=1.35, chi=200.0, c_m=1.0)
    base.update(kw)
    return ConductivityParams(**base)


def params_3d(**kw) -> ConductivityParams:
    base = dict(g_i_l=3.0, g_i_t=1.0, g_i_n=0.31, g_e_l=2.0, g_e_t=1.65, g_e_n=1.35,
                chi=200.0, c_m=1.0, k_cavity=6.0, k_other=2.0)
    base.update(kw)
    return ConductivityParams(**base)


def cfg0(cells: int = 64, inner: str = "exact", steps: int = 100) -> Workload:
    """2D tissue square, x fibres, strip stimulus x < 0.1 cm for 2 ms."""
    mesh = build_rect_mesh((cells, cells))
    proto = StimulusProtocol(sites=(StimulusBox((-np.inf, -np.inf), (0.1, np.inf)),),
                             amplitude=AMPLITUDE, duration=DURATION)
    return Workload("cfg0", mesh, params_2d(), UniformFibers((1.0, 0.0)), proto, steps=steps,
                    inner=inner,
                    probes=_probes(mesh, [(0.05, 0.5), (0.25, 0.5), (0.5, 0.5), (0.75, 0.5),
                                          (0.95, 0.5)]),
                    description=f"2D tissue {cells}x{cells} P1, x fibres")


def cfg1(cells: int = 512, inner: str = "exact", steps: int = 200) -> Workload:
    """2D elliptical heart in a [0,20]² torso (blood cavity 6.0, torso 2.0)."""
    mesh = build_ellipse_torso_2d(cells)
    proto = StimulusProtocol(sites=(StimulusSite((6.5, 10.0)),), radius=0.3,
                             amplitude=AMPLITUDE, duration=DURATION)
    params = params_2d(k_cavity=6.0, k_other=2.0)
    return Workload("cfg1", mesh, params, CircumferentialFibers((10.0, 10.0)), proto,
                    steps=steps, inner=inner,
                    probes=_probes(mesh, [(6.5, 10.0), (10.0, 13.5), (13.5, 10.0), (10.0, 6.5)]),
                    description=f"2D heart-in-torso {cells}x{cells} on [0,20]^2")


def cfg2(cells=(128, 128, 64), inner: str = "ic0", steps: int = 50, name: str = "cfg2") -> Workload:
    """3D orthotropic slab 1×1×0.5 cm, fibres rotating 120° through the wall."""
    mesh = build_box_mesh(cells, (1.0, 1.0, 0.5), validate=False)
    proto = StimulusProtocol(sites=(StimulusSite((0.0, 0.0, 0.0)),), radius=0.1,
                             amplitude=AMPLITUDE, duration=DURATION)
    return Workload(name, mesh, params_3d(), TransmuralRotation(-60.0, 60.0, 0.0, 0.5), proto,
                    steps=steps, inner=inner,
                    probes=_probes(mesh, [(0.0, 0.0, 0.0), (0.25, 0.25, 0.25), (0.5, 0.5, 0.25),
                                          (1.0, 1.0, 0.5)]),
                    description=f"3D slab {cells[0]}x{cells[1]}x{cells[2]} Kuhn P1")


def cfg3(cells=(256, 256, 128), inner: str = "ic0", steps: int = 20) -> Workload:
    return cfg2(cells, inner, steps, name="cfg3")


def cfg4(cells: int = 384, inner: str = "ic0", steps: int = 20) -> Workload:
    """3D ellipsoidal ventricle (5×4×4 cm, 1 cm wall) in a 20 cm torso box."""
    L = 20.0
    mesh = build_ellipsoid_torso_3d(cells, L, (5.0, 4.0, 4.0), 1.0)
    c = L / 2
    apex = (c - 4.5, c, c)
    proto = StimulusProtocol(sites=(StimulusSite(apex),), radius=0.3, amplitude=AMPLITUDE,
                             duration=DURATION)
    fibers = EllipsoidHelical((c, c, c), (5.0, 4.0, 4.0), 1.0)
    return Workload("cfg4", mesh, params_3d(), fibers, proto, steps=steps, inner=inner,
                    probes=_probes(mesh, [apex]), description=f"3D heart-in-torso {cells}^3")


BUILDERS = {"cfg0": cfg0, "cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4}


def sanity_rhs(n: int, m: int, seed: int = 0):
    """Seeded uniform[-1,1] RHS with the u-block projected to mean zero
    (tests/test_krylov.py:21-24 in the reference; BASELINE config 0)."""
    rng = np.random.default_rng(seed)
    u = rng.uniform(-1.0, 1.0, n)
    v = rng.uniform(-1.0, 1.0, m)
    u -= u.mean()
    return u, v
