"""Conductivity tensors at element centroids (host setup).

Same parameters and tensor kinds as the reference (`bd/conductivity.py:23-240`):
transversely isotropic heart tensors g_l f fᵀ + g_t (I − f fᵀ), isotropic organ
values in the torso, the harmonic-mean monodomain tensor.  Two extensions the
BASELINE configurations need, both through the reference's own extension
point (a ``TensorField`` with a pluggable fibre model):

* fibre models: the reference fields (rotating 3D / circular 2D), uniform
  fibres (config 0), circumferential fibres about any centre (config 1), a
  (fibre, sheet, normal) frame rotating through the wall (configs 2/3) and a
  helical frame on an ellipsoidal shell (config 4);
* orthotropic eigenvalues: ``g_i_n`` / ``g_e_n`` give the third (normal)
  conductivity; σ = Σ_k g_k e_k e_kᵀ over the frame.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import NumericalDegeneracyError
from .mesh import Region

CHI_DEFAULT = {2: 1500.0, 3: 500.0}


@dataclass(frozen=True)
class ConductivityParams:
    """Conductivities (mS/cm), surface-to-volume ratio chi (1/cm), c_m (uF/cm²).

    g_*_l / g_*_t as the reference (bd/conductivity.py:23-57); the optional
    g_i_n / g_e_n make the heart tensors orthotropic (sheet = t, normal = n).
    """

    g_i_l: float = 1.741
    g_i_t: float = 0.1934
    g_e_l: float = 3.906
    g_e_t: float = 1.970
    k_lung: float = 0.5
    k_cavity: float = 6.7
    k_other: float = 2.2
    chi: float = 500.0
    c_m: float = 1.0
    g_i_n: float | None = None
    g_e_n: float | None = None

    def __post_init__(self):
        for name in ("g_i_l", "g_i_t", "g_e_l", "g_e_t", "k_lung", "k_cavity", "k_other",
                     "chi", "c_m"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be strictly positive")
        for name in ("g_i_n", "g_e_n"):
            val = getattr(self, name)
            if val is not None and val <= 0:
                raise ValueError(f"{name} must be strictly positive")

    @property
    def orthotropic(self) -> bool:
        return self.g_i_n is not None or self.g_e_n is not None

    def torso_conductivity(self, tag: int) -> float:
        if tag == Region.TORSO_LUNG:
            return self.k_lung
        if tag == Region.TORSO_CAVITY:
            return self.k_cavity
        if tag == Region.TORSO_OTHER:
            return self.k_other
        raise ValueError(f"unknown torso region tag {tag}")


def default_params(dim: int, **overrides) -> ConductivityParams:
    overrides.setdefault("chi", CHI_DEFAULT[dim])
    return ConductivityParams(**overrides)


# ---- fibre models: centroids (n, d) -> orthonormal frames (n, d, d), rows = (f, s[, n])
class FiberModel:
    def frames(self, centroids: np.ndarray) -> np.ndarray:  # pragma: no cover - interface
        raise NotImplementedError

    def fibers(self, centroids: np.ndarray) -> np.ndarray:
        return self.frames(centroids)[:, 0, :]


class ReferenceFibers(FiberModel):
    """The reference fields (bd/conductivity.py:66-88, 227-240): 3D horizontal
    fibre rotating from +π/4 (z=0) to −π/4 (z=1); 2D circular about (0.5,0.5)."""

    def __init__(self, dim: int, center=(0.5, 0.5)):
        self.dim = dim
        self.center = center

    def fibers(self, centroids):
        if self.dim == 3:
            z = np.clip(centroids[:, 2], 0.0, 1.0)
            theta = np.pi / 4 - np.pi / 2 * z
            return np.column_stack([np.cos(theta), np.sin(theta), np.zeros_like(theta)])
        return CircumferentialFibers(self.center).fibers(centroids)

    def frames(self, centroids):
        return _complete_frame(self.fibers(centroids))


class UniformFibers(FiberModel):
    """Constant fibre direction (config 0: along x)."""

    def __init__(self, direction):
        d = np.asarray(direction, dtype=float)
        self.direction = d / np.linalg.norm(d)

    def fibers(self, centroids):
        return np.tile(self.direction, (centroids.shape[0], 1))

    def frames(self, centroids):
        return _complete_frame(self.fibers(centroids))


class CircumferentialFibers(FiberModel):
    """Unit tangent of the circle about ``center``; x-axis at the centre itself."""

    def __init__(self, center=(0.5, 0.5)):
        self.center = center

    def fibers(self, centroids):
        dx = centroids[:, 0] - self.center[0]
        dy = centroids[:, 1] - self.center[1]
        r = np.hypot(dx, dy)
        out = np.column_stack([-dy, dx])
        deg = r == 0.0
        r = np.where(deg, 1.0, r)
        out /= r[:, None]
        out[deg] = (1.0, 0.0)
        return out

    def frames(self, centroids):
        return _complete_frame(self.fibers(centroids))


class TransmuralRotation(FiberModel):
    """Fibre angle linear in z from ``angle0`` at ``z0`` to ``angle1`` at ``z1``
    (degrees, in the x–y plane); sheet = in-plane perpendicular, normal = e_z.
    Configs 2/3 rotate through 120°: −60° at the bottom, +60° at the top."""

    def __init__(self, angle0=-60.0, angle1=60.0, z0=0.0, z1=0.5):
        self.angle0, self.angle1, self.z0, self.z1 = angle0, angle1, z0, z1

    def frames(self, centroids):
        z = np.clip((centroids[:, 2] - self.z0) / (self.z1 - self.z0), 0.0, 1.0)
        th = np.deg2rad(self.angle0 + (self.angle1 - self.angle0) * z)
        c, s = np.cos(th), np.sin(th)
        zero, one = np.zeros_like(th), np.ones_like(th)
        f = np.column_stack([c, s, zero])
        sh = np.column_stack([-s, c, zero])
        nn = np.column_stack([zero, zero, one])
        return np.stack([f, sh, nn], axis=1)


class EllipsoidHelical(FiberModel):
    """Config 4 helical fibres on an ellipsoidal shell: normal n = normalised
    gradient of the ellipsoidal level function; transmural depth from the
    epicardial (outer) to the endocardial (inner) level set; fibre angle
    −60° (epi) → +60° (endo) about n from the circumferential direction
    (e_z × n, falling back to e_x at the poles)."""

    def __init__(self, center, outer, wall, angle_epi=-60.0, angle_endo=60.0):
        self.center = np.asarray(center, float)
        self.outer = np.asarray(outer, float)
        self.inner = self.outer - wall
        self.angle_epi, self.angle_endo = angle_epi, angle_endo

    def frames(self, centroids):
        x = centroids - self.center
        g = 2.0 * x / self.outer ** 2
        n = g / np.maximum(np.linalg.norm(g, axis=1, keepdims=True), 1e-300)
        ro = np.sqrt(((x / self.outer) ** 2).sum(axis=1))
        ri = np.sqrt(((x / self.inner) ** 2).sum(axis=1))
        # depth 0 at the epicardium (ro = 1), 1 at the endocardium (ri = 1)
        depth = np.clip((1.0 - ro) / np.maximum(ri - ro, 1e-300), 0.0, 1.0)
        th = np.deg2rad(self.angle_epi + (self.angle_endo - self.angle_epi) * depth)
        circ = np.cross(np.array([0.0, 0.0, 1.0]), n)
        norm = np.linalg.norm(circ, axis=1, keepdims=True)
        pole = norm[:, 0] < 1e-12
        circ = np.where(pole[:, None], np.array([1.0, 0.0, 0.0]), circ / np.maximum(norm, 1e-300))
        long_ = np.cross(n, circ)
        f = np.cos(th)[:, None] * circ + np.sin(th)[:, None] * long_
        s = np.cross(n, f)
        return np.stack([f, s, n], axis=1)


def _complete_frame(f: np.ndarray) -> np.ndarray:
    """Orthonormal frame whose first row is f (2D: [f, f⊥]; 3D: any completion)."""
    if f.shape[1] == 2:
        return np.stack([f, np.column_stack([-f[:, 1], f[:, 0]])], axis=1)
    ref = np.where((np.abs(f[:, 2]) < 0.9)[:, None], np.array([0.0, 0.0, 1.0]),
                   np.array([1.0, 0.0, 0.0]))
    s = np.cross(ref, f)
    s /= np.linalg.norm(s, axis=1, keepdims=True)
    n = np.cross(f, s)
    return np.stack([f, s, n], axis=1)


def tensor_from_fiber(f, g_l: float, g_t: float) -> np.ndarray:
    """Transversely isotropic tensor g_l f fᵀ + g_t (I − f fᵀ)."""
    f = np.asarray(f, dtype=float)
    if abs(np.dot(f, f) - 1.0) > 1e-12:
        raise ValueError("fibre direction must be a unit vector")
    proj = np.outer(f, f)
    return g_l * proj + g_t * (np.eye(f.size) - proj)


def harmonic_mean_tensor(si, se) -> np.ndarray:
    si = np.asarray(si, dtype=float)
    se = np.asarray(se, dtype=float)
    try:
        out = np.linalg.inv(np.linalg.inv(si) + np.linalg.inv(se))
    except np.linalg.LinAlgError as exc:
        raise NumericalDegeneracyError(f"singular conductivity tensor: {exc}") from exc
    if not np.isfinite(out).all():
        raise NumericalDegeneracyError("harmonic mean produced non-finite entries")
    return 0.5 * (out + out.T)


class TensorField:
    """(centroid, tag) → SPD tensor; kinds intra / extra / mono / bar1 / bar_e
    as the reference (bd/conductivity.py:142-224), with a pluggable fibre
    model (default: the reference fields)."""

    KINDS = ("intra", "extra", "mono", "bar1", "bar_e")

    def __init__(self, params: ConductivityParams, dim: int, kind: str,
                 fibers: FiberModel | None = None):
        if kind not in self.KINDS:
            raise ValueError(f"unknown tensor field kind {kind!r}")
        self.params = params
        self.dim = dim
        self.kind = kind
        self.fibers = fibers if fibers is not None else ReferenceFibers(dim)

    def __call__(self, centroid, tag: int) -> np.ndarray:
        return self.evaluate_batch(np.asarray(centroid, float)[None, :], np.array([tag]))[0]

    def _heart_tensors(self, centroids):
        p, d = self.params, self.dim
        if not p.orthotropic:
            f = self.fibers.fibers(centroids)
            proj = np.einsum("ni,nj->nij", f, f)
            eye = np.eye(d)
            intra = p.g_i_l * proj + p.g_i_t * (eye - proj)
            extra = p.g_e_l * proj + p.g_e_t * (eye - proj)
            return intra, extra
        fr = self.fibers.frames(centroids)  # (n, d, d), rows e_k
        gi = [p.g_i_l, p.g_i_t, p.g_i_n if p.g_i_n is not None else p.g_i_t][:d]
        ge = [p.g_e_l, p.g_e_t, p.g_e_n if p.g_e_n is not None else p.g_e_t][:d]
        intra = sum(gi[k] * np.einsum("ni,nj->nij", fr[:, k], fr[:, k]) for k in range(d))
        extra = sum(ge[k] * np.einsum("ni,nj->nij", fr[:, k], fr[:, k]) for k in range(d))
        return intra, extra

    def evaluate_batch(self, centroids: np.ndarray, tags: np.ndarray) -> np.ndarray:
        centroids = np.asarray(centroids, dtype=float)
        tags = np.asarray(tags)
        n, d = centroids.shape[0], self.dim
        p = self.params
        out = np.zeros((n, d, d))
        heart = tags == Region.HEART
        if self.kind in ("intra", "extra", "mono") and not heart.all():
            raise ValueError(f"{self.kind!r} tensor is only defined on heart elements")
        if heart.any():
            intra, extra = self._heart_tensors(centroids[heart])
            if self.kind == "intra":
                out[heart] = intra
            elif self.kind in ("extra", "bar_e"):
                out[heart] = extra
            elif self.kind == "bar1":
                out[heart] = intra + extra
            else:
                mono = np.linalg.inv(np.linalg.inv(intra) + np.linalg.inv(extra))
                out[heart] = 0.5 * (mono + mono.transpose(0, 2, 1))
        if self.kind in ("bar1", "bar_e"):
            known = heart.copy()
            for t in (Region.TORSO_LUNG, Region.TORSO_CAVITY, Region.TORSO_OTHER):
                mask = tags == t
                if mask.any():
                    out[mask] = p.torso_conductivity(t) * np.eye(d)
                known |= mask
            if not known.all():
                raise ValueError("unknown region tag in mesh")
        return out
