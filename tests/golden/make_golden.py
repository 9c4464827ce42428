"""Generate the golden fixtures from the REAL reference (build container only).

Imports /root/reference/pkg/src/bidomain through tests/golden/refshim.py and
records its outputs on seeded inputs into tests/golden/*.npz.  The fixtures
pin both the oracle (tests/test_oracle_golden.py, CPU) and the GPU path
(tests/test_gpu_parity.py) to the reference itself.  /root/reference does not
exist on the GPU box; the fixtures travel instead.

Cases
  small_<name>   reference conftest instances (heart_torso_2d(8), square(4),
                 cube(2)): matrices, Λx, P^{-1}y per inner, _bulk_inverse(1),
                 IC(0) factors, PCG solves per inner.
  cfg0           BASELINE config 0 (64x64 square, x fibres, σ/χ of config 0):
                 matrices, the seeded sanity solve per inner, and 100 time
                 steps (strip stimulus) per inner: iteration counts, probe
                 traces and states at steps 10/50/100.
  cfg1s / cfg2s  reduced configs 1/2 built with this repo's builders (ellipse
                 heart-in-torso 64x64; orthotropic slab 12x12x6), fed to the
                 reference through its public constructor + monodomain_matrix=.

Run:  python tests/golden/make_golden.py [--only NAME]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, REPO)

import refshim  # noqa: E402

bd = refshim.import_reference()
from bidomain import assembly as ref_assembly  # noqa: E402
from bidomain import ionic as ref_ionic  # noqa: E402
from bidomain.conductivity import default_params  # noqa: E402
from bidomain.krylov import pcg_solve  # noqa: E402
from bidomain.mesh import (build_cube_mesh, build_heart_torso_2d,  # noqa: E402
                           build_square_mesh)
from bidomain.precond import BlockLUPreconditioner, IncompleteCholesky0  # noqa: E402
from bidomain.system import BidomainSystem, BlockVector  # noqa: E402
from bidomain.errors import NonConvergenceError  # noqa: E402

INNERS = ("exact", "ic0", "jacobi")


def put_csr(out, key, a):
    a = sp.csr_matrix(a)
    out[key + "_indptr"] = a.indptr.astype(np.int64)
    out[key + "_indices"] = a.indices.astype(np.int32)
    out[key + "_data"] = a.data.astype(np.float64)
    out[key + "_shape"] = np.array(a.shape, dtype=np.int64)


def put_stats(out, key, st):
    out[key + "_iters"] = np.int64(st.iterations)
    out[key + "_res"] = np.asarray(st.residual_history, dtype=float)
    out[key + "_prec"] = np.asarray(st.preconditioned_history, dtype=float)
    out[key + "_counts"] = np.array([st.mv_count, st.p1_count, st.pk_count], dtype=np.int64)


def system_arrays(out, sysm, km):
    put_csr(out, "S1", sysm.stiff_total)
    put_csr(out, "Si", sysm.stiff_intra)
    if sysm.stiff_extra is not None:
        put_csr(out, "Se", sysm.stiff_extra)
    put_csr(out, "Km", km)
    out["mass"] = sysm.mass_diag
    out["mh"] = sysm.heart_mass_diag
    out["gamma"] = np.float64(sysm.gamma)


def small_case(name, mesh, params, dt, seed=20240901):
    out = {}
    sysm = BidomainSystem.build(mesh, params, dt)
    rng = np.random.default_rng(seed)
    x = BlockVector(rng.standard_normal(sysm.n), rng.standard_normal(sysm.n_heart))
    ax = sysm.apply(x)
    out["x_u"], out["x_v"], out["lam_u"], out["lam_v"] = x.u, x.v, ax.u, ax.v
    nz = sysm.normalize(x)
    out["norm_u"] = nz.u
    y = BlockVector(rng.standard_normal(sysm.n), rng.standard_normal(sysm.n_heart))
    out["y_u"], out["y_v"] = y.u, y.v
    rhs = BlockVector(rng.standard_normal(sysm.n), rng.standard_normal(sysm.n_heart))
    rhs.u -= rhs.u.mean()
    out["b_u"], out["b_v"] = rhs.u, rhs.v
    km = None
    for inner in INNERS:
        pre = BlockLUPreconditioner(sysm, inner=inner)
        km = pre.monodomain_matrix
        out[f"beta"] = np.float64(pre.regularized.beta)
        z = pre.apply_inverse(y)
        out[f"pinv_{inner}_u"], out[f"pinv_{inner}_v"] = z.u, z.v
        out[f"bulk1_{inner}"] = pre._bulk_inverse(np.ones(sysm.n))
        if inner == "ic0":
            put_csr(out, "L1", pre.inner_bulk.lower_factor)
            put_csr(out, "LK", pre.inner_schur.lower_factor)
            out["ic0_restarts"] = np.array([pre.inner_bulk.restarts_used,
                                            pre.inner_schur.restarts_used])
        pre.reset_counters()
        xs, st = pcg_solve(sysm, pre, rhs, tol=1e-10, max_iter=2000)
        out[f"pcg_{inner}_u"], out[f"pcg_{inner}_v"] = xs.u, xs.v
        put_stats(out, f"pcg_{inner}", st)
    system_arrays(out, sysm, km)
    return out


class FieldWithFibers:
    """Duck-typed TensorField for the reference's assemble_stiffness with a
    custom fibre model (the reference's extension point, tests/test_assembly.py
    pattern); same formulas as bd/conductivity.py:181-224."""

    def __init__(self, params, dim, kind, frames_fn, orthotropic=None):
        self.params, self.dim, self.kind = params, dim, kind
        self.frames_fn = frames_fn
        self.ortho = orthotropic

    def evaluate_batch(self, centroids, tags):
        p, d = self.params, self.dim
        out = np.zeros((centroids.shape[0], d, d))
        heart = tags == 0
        if heart.any():
            fr = self.frames_fn(centroids[heart])
            eye = np.eye(d)
            if self.ortho is None:
                f = fr[:, 0, :]
                proj = np.einsum("ni,nj->nij", f, f)
                intra = p.g_i_l * proj + p.g_i_t * (eye - proj)
                extra = p.g_e_l * proj + p.g_e_t * (eye - proj)
            else:
                gi, ge = self.ortho
                intra = sum(gi[k] * np.einsum("ni,nj->nij", fr[:, k], fr[:, k]) for k in range(d))
                extra = sum(ge[k] * np.einsum("ni,nj->nij", fr[:, k], fr[:, k]) for k in range(d))
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
            for t in (1, 2, 3):
                m = tags == t
                if m.any():
                    out[m] = p.torso_conductivity(t) * np.eye(d)
        return out


def build_ref_system(mesh, params, dt, frames_fn, ortho=None):
    """BidomainSystem + K_m assembled by the reference's own assembly with a
    custom-fibre field (precond.py:34-47 restated around it)."""
    Space = ref_assembly.Space
    mk = lambda kind: FieldWithFibers(params, mesh.dim, kind, frames_fn, ortho)  # noqa: E731
    s1 = ref_assembly.assemble_stiffness(mesh, mk("bar1"))
    si = ref_assembly.assemble_stiffness(mesh, mk("intra"), Space.HEART_ONLY)
    se = ref_assembly.assemble_stiffness(mesh, mk("bar_e"))
    mass = ref_assembly.lumped_mass_diagonal(mesh)
    mh = ref_assembly.lumped_mass_diagonal(mesh, Space.HEART_ONLY)
    gam = params.chi * params.c_m / dt
    sysm = BidomainSystem(s1, si, se, mass, mh, gam, mesh=mesh, params=params)
    sm = ref_assembly.assemble_stiffness(mesh, mk("mono"), Space.HEART_ONLY)
    km = (sm + gam * sp.diags(mh)).tocsr()
    km.sum_duplicates()
    km.sort_indices()
    return sysm, km


def run_steps(sysm, pre, points, stim_fn, steps, dt, tol, probes, keep=(10, 50, 100),
              max_iter=5000):
    """The reference time_step (simulate.py:134-170) with a stimulus vector
    from stim_fn(points, t) (the strip is not a StimulusProtocol ball)."""
    ionp = ref_ionic.IonicParams()
    n, m = sysm.n, sysm.n_heart
    u, v, w = np.zeros(n), np.full(m, ionp.v_rest), np.ones(m)
    t = 0.0
    iters, trace, states = [], [v[probes].copy()], {}
    t0 = time.perf_counter()
    for k in range(steps):
        ion = ref_ionic.ionic_current(v, w, ionp, sysm.params.c_m)
        stim = stim_fn(points, t)
        rhs = sysm.build_rhs(v, ion, stim, sysm.params.chi)
        x, st = pcg_solve(sysm, pre, rhs, tol=tol, max_iter=max_iter, x0=BlockVector(u, v))
        u, v = x.u, x.v
        w = ref_ionic.update_gate(w, v, dt, ionp)
        t += dt
        iters.append(st.iterations)
        trace.append(v[probes].copy())
        if (k + 1) in keep:
            states[k + 1] = (u.copy(), v.copy(), w.copy())
    return np.array(iters), np.array(trace), states, time.perf_counter() - t0


def cfg_case(out, sysm, km, points, stim_fn, steps, dt, probes, inners, tol=1e-10, seed=0):
    system_arrays(out, sysm, km)
    out["probes"] = probes
    out["points"] = points
    # seeded sanity solve
    rng = np.random.default_rng(seed)
    bu = rng.uniform(-1.0, 1.0, sysm.n)
    bv = rng.uniform(-1.0, 1.0, sysm.n_heart)
    bu -= bu.mean()
    out["sanity_b_u"], out["sanity_b_v"] = bu, bv
    for inner in inners:
        t0 = time.perf_counter()
        pre = BlockLUPreconditioner(sysm, inner=inner, monodomain_matrix=km)
        if inner == "ic0":
            put_csr(out, "L1", pre.inner_bulk.lower_factor)
            put_csr(out, "LK", pre.inner_schur.lower_factor)
        out["beta"] = np.float64(pre.regularized.beta)
        try:
            x, st = pcg_solve(sysm, pre, BlockVector(bu, bv), tol=tol, max_iter=5000)
            out[f"sanity_{inner}_u"], out[f"sanity_{inner}_v"] = x.u, x.v
            put_stats(out, f"sanity_{inner}", st)
        except NonConvergenceError as exc:
            print(f"  sanity {inner}: no convergence ({exc})")
        if steps:
            iters, trace, states, secs = run_steps(sysm, pre, points, stim_fn, steps, dt, tol,
                                                   probes)
            out[f"steps_{inner}_iters"] = iters
            out[f"steps_{inner}_trace"] = trace
            for k, (u, v, w) in states.items():
                out[f"steps_{inner}_u{k}"], out[f"steps_{inner}_v{k}"] = u, v
                out[f"steps_{inner}_w{k}"] = w
            print(f"  {inner}: {steps} steps, it/step {iters.mean():.2f}, {secs:.1f}s")
        print(f"  {inner} done in {time.perf_counter() - t0:.1f}s")


def make_cfg0(cells=64, steps=100):
    from paper_1711_08708_b200 import configs

    wl = configs.cfg0(cells)
    mesh = build_square_mesh(cells)
    assert np.array_equal(mesh.vertices, wl.mesh.vertices)
    assert np.array_equal(mesh.elements, wl.mesh.elements)
    params = default_params(2, g_i_l=3.0, g_i_t=1.0, g_e_l=2.0, g_e_t=1.35, chi=200.0, c_m=1.0)

    def frames(c):
        f = np.tile(np.array([1.0, 0.0]), (c.shape[0], 1))
        return np.stack([f, np.column_stack([-f[:, 1], f[:, 0]])], axis=1)

    sysm, km = build_ref_system(mesh, params, 0.05, frames)
    pts = mesh.vertices[: sysm.n_heart]

    def stim(points, t):  # strip x < 0.1 for t in [0, 2)
        s = np.zeros(points.shape[0])
        if 0.0 <= t < configs.DURATION:
            s[points[:, 0] < 0.1] = configs.AMPLITUDE
        return s

    out = {}
    cfg_case(out, sysm, km, pts, stim, steps, 0.05, wl.probes, INNERS)
    return out


def make_cfg1s(cells=64, steps=40):
    from paper_1711_08708_b200 import configs

    wl = configs.cfg1(cells)
    mesh = wl.mesh
    params = default_params(2, g_i_l=3.0, g_i_t=1.0, g_e_l=2.0, g_e_t=1.35, chi=200.0, c_m=1.0,
                            k_cavity=6.0, k_other=2.0)
    sysm, km = build_ref_system(mesh, params, 0.05, wl.fibers.frames)
    pts = mesh.vertices[: sysm.n_heart]
    proto = ref_ionic.StimulusProtocol(
        sites=(ref_ionic.StimulusSite(tuple(wl.protocol.sites[0].center)),),
        radius=wl.protocol.radius, amplitude=wl.protocol.amplitude, duration=wl.protocol.duration)
    out = {"tags": mesh.tags, "n_heart": np.int64(mesh.heart_vertex_count)}
    cfg_case(out, sysm, km, pts, lambda p, t: ref_ionic.stimulus_vector(p, t, proto), steps,
             0.05, wl.probes, ("exact", "ic0"))
    return out


def make_cfg2s(cells=(12, 12, 6), steps=40):
    from paper_1711_08708_b200 import configs

    wl = configs.cfg2(cells)
    mesh = wl.mesh
    p = wl.params
    params = default_params(3, g_i_l=p.g_i_l, g_i_t=p.g_i_t, g_e_l=p.g_e_l, g_e_t=p.g_e_t,
                            chi=200.0, c_m=1.0, k_cavity=6.0, k_other=2.0)
    ortho = ((p.g_i_l, p.g_i_t, p.g_i_n), (p.g_e_l, p.g_e_t, p.g_e_n))
    sysm, km = build_ref_system(mesh, params, 0.05, wl.fibers.frames, ortho)
    pts = mesh.vertices[: sysm.n_heart]
    proto = ref_ionic.StimulusProtocol(sites=(ref_ionic.StimulusSite((0.0, 0.0, 0.0)),),
                                       radius=0.15, amplitude=wl.protocol.amplitude,
                                       duration=wl.protocol.duration)
    out = {"stim_radius": np.float64(0.15)}
    cfg_case(out, sysm, km, pts, lambda q, t: ref_ionic.stimulus_vector(q, t, proto), steps,
             0.05, wl.probes, ("ic0", "exact", "jacobi"))
    return out


def ic0_kat():
    """Known-answer factors (tests/test_precond.py:144-198 matrices)."""
    out = {}
    n = 15
    tri = sp.diags([3.0 * np.ones(n), -np.ones(n - 1), -np.ones(n - 1)], [0, 1, -1], format="csr")
    ic = IncompleteCholesky0()
    ic.setup(tri)
    put_csr(out, "tri", tri)
    put_csr(out, "tri_L", ic.lower_factor)
    relaxed = sp.csr_matrix(np.array([[3.45, -2.0, 0.0, 2.0], [-2.0, 3.45, -2.0, 0.0],
                                      [0.0, -2.0, 3.45, -2.0], [2.0, 0.0, -2.0, 3.45]]))
    ic = IncompleteCholesky0()
    ic.setup(relaxed)
    put_csr(out, "relaxed", relaxed)
    put_csr(out, "relaxed_L", ic.lower_factor)
    out["relaxed_restarts"] = np.int64(ic.restarts_used)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    jobs = {
        "small_coupled2d": lambda: small_case("coupled2d", build_heart_torso_2d(8),
                                              default_params(2), 0.05),
        "small_square4": lambda: small_case("square4", build_square_mesh(4), default_params(2), 0.05),
        "small_cube2": lambda: small_case("cube2", build_cube_mesh(2), default_params(3), 0.2),
        "ic0_kat": ic0_kat,
        "cfg0": make_cfg0,
        "cfg1s": make_cfg1s,
        "cfg2s": make_cfg2s,
    }
    for name, fn in jobs.items():
        if args.only and name != args.only:
            continue
        t0 = time.perf_counter()
        print(f"[golden] {name} ...", flush=True)
        out = fn()
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(f"[golden] {name}: {os.path.getsize(path) / 1e3:.0f} kB in "
              f"{time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
