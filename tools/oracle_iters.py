"""Iteration-level oracle record for configurations whose full time step is
out of reach on the CPU (config 3: 8.5M vertices, ~600 PCG iterations per
step at ~15 s per oracle iteration).

Runs the CPU oracle on the FIRST time step from rest (membrane RHS at t=0,
warm start x0 = (u_0, v_0), tol 1e-10) for --iters PCG iterations
(krylov.py:100-131) and records the residual and r·z histories and the
normalised iterate after those iterations (norms, Gaussian projections and a
strided subsample, as tools/oracle_fullsize.py) into
tests/golden/<config>_<inner>_iters<K>.json (+ _states.npz).

  python tools/oracle_iters.py --config cfg3 --iters 30
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tools"))

from oracle import bidomain_oracle as orc  # noqa: E402
from oracle_fullsize import PROJ_SEED, projection_vectors  # noqa: E402
from paper_1711_08708_b200 import configs  # noqa: E402
from paper_1711_08708_b200.precond import build_monodomain_matrix  # noqa: E402
from paper_1711_08708_b200.system import BidomainSystem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--sub-stride", type=int, default=97)
    ap.add_argument("--proj-k", type=int, default=16)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    t0 = time.perf_counter()
    wl = configs.BUILDERS[a.config]()
    sysm = BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False)
    km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers)
    t_asm = time.perf_counter() - t0
    print(f"assembly {t_asm:.0f}s n={sysm.n} m={sysm.n_heart}", flush=True)
    t0 = time.perf_counter()
    pre = orc.BlockLU(sysm.stiff_total, sysm.stiff_intra, km, wl.inner)
    t_setup = time.perf_counter() - t0
    print(f"preconditioner {t_setup:.0f}s", flush=True)
    n, m = sysm.n, sysm.n_heart
    u, v, w = np.zeros(n), np.full(m, wl.ionic.v_rest), np.ones(m)
    from paper_1711_08708_b200.ionic import stimulus_vector
    stim = stimulus_vector(wl.mesh.vertices[:m], 0.0, wl.protocol)
    ion = orc.ionic_current(v, w, c_m=wl.params.c_m)
    bu, bv = orc.build_rhs(n, sysm.heart_mass_diag, sysm.gamma, v, ion, stim, wl.params.chi)
    t0 = time.perf_counter()
    try:
        orc.pcg(sysm.stiff_total, sysm.stiff_intra, sysm.heart_mass_diag, sysm.mass_diag,
                sysm.gamma, pre, bu, bv, tol=wl.tol, max_iter=a.iters, x0=(u, v))
        raise SystemExit("converged before --iters; record a full step instead")
    except orc.OracleNoConvergence as e:
        st = e.stats
    t_pcg = time.perf_counter() - t0
    xu, xv = st["iterate"]
    gu, gv = projection_vectors(n, m, a.proj_k)
    tag = f"{a.config}_{wl.inner}_iters{a.iters}"
    out = a.out or os.path.join(REPO, "tests", "golden", f"{tag}.json")
    npz = out.replace(".json", "_states.npz")
    rec = {"config": a.config, "inner": wl.inner, "n": n, "m": m, "tol": wl.tol,
           "iters": a.iters, "nnz_S1": int(sysm.stiff_total.nnz), "nnz_Km": int(km.nnz),
           "checksum_S1": float(np.abs(sysm.stiff_total.data).sum()),
           "checksum_Km": float(np.abs(km.data).sum()),
           "assembly_s": t_asm, "setup_s": t_setup, "pcg_s": t_pcg,
           "residual_history": st["residual_history"],
           "preconditioned_history": st["preconditioned_history"],
           "mv_count": st["mv_count"], "p1_count": st["p1_count"], "pk_count": st["pk_count"],
           "u_norm": float(np.linalg.norm(xu)), "v_norm": float(np.linalg.norm(xv)),
           "proj_seed": PROJ_SEED, "proj_k": a.proj_k,
           "u_proj": (gu @ xu).tolist(), "v_proj": (gv @ xv).tolist(),
           "sub_stride": a.sub_stride, "states_file": os.path.basename(npz)}
    np.savez(npz, u=xu[::a.sub_stride], v=xv[::a.sub_stride])
    with open(out, "w") as fh:
        json.dump(rec, fh)
    print(f"{a.iters} iterations in {t_pcg:.0f}s; final rel residual "
          f"{st['residual_history'][-1]:.3e}", flush=True)


if __name__ == "__main__":
    main()
