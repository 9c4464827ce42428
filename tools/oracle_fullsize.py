"""Run the CPU oracle on a FULL-size configuration and record per-step PCG
iteration counts, wall times and probe traces into tests/golden/<name>_oracle.json.

Test infrastructure: the fixture pins the GPU path at full size (iteration
counts ±2, probe traces 1e-6, state rel-L2 1e-8) and gives the CPU reference
arm of bench.py the oracle's own iterations per step.  Inputs are built with
this repo's (deterministic) builders; the GPU test rebuilds the identical
matrices.

State evidence, per step:
* ``u_norm``/``v_norm``/``w_norm``: full-state 2-norms;
* ``u_proj``/``v_proj``: projections of the full u and v on ``proj_k`` seeded
  Gaussian vectors (``numpy.random.default_rng(proj_seed)``, u first, then v).
  For two states x, y, mean_k (g_k·(x−y))² is an unbiased estimate of
  ‖x−y‖² (Johnson–Lindenstrauss), so the test bounds the FULL-state rel-L2
  without storing the state;
* at the steps listed in ``--sub-steps``: a stride-``sub_stride`` subsample of
  u and v, written to ``<tag>_<inner>_oracle_states.npz`` (float64).

  python tools/oracle_fullsize.py --config cfg2 --steps 50
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from oracle import bidomain_oracle as orc  # noqa: E402
from paper_1711_08708_b200 import configs  # noqa: E402
from paper_1711_08708_b200.precond import build_monodomain_matrix  # noqa: E402
from paper_1711_08708_b200.system import BidomainSystem  # noqa: E402

PROJ_SEED = 20261020


def projection_vectors(n, m, k, seed=PROJ_SEED):
    """The Gaussian test vectors of the fixture (shared with the GPU tests)."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((k, n)), rng.standard_normal((k, m))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--steps", type=int, default=13)
    ap.add_argument("--inner", default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--cells", type=int, default=None, help="mesh size (cfg0/1/4 builders)")
    ap.add_argument("--sub-stride", type=int, default=29)
    ap.add_argument("--sub-steps", default="1,2,3,5,10,20,30,40,41,45,50,100,150,200")
    ap.add_argument("--proj-k", type=int, default=32)
    ap.add_argument("--scipy-trsv", action="store_true",
                    help="IC(0) apply through scipy's spsolve_triangular instead of its "
                         "bit-identical C restatement (oracle_trsv_*; ~10x slower)")
    a = ap.parse_args()
    t0 = time.perf_counter()
    wl = configs.BUILDERS[a.config](a.cells) if a.cells else configs.BUILDERS[a.config]()
    inner = a.inner or wl.inner
    sysm = BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False)
    km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers)
    t_asm = time.perf_counter() - t0
    t0 = time.perf_counter()
    pre = orc.BlockLU(sysm.stiff_total, sysm.stiff_intra, km, inner,
                      fast_apply=not a.scipy_trsv)
    t_setup = time.perf_counter() - t0
    tag = f"{a.config}_{a.cells}" if a.cells else a.config
    out_path = a.out or os.path.join(REPO, "tests", "golden", f"{tag}_{inner}_oracle.json")
    npz_path = out_path.replace(".json", "_states.npz")
    sub_steps = sorted({int(s) for s in a.sub_steps.split(",") if s})
    rec = {"config": a.config, "cells": a.cells, "inner": inner, "n": sysm.n, "m": sysm.n_heart,
           "nnz_S1": int(sysm.stiff_total.nnz), "nnz_Si": int(sysm.stiff_intra.nnz),
           "nnz_Km": int(km.nnz), "assembly_s": t_asm, "setup_s": t_setup,
           "checksum_S1": float(np.abs(sysm.stiff_total.data).sum()),
           "checksum_Km": float(np.abs(km.data).sum()), "probes": wl.probes.tolist(),
           "tol": wl.tol, "dt": wl.dt, "iters": [], "step_s": [], "trace": [], "u_norm": [],
           "v_norm": [], "w_norm": [], "proj_seed": PROJ_SEED, "proj_k": a.proj_k,
           "u_proj": [], "v_proj": [], "sub_stride": a.sub_stride, "sub_steps": [],
           "states_file": os.path.basename(npz_path)}
    print(json.dumps({k: v for k, v in rec.items() if not isinstance(v, list)}), flush=True)
    n, m = sysm.n, sysm.n_heart
    gu, gv = projection_vectors(n, m, a.proj_k)
    state = (np.zeros(n), np.full(m, wl.ionic.v_rest), np.ones(m))
    pts = wl.mesh.vertices[:m]
    from paper_1711_08708_b200.ionic import stimulus_vector
    subs = {}
    t = 0.0
    for k in range(a.steps):
        stim = stimulus_vector(pts, t, wl.protocol)
        ts = time.perf_counter()
        state, st = orc.time_step(state, sysm.stiff_total, sysm.stiff_intra, sysm.heart_mass_diag,
                                  sysm.mass_diag, sysm.gamma, pre, wl.params.chi, wl.params.c_m,
                                  stim, wl.dt, tol=wl.tol, max_iter=20000)
        t += wl.dt
        rec["iters"].append(int(st["iterations"]))
        rec["step_s"].append(time.perf_counter() - ts)
        rec["trace"].append(state[1][wl.probes].tolist())
        rec["u_norm"].append(float(np.linalg.norm(state[0])))
        rec["v_norm"].append(float(np.linalg.norm(state[1])))
        rec["w_norm"].append(float(np.linalg.norm(state[2])))
        rec["u_proj"].append((gu @ state[0]).tolist())
        rec["v_proj"].append((gv @ state[1]).tolist())
        if (k + 1) in sub_steps:
            rec["sub_steps"].append(k + 1)
            subs[f"u_{k + 1}"] = state[0][::a.sub_stride].copy()
            subs[f"v_{k + 1}"] = state[1][::a.sub_stride].copy()
            np.savez(npz_path, **subs)
        print(f"step {k + 1}: {st['iterations']} it, {rec['step_s'][-1]:.1f}s", flush=True)
        with open(out_path + ".tmp", "w") as fh:
            json.dump(rec, fh)
        os.replace(out_path + ".tmp", out_path)


if __name__ == "__main__":
    main()
