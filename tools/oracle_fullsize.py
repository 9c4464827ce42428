"""Run the CPU oracle on a FULL-size configuration and record per-step PCG
iteration counts, wall times and probe traces into tests/golden/<name>_oracle.json.

Test infrastructure: the fixture pins the GPU path at full size (iteration
counts ±2, probe traces 1e-6) and gives the CPU reference arm of bench.py the
oracle's own iterations per step.  Inputs are built with this repo's
(deterministic) builders; the GPU test rebuilds the identical matrices.

  python tools/oracle_fullsize.py --config cfg2 --steps 13
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--steps", type=int, default=13)
    ap.add_argument("--inner", default=None)
    ap.add_argument("--out", default=None)
    ap.add_argument("--cells", type=int, default=None, help="mesh size (cfg0/1/4 builders)")
    a = ap.parse_args()
    t0 = time.perf_counter()
    wl = configs.BUILDERS[a.config](a.cells) if a.cells else configs.BUILDERS[a.config]()
    inner = a.inner or wl.inner
    sysm = BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False)
    km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers)
    t_asm = time.perf_counter() - t0
    t0 = time.perf_counter()
    pre = orc.BlockLU(sysm.stiff_total, sysm.stiff_intra, km, inner)
    t_setup = time.perf_counter() - t0
    tag = f"{a.config}_{a.cells}" if a.cells else a.config
    out_path = a.out or os.path.join(REPO, "tests", "golden", f"{tag}_{inner}_oracle.json")
    rec = {"config": a.config, "cells": a.cells, "inner": inner, "n": sysm.n, "m": sysm.n_heart,
           "nnz_S1": int(sysm.stiff_total.nnz), "nnz_Si": int(sysm.stiff_intra.nnz),
           "nnz_Km": int(km.nnz), "assembly_s": t_asm, "setup_s": t_setup,
           "checksum_S1": float(np.abs(sysm.stiff_total.data).sum()),
           "checksum_Km": float(np.abs(km.data).sum()), "probes": wl.probes.tolist(),
           "tol": wl.tol, "dt": wl.dt, "iters": [], "step_s": [], "trace": [], "u_norm": [],
           "v_norm": [], "sub_stride": 97, "u_sub": [], "v_sub": []}
    print(json.dumps({k: v for k, v in rec.items() if not isinstance(v, list)}), flush=True)
    n, m = sysm.n, sysm.n_heart
    state = (np.zeros(n), np.full(m, wl.ionic.v_rest), np.ones(m))
    pts = wl.mesh.vertices[:m]
    from paper_1711_08708_b200.ionic import stimulus_vector
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
        if k < 3:  # strided subsample of the state for a rel-L2 check
            rec["u_sub"].append(state[0][::97].tolist())
            rec["v_sub"].append(state[1][::97].tolist())
        print(f"step {k + 1}: {st['iterations']} it, {rec['step_s'][-1]:.1f}s", flush=True)
        with open(out_path, "w") as fh:
            json.dump(rec, fh)


if __name__ == "__main__":
    main()
