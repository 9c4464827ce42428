"""Profiling driver: the bench workload (cfg2) — setup, one warm-up step, then
`--steps` time steps — with nothing else, so ncu launch lists / captures map
onto the bench's kernels.  Prints the library launch count per step."""
import argparse, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import paper_1711_08708_b200 as bd
from paper_1711_08708_b200 import configs, _lib
from paper_1711_08708_b200.precond import build_monodomain_matrix

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
wl = configs.BUILDERS[a.workload]()
sysm = bd.BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False,
                               assembly="device")
km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers, assembly="device")
pre = bd.BlockLUPreconditioner(sysm, inner=wl.inner, monodomain_matrix=km)
state = bd.SimState.resting(sysm.n, sysm.n_heart, wl.ionic)
pts = wl.mesh.vertices[: sysm.n_heart]
ctx = _lib.Context.default()
for k in range(1 + a.steps):
    l0 = ctx.launches()
    t0 = time.perf_counter()
    state, st = bd.time_step(state, sysm, pre, wl.ionic, wl.protocol, wl.dt, tol=wl.tol,
                             max_iter=20000, heart_points=pts)
    torch.cuda.synchronize()
    print(f"step {k}: {st.iterations} it, {time.perf_counter() - t0:.3f}s, "
          f"launches {ctx.launches() - l0}", flush=True)
