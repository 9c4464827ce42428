"""Dev tool: setup + a few time steps of a BASELINE config, with timings."""
import argparse, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1711_08708_b200 as bd
from paper_1711_08708_b200 import configs
from paper_1711_08708_b200.precond import build_monodomain_matrix
ap = argparse.ArgumentParser(); ap.add_argument("--workload", default="cfg1"); ap.add_argument("--inner", default=None)
ap.add_argument("--steps", type=int, default=3); ap.add_argument("--cells", default=None)
a = ap.parse_args()
t0 = time.perf_counter()
b = configs.BUILDERS[a.workload]
wl = b(int(a.cells)) if a.cells else b()
if a.inner: wl.inner = a.inner
sysm = bd.BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False,
                               assembly="device")
km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers, assembly="device")
t1 = time.perf_counter()
pre = bd.BlockLUPreconditioner(sysm, inner=wl.inner, monodomain_matrix=km)
t2 = time.perf_counter()
print(f"{wl.name} n={sysm.n} m={sysm.n_heart} inner={wl.inner} assembly {t1-t0:.1f}s precond {t2-t1:.1f}s", pre.inner_bulk.factor_info(), pre.inner_schur.factor_info(), flush=True)
state = bd.SimState.resting(sysm.n, sysm.n_heart, wl.ionic)
pts = wl.mesh.vertices[: sysm.n_heart]
for k in range(a.steps):
    ts = time.perf_counter()
    state, st = bd.time_step(state, sysm, pre, wl.ionic, wl.protocol, wl.dt, tol=wl.tol, max_iter=20000, heart_points=pts)
    torch.cuda.synchronize()
    print(f"step {k}: {st.iterations} it, {time.perf_counter()-ts:.4f}s, dev {st.device_time_ms:.2f} ms", flush=True)
