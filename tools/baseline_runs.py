"""Every BASELINE configuration at its stated step count on one GPU: setup
times, PCG iterations per step, device time per step and wall time of the
whole run (cfg0 100 steps exact, cfg1 200 steps exact, cfg2 50 steps ic0,
cfg3 20 steps ic0 on one GPU, cfg4 20 steps ic0 at the 192^3 sweep point).

  python tools/baseline_runs.py --configs cfg0,cfg1,cfg2,cfg3,cfg4 --out profiles/r01_baseline_runs.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import paper_1711_08708_b200 as bd  # noqa: E402
from paper_1711_08708_b200 import configs  # noqa: E402
from paper_1711_08708_b200.precond import build_monodomain_matrix  # noqa: E402

RUNS = {  # name -> (builder args, steps)
    "cfg0": ((), 100),
    "cfg1": ((), 200),
    "cfg2": ((), 50),
    "cfg3": ((), 20),
    "cfg4": ((192,), 20),
}


def run(name):
    args, steps = RUNS[name]
    t0 = time.perf_counter()
    wl = configs.BUILDERS[name](*args)
    t_mesh = time.perf_counter() - t0
    t0 = time.perf_counter()
    sysm = bd.BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False,
                                   assembly="device")
    km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers, assembly="device")
    t_asm = time.perf_counter() - t0
    t0 = time.perf_counter()
    pre = bd.BlockLUPreconditioner(sysm, inner=wl.inner, monodomain_matrix=km)
    t_pre = time.perf_counter() - t0
    state = bd.SimState.resting(sysm.n, sysm.n_heart, wl.ionic)
    pts = wl.mesh.vertices[: sysm.n_heart]
    its, dev = [], []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        state, st = bd.time_step(state, sysm, pre, wl.ionic, wl.protocol, wl.dt, tol=wl.tol,
                                 max_iter=20000, heart_points=pts)
        its.append(int(st.iterations))
        dev.append(float(st.device_time_ms))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    rec = {"config": name, "description": wl.description, "inner": wl.inner, "n": sysm.n,
           "m": sysm.n_heart, "steps": steps, "iters_per_step_mean": float(np.mean(its)),
           "iters_first_last": [its[0], its[-1]], "device_ms_per_step": float(np.mean(dev)),
           "wall_s_run": round(wall, 3), "steps_per_s": round(steps / wall, 4),
           "setup_s": {"mesh": round(t_mesh, 1), "assembly": round(t_asm, 1),
                       "precond": round(t_pre, 1)}}
    print(json.dumps(rec), flush=True)
    del pre, sysm, km, state
    torch.cuda.empty_cache()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg0,cfg1,cfg2,cfg3,cfg4")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    recs = [run(c) for c in a.configs.split(",")]
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(recs, fh, indent=1)


if __name__ == "__main__":
    main()
