"""Config-4 mesh-size sweep on one GPU (BASELINE cfg4: "a mesh-size sweep from
96^3 to 384^3 to check the n*log^alpha(n) cost trend").

3D ellipsoidal ventricle in a 20 cm torso box at cells^3; device assembly,
IC(0) inners, `steps` semi-implicit steps from rest (apex stimulus).  Prints
one JSON record per size, then the trend: growth rates of iterations*n between
sizes (bd/bench.py:30-36), the least-squares slope of log(iters*n) vs log n,
and alpha of iters ~ log(n)^alpha.  Sizes above ~300^3 assemble in row blocks
(assembly.DeviceAssembler, BD_ASSEMBLY_MAX_PAIRS) and need
BD_ASSEMBLY_REFZEROS=snap (no host assembly of a 57M-vertex torso); a watchdog
exits cleanly if host memory runs low.

  python tools/cfg4_sweep.py --cells 96,128,160,192 --steps 20
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
from paper_1711_08708_b200.study import growth_rate, least_squares_slope  # noqa: E402


def run(cells, steps):
    t0 = time.perf_counter()
    wl = configs.cfg4(cells)
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
    iters, dev_ms = [], []
    for _ in range(steps):
        state, st = bd.time_step(state, sysm, pre, wl.ionic, wl.protocol, wl.dt, tol=wl.tol,
                                 max_iter=20000, heart_points=pts)
        iters.append(int(st.iterations))
        dev_ms.append(float(st.device_time_ms))
    torch.cuda.synchronize()
    rec = {"cells": cells, "n": sysm.n, "m": sysm.n_heart, "dof": sysm.dof, "steps": steps,
           "iters": iters, "iters_mean": float(np.mean(iters)),
           "ms_per_step": float(np.mean(dev_ms)),
           "ms_per_iter": float(np.sum(dev_ms) / max(1, np.sum(iters))),
           "setup_s": {"mesh": round(t_mesh, 1), "assembly": round(t_asm, 1),
                       "precond": round(t_pre, 1)},
           "probe_v_final": state.v.cpu().numpy()[wl.probes].tolist(),
           "gpu_mem_used_gb": round((torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 1e9,
                                    1),
           "host_peak_rss_gb": round(__import__("resource").getrusage(
               __import__("resource").RUSAGE_SELF).ru_maxrss / 1e6, 1)}
    print(json.dumps(rec), flush=True)
    del pre, sysm, km, state
    torch.cuda.empty_cache()
    return rec


def _memory_watchdog(min_free_gb=10.0):
    """Exit cleanly before the host runs out of memory (a host OOM would take
    the box down); reports the peak host RSS."""
    import threading

    import psutil

    def watch():
        while True:
            if psutil.virtual_memory().available < min_free_gb * 1e9:
                print(json.dumps({"aborted": "host memory below %.0f GB free" % min_free_gb,
                                  "rss_gb": round(psutil.Process().memory_info().rss / 1e9, 1)}),
                      flush=True)
                os._exit(99)
            time.sleep(0.5)

    threading.Thread(target=watch, daemon=True).start()


def main():
    _memory_watchdog()
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", default="96,128,160,192")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    recs = [run(int(c), a.steps) for c in a.cells.split(",")]
    trend = {}
    if len(recs) >= 2:
        n = [r["n"] for r in recs]
        cost = [r["iters_mean"] * r["n"] for r in recs]
        trend["growth_iters_x_n"] = [round(growth_rate(c0, c1, n0, n1), 4) for c0, c1, n0, n1 in
                                     zip(cost, cost[1:], n, n[1:])]
        trend["slope_log_cost_vs_log_n"] = round(least_squares_slope(n, cost), 4)
        x = np.log(np.log(np.asarray(n, float)))
        y = np.log(np.asarray([r["iters_mean"] for r in recs]))
        trend["alpha_iters_vs_log_n"] = round(float(np.polyfit(x, y, 1)[0]), 3)
        trend["slope_log_iters_vs_log_n"] = round(least_squares_slope(n, [r["iters_mean"] for r in recs]), 4)
    print(json.dumps({"trend": trend}), flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump({"records": recs, "trend": trend}, fh, indent=1)


if __name__ == "__main__":
    main()
