"""Dev tool: time the Λ apply on cfg2 (new k_lambda2 vs old k_lambda)."""
import os, sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
import torch
import paper_1711_08708_b200 as bd
from paper_1711_08708_b200 import configs
wl = configs.cfg2()
sysm = bd.BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False)
x = bd.BlockVector(np.random.default_rng(0).standard_normal(sysm.n), np.random.default_rng(1).standard_normal(sysm.n_heart))
res = {}
for mode in ("0", "1"):
    os.environ["BD_LAMBDA"] = mode
    q = sysm.apply(x); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): q = sysm.apply(x)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    byts = 12 * (sysm.stiff_total.nnz + sysm.stiff_intra.nnz) + 8 * (5 * sysm.n + 6 * sysm.n_heart)
    print(f"lambda mode {mode}: {ms*1e3:.1f} us -> {byts/ms/1e6:.0f} GB/s algorithmic")
    res[mode] = q.buf.cpu().numpy()
print("max rel diff", np.abs(res["0"] - res["1"]).max() / np.abs(res["1"]).max())
