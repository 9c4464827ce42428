"""Dev tool: time one IC(0) inner apply (forward+backward triangular pass) on a
config-2-style slab, tiled cooperative kernel vs the global sync-free kernel."""
import os, sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
import torch
import paper_1711_08708_b200 as bd
from paper_1711_08708_b200 import configs
from paper_1711_08708_b200.assembly import assemble_stiffness
from paper_1711_08708_b200.conductivity import TensorField
from paper_1711_08708_b200.precond import regularize_stiffness

cells = tuple(int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "128,128,64").split(","))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
wl = configs.cfg2(cells)
t0 = time.time()
from paper_1711_08708_b200.assembly import DeviceAssembler
S1 = DeviceAssembler(wl.mesh, wl.params, wl.fibers).stiffness("bar1")
g = regularize_stiffness(S1).grounded()
print(f"n={g.shape[0]} nnz={g.nnz} assembly {time.time()-t0:.1f}s", flush=True)
rng = np.random.default_rng(0)
y = torch.as_tensor(rng.standard_normal(g.shape[0])).cuda()
res = {}
for mode in os.environ.get("MODES", "persist,tiled,syncfree").split(","):
    mode_k, _, ring = mode.partition("%")  # e.g. btile@reg%static+persm3
    base, _, kern = mode_k.partition("@")  # e.g. btile@smem / btile@reg
    os.environ["BD_TRSV"] = base
    # suffix knobs: %static / %dyn (BD_RT_STATIC), %persmN (BD_BTILE_PERSM)
    for knob in filter(None, ring.split("+")):
        if knob in ("static", "dyn"):
            os.environ["BD_RT_STATIC"] = "1" if knob == "static" else "0"
        elif knob.startswith("persm"):
            os.environ["BD_BTILE_PERSM"] = knob[5:]
    if kern:
        os.environ["BD_BTILE_KERNEL"] = kern
    inner = bd.IncompleteCholesky0(); t0 = time.time(); inner.setup(g, coords=wl.mesh.vertices)
    print(mode, "setup", round(time.time()-t0, 2), "s", inner.factor_info(), flush=True)
    z = inner.apply_inverse(y); torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for k in range(reps):
        z = inner.apply_inverse(y)
        ev[k + 1].record()
    torch.cuda.synchronize()
    per = np.array([ev[k].elapsed_time(ev[k + 1]) for k in range(reps)])
    ms = float(np.median(per))
    print(f"{mode}: per-rep us min {per.min()*1e3:.1f} median {ms*1e3:.1f} max {per.max()*1e3:.1f}")
    slow = np.nonzero(per > 1.5 * ms)[0]
    print(f"{mode}: slow reps (>1.5x median): {slow.tolist()} -> {(per[slow]*1e3).round(0).tolist()}")
    nnz = inner.factor_info()["nnz"]; n = g.shape[0]
    byts = 2 * (12 * nnz + 4 * (n + 1) + 16 * n)
    print(f"{mode}: {ms*1e3:.1f} us per apply (median, fwd+bwd) -> {byts/ms/1e6:.0f} GB/s algorithmic", flush=True)
    res[mode] = z.cpu().numpy()
ks = list(res)
for k in ks[1:]:
    d = np.abs(res[k] - res[ks[0]]).max() / np.abs(res[ks[0]]).max()
    print(f"max rel diff {k} vs {ks[0]}", d)
# residual check: L L^T z = y approx? check symmetric positivity instead

