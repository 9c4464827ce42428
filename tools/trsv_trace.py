"""Dev tool: step trace of the tiled triangular solve (forward pass) on cfg2."""
import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, '/root/repo')
import torch
import paper_1711_08708_b200 as bd
from paper_1711_08708_b200 import configs, _lib
from paper_1711_08708_b200.assembly import assemble_stiffness
from paper_1711_08708_b200.conductivity import TensorField
from paper_1711_08708_b200.precond import regularize_stiffness
cells = tuple(int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "128,128,64").split(","))
wl = configs.cfg2(cells)
S1 = assemble_stiffness(wl.mesh, TensorField(wl.params, 3, "bar1", wl.fibers))
g = regularize_stiffness(S1).grounded()
inner = bd.IncompleteCholesky0(); inner.setup(g, coords=wl.mesh.vertices)
L = _lib.lib()
L.bd_inner_tile_info.argtypes = [C.c_void_p, C.c_void_p]; L.bd_debug_tile_trace.argtypes = [C.c_void_p, C.c_int]
info = (C.c_int64 * 8)(); L.bd_inner_tile_info(inner.handle, info); info = list(info)
print("tile info parts,threads,G,smem,max_rows,max_steps,Lsteps,Usteps:", info)
P, S = info[0], info[5]
buf = torch.zeros(P * S * 5, dtype=torch.int64, device='cuda')
y = torch.as_tensor(np.random.default_rng(0).standard_normal(g.shape[0])).cuda()
inner.apply_inverse(y); torch.cuda.synchronize()
L.bd_debug_tile_trace(C.c_void_p(buf.data_ptr()), S)
inner.apply_inverse(y); torch.cuda.synchronize()
L.bd_debug_tile_trace(None, 0)
tr = buf.view(P, S, 5).cpu().numpy().astype(np.int64)
# forward pass recorded first then overwritten by backward; the trace holds the backward pass
t0 = tr[:, :, 0][tr[:, :, 0] > 0].min()
tops = np.where(tr[:, :, 0] > 0, tr[:, :, 0] - t0, -1)
ends = np.where(tr[:, :, 2] > 0, tr[:, :, 2] - t0, -1)
nsteps = (tr[:, :, 0] > 0).sum(axis=1)
print("steps per part min/mean/max", nsteps.min(), nsteps.mean(), nsteps.max())
dur = ends - tops
valid = tops >= 0
print("step duration us: median %.2f p90 %.2f max %.2f" % (np.median(dur[valid]) / 1e3, np.percentile(dur[valid], 90) / 1e3, dur[valid].max() / 1e3))
gap = tops[:, 1:] - ends[:, :-1]
vg = (tops[:, 1:] >= 0)
print("gap between steps us: median %.3f" % (np.median(gap[vg]) / 1e3))
print("spins per step: mean %.2f, steps with spins %.1f%%" % (tr[:, :, 1][valid].mean(), 100 * (tr[:, :, 1][valid] > 0).mean()))
first = np.array([tops[p][0] for p in range(P)]); last = np.array([ends[p][nsteps[p] - 1] for p in range(P)])
print("part start us: min %.1f median %.1f max %.1f" % (first.min() / 1e3, np.median(first) / 1e3, first.max() / 1e3))
print("part end us: min %.1f median %.1f max %.1f" % (last.min() / 1e3, np.median(last) / 1e3, last.max() / 1e3))
for p in (0, 1, P // 2, P - 1):
    print(f"part {p}: steps {nsteps[p]}, first 5 durations", (dur[p][:5] / 1e3).round(2), "spins", tr[p, :5, 1], "start", first[p] / 1e3)
np.save("/root/repo/gpurun_out/trace.npy", tr)
for p in (P - 1, P // 2, 0):
    v = tops[p] >= 0
    w = (tr[p, :, 3] - t0 - tops[p])[v] / 1e3; dn = (tr[p, :, 4] - t0 - tops[p])[v] / 1e3; e = dur[p][v] / 1e3
    print(f"part {p}: median top->max(wait done) {np.median(w):.2f} us, top->max(compute done) {np.median(dn):.2f} us, step {np.median(e):.2f} us")
