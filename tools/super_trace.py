"""Dev tool: per-task trace of the supernodal solve of the bulk exact factor
(cfg1); argv[1] = "fwd" traces the forward pass, default the backward one."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, '/root/repo')
import torch
import paper_1711_08708_b200 as bd
from paper_1711_08708_b200 import configs, _lib
from paper_1711_08708_b200.assembly import assemble_stiffness
from paper_1711_08708_b200.conductivity import TensorField
from paper_1711_08708_b200.precond import regularize_stiffness
wl = configs.cfg1()
from paper_1711_08708_b200.assembly import DeviceAssembler
g = regularize_stiffness(DeviceAssembler(wl.mesh, wl.params, wl.fibers).stiffness("bar1")).grounded()
inner = bd.ExactFactorization(); inner.setup(g)
L = _lib.lib(); L.bd_debug_tile_trace.argtypes = [C.c_void_p, C.c_int]
NT = 200000
buf = torch.zeros(NT * 4, dtype=torch.int64, device='cuda')
y = torch.as_tensor(np.random.default_rng(0).standard_normal(g.shape[0])).cuda()
inner.apply_inverse(y); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); inner.apply_inverse(y); e1.record(); torch.cuda.synchronize()
print("apply (fwd+bwd) ms", e0.elapsed_time(e1))
L.bd_debug_tile_trace(C.c_void_p(buf.data_ptr()), -NT if sys.argv[1:2] == ["fwd"] else NT)
inner.apply_inverse(y); torch.cuda.synchronize()
L.bd_debug_tile_trace(None, 0)
tr = buf.view(NT, 4).cpu().numpy()
tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min()
beg, end = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3
big = (tr[:, 3] & (1 << 19)) != 0
ext_ns = tr[:, 3] >> 20
print("tasks", len(tr), "big", big.sum(), "span us %.1f" % end.max())
print("small task dur us: median %.2f p90 %.2f max %.2f" % (np.median((end-beg)[~big]), np.percentile((end-beg)[~big], 90), (end-beg)[~big].max()))
if big.any():
    d = (end - beg)[big]; sz = tr[big, 3] & 0x7ffff; ex = ext_ns[big] / 1e3
    order = np.argsort(beg[big])
    print("big tasks (start, dur, wait+ext phase, dense phase, size): ")
    for k in order[-16:]:
        print("  %.1f %.1f %.1f %.1f %d" % (beg[big][k], d[k], ex[k], d[k] - ex[k], sz[k]))
    print("big: sum dense-phase us %.1f, median dense %.2f" % ((d - ex).sum(), np.median(d - ex)))
# activity timeline: number of tasks running vs time
ts = np.linspace(0, end.max(), 30)
print("running tasks over time:", [int(((beg <= x) & (end >= x)).sum()) for x in ts])
