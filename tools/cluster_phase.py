"""Dev tool: per-level phase cycles of k_trsv_cluster (CTA 0, thread 0)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, '/root/repo')
os.environ["BD_TRSV"] = "cluster"
import torch
import paper_1711_08708_b200 as bd
from paper_1711_08708_b200 import configs, _lib
from paper_1711_08708_b200.assembly import assemble_stiffness
from paper_1711_08708_b200.conductivity import TensorField
from paper_1711_08708_b200.precond import regularize_stiffness
cells = tuple(int(c) for c in sys.argv[1].split(","))
wl = configs.cfg2(cells)
g = regularize_stiffness(assemble_stiffness(wl.mesh, TensorField(wl.params, 3, "bar1", wl.fibers))).grounded()
inner = bd.IncompleteCholesky0(); inner.setup(g, coords=wl.mesh.vertices)
L = _lib.lib(); L.bd_debug_tile_trace.argtypes = [C.c_void_p, C.c_int]
S = 2000
buf = torch.zeros(S * 6, dtype=torch.int64, device='cuda')
y = torch.as_tensor(np.random.default_rng(0).standard_normal(g.shape[0])).cuda()
inner.apply_inverse(y); torch.cuda.synchronize()
L.bd_debug_tile_trace(C.c_void_p(buf.data_ptr()), S)
inner.apply_inverse(y); torch.cuda.synchronize()
L.bd_debug_tile_trace(None, 0)
tr = buf.view(S, 6).cpu().numpy(); tr = tr[tr.sum(axis=1) > 0]
print("levels", len(tr), "median cycles: issue %d compute %d syncthreads %d exports %d cpwait %d cluster.sync %d" % tuple(np.median(tr, axis=0)))
