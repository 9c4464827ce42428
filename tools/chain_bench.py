"""Dev tool: per-level latency floor of the triangular-solve kernels on a pure
chain (tridiagonal SPD -> bidiagonal IC(0) factor, one row per level)."""
import os, sys
import numpy as np, scipy.sparse as sp
sys.path.insert(0, '/root/repo')
import torch
import paper_1711_08708_b200 as bd
n = 4000
a = sp.diags([4.0 * np.ones(n), -np.ones(n - 1), -np.ones(n - 1)], [0, 1, -1], format="csr")
y = torch.as_tensor(np.random.default_rng(0).standard_normal(n)).cuda()
for mode in ("persist", "syncfree"):
    os.environ["BD_TRSV"] = mode
    ic = bd.IncompleteCholesky0(); ic.setup(a)
    ic.apply_inverse(y); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): ic.apply_inverse(y)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{mode}: {ms*1e3:.0f} us per fwd+bwd over 2x{n} levels -> {ms*1e3/(2*n):.3f} us/level")
