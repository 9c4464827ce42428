"""Which stiffness entries does the host assembly round to exactly 0.0, and
are they exactly the entries whose element contributions cancel in exact
arithmetic?  For every CSR entry: s = the host sum, b = Σ|contributions|.
Prints the zero count, the entries with 0 < |s|/b < 1e-12 (residues the host
keeps) and the smallest |s|/b among the kept entries (the separation margin
of the device's snap rule, csrc/bd_assembly.cuh)."""
import sys
import time

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1711_08708_b200 import configs  # noqa: E402
from paper_1711_08708_b200.assembly import (CHUNK, Space, _grads_volumes, _select,  # noqa: E402
                                            assemble_stiffness)
from paper_1711_08708_b200.conductivity import TensorField  # noqa: E402


def abs_assembly(mesh, field, space):
    elements, tags, n = _select(mesh, space)
    ar = mesh.dim + 1
    tot = None
    for s in range(0, len(elements), CHUNK):
        el = elements[s:s + CHUNK]
        g, v = _grads_volumes(mesh.vertices, el, mesh.dim)
        sig = field.evaluate_batch(mesh.vertices[el].mean(axis=1), tags[s:s + CHUNK])
        loc = np.einsum("eid,edk,ejk->eij", g, sig, g)
        loc = np.abs(0.5 * (loc + loc.transpose(0, 2, 1)) * v[:, None, None])
        part = sp.coo_matrix((loc.ravel(), (np.repeat(el, ar, axis=1).ravel(),
                                            np.tile(el, (1, ar)).ravel())), shape=(n, n)).tocsr()
        tot = part if tot is None else tot + part
    tot.sum_duplicates()
    tot.sort_indices()
    return tot


def check(name, mesh, field, space):
    t0 = time.time()
    s = assemble_stiffness(mesh, field, space)
    b = abs_assembly(mesh, field, space)
    # host values on b's pattern (0 where the host dropped the entry)
    n = b.shape[0]
    kb = np.repeat(np.arange(n, dtype=np.int64), np.diff(b.indptr)) * n + b.indices
    ks = np.repeat(np.arange(n, dtype=np.int64), np.diff(s.indptr)) * n + s.indices
    pos = np.searchsorted(kb, ks)
    assert np.array_equal(kb[pos], ks), "host pattern not inside the |.| pattern"
    sv = np.zeros(b.nnz)
    sv[pos] = s.data

    class _V:
        data = sv
    s_on_b = _V
    r = np.abs(s_on_b.data) / b.data
    zero = s_on_b.data == 0.0
    small = (~zero) & (r < 1e-12)
    kept = r[~zero]
    print(f"{name}: nnz(b)={b.nnz} nnz(host)={s.nnz} explicit_zero_in_host={(s.data == 0).sum()} "
          f"cancelled={zero.sum()} residues_kept(<1e-12)={small.sum()} "
          f"min kept |s|/b={kept.min():.3e} max cancelled... ({time.time() - t0:.0f}s)", flush=True)
    pos = r[r > 0]
    h, e = np.histogram(np.log10(pos), bins=np.arange(-17, 1))
    print("   log10(|s|/b) histogram:", {int(a): int(c) for a, c in zip(e[:-1], h) if c})
    return r, zero


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "cfg4_48"
    if which.startswith("cfg4_"):
        wl = configs.cfg4(int(which.split("_")[1]))
    elif which == "cfg1":
        wl = configs.cfg1()
    elif which == "cfg2":
        wl = configs.cfg2()
    elif which.startswith("cfg2_"):
        c = int(which.split("_")[1])
        wl = configs.cfg2((c, c, c // 2))
    d = wl.mesh.dim
    for kind, space in (("bar1", Space.FULL), ("intra", Space.HEART_ONLY), ("mono", Space.HEART_ONLY)):
        check(f"{which} {kind}", wl.mesh, TensorField(wl.params, d, kind, wl.fibers), space)
