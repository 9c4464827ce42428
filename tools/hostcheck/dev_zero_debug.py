"""GPU debug: compare the device-assembled blocks' exact zeros / residues with
the host assembly per tensor kind (prints counts and a few sample entries)."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1711_08708_b200 import configs  # noqa: E402
from paper_1711_08708_b200.assembly import DeviceAssembler, Space, assemble_stiffness  # noqa: E402
from paper_1711_08708_b200.conductivity import TensorField  # noqa: E402

wl = configs.cfg4(int(sys.argv[1]) if len(sys.argv) > 1 else 12)
for refz in ("0", "1"):
    import os
    os.environ["BD_ASSEMBLY_REFZEROS"] = refz
    da = DeviceAssembler(wl.mesh, wl.params, wl.fibers)
    for kind, space in (("bar1", Space.FULL), ("bar_e", Space.FULL), ("intra", Space.HEART_ONLY),
                        ("mono", Space.HEART_ONLY)):
        h = assemble_stiffness(wl.mesh, TensorField(wl.params, 3, kind, wl.fibers), space)
        d = da.stiffness(kind)
        hz, dz = h.data == 0, d.data == 0
        a = np.flatnonzero(hz & ~dz)
        b = np.flatnonzero(~hz & dz)
        print(f"refzeros={refz} {kind}: host zeros {hz.sum()} dev zeros {dz.sum()} "
              f"host0&dev!=0 {a.size} host!=0&dev0 {b.size}", flush=True)
        for idx in list(a[:3]) + list(b[:3]):
            r = np.searchsorted(h.indptr, idx, side="right") - 1
            print(f"   ({r},{h.indices[idx]}) host {h.data[idx]!r} dev {d.data[idx]!r}")
