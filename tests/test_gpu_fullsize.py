"""GPU, FULL size BASELINE config 2 (128x128x64 slab, 1,081,665 vertices,
2.16M unknowns, ic0, tol 1e-10) against the CPU oracle run on identical
inputs (tests/golden/cfg2_ic0_oracle.json + _states.npz, recorded by
`tools/oracle_fullsize.py --config cfg2 --steps 50`):

* every recorded step (BD_FULLSIZE_STEPS caps it): PCG iterations within ±2,
  probe traces within 1e-6 relative, full-state norms and the projected
  full-state rel-L2 (tests/fullsize_util.py) within 1e-8;
* at the recorded subsample steps: exact rel-L2 of a stride-29 subsample
  within 1e-8;
* for BOTH the host-assembled operators (the oracle's inputs) and the
  device-assembled ones that bench.py times;
* size-independent properties at full size: true residual of a fresh sanity
  solve, mass normalisation."""
import os

import numpy as np
import pytest

from fullsize_util import StateChecker, load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["host", "device"])
def run(request):
    import paper_1711_08708_b200 as bd
    from paper_1711_08708_b200 import configs
    from paper_1711_08708_b200.precond import build_monodomain_matrix
    ref, states = load("cfg2_ic0_oracle")
    if ref is None:
        pytest.skip("full-size oracle fixture not recorded")
    mode = request.param
    wl = configs.cfg2()
    sysm = bd.BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False,
                                   assembly=mode)
    km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers, assembly=mode)
    # same operator: sizes and entry checksums (the device keeps the explicit
    # zeros that the chunked host sum drops, so nnz may only grow)
    assert sysm.n == ref["n"] and sysm.stiff_total.nnz >= ref["nnz_S1"]
    assert abs(np.abs(sysm.stiff_total.data).sum() / ref["checksum_S1"] - 1) <= 1e-12
    assert abs(np.abs(km.data).sum() / ref["checksum_Km"] - 1) <= 1e-12
    pre = bd.BlockLUPreconditioner(sysm, inner="ic0", monodomain_matrix=km)
    state = bd.SimState.resting(sysm.n, sysm.n_heart, wl.ionic)
    pts = wl.mesh.vertices[: sysm.n_heart]
    steps = min(len(ref["iters"]), int(os.environ.get("BD_FULLSIZE_STEPS", "50")))
    chk = StateChecker(ref, states)
    iters, trace = [], []
    for k in range(steps):
        state, st = bd.time_step(state, sysm, pre, wl.ionic, wl.protocol, wl.dt, tol=wl.tol,
                                 max_iter=20000, heart_points=pts)
        iters.append(st.iterations)
        u, v = state.u.cpu().numpy(), state.v.cpu().numpy()
        trace.append(v[wl.probes])
        chk.check(k + 1, u, v)
    print(f"cfg2 {mode}: {steps} steps, worst projected rel-L2 {chk.worst_proj:.2e}, "
          f"worst subsample rel-L2 {chk.worst_sub:.2e}")
    return ref, iters, np.array(trace), sysm, pre


def test_fullsize_iterations_and_traces(run):
    ref, iters, trace, *_ = run
    k = len(iters)
    assert np.max(np.abs(np.array(iters) - np.array(ref["iters"][:k]))) <= 2
    rt = np.array(ref["trace"][:k])
    assert np.max(np.abs(trace - rt) / np.maximum(np.abs(rt), 1.0)) <= 1e-6


def test_fullsize_properties(run):
    """True residual of a fresh sanity solve and the mass normalisation at full size."""
    import paper_1711_08708_b200 as bd
    from paper_1711_08708_b200 import configs
    ref, iters, trace, sysm, pre = run
    bu, bv = configs.sanity_rhs(sysm.n, sysm.n_heart, seed=0)
    rhs = bd.BlockVector(bu, bv)
    x, st = bd.pcg_solve(sysm, pre, rhs, tol=1e-10, max_iter=20000)
    assert st.converged and len(st.residual_history) == st.iterations + 1
    q = sysm.apply(x)
    r = (q.buf - rhs.buf).norm().item() / rhs.buf.norm().item()
    assert r <= 1e-9
    xu = x.u.cpu().numpy()
    assert abs(sysm.weighted_mean_u(x.u)) <= 1e-10 * max(1.0, np.abs(xu).max())
