"""GPU, FULL size BASELINE config 1: the 513² heart-in-torso mesh (263,169
vertices, 16,004 heart vertices), exact inner, tol 1e-10, all 200 steps,
against the CPU oracle run recorded by `tools/oracle_fullsize.py --config
cfg1 --steps 200` (tests/golden/cfg1_exact_oracle.json + _states.npz).

Per step: PCG iterations within ±2, probe traces within 1e-6 relative, full
state norms and the projected full-state rel-L2 within 1e-8; at 14 recorded
steps the exact rel-L2 of a stride-29 subsample within 1e-8 (BASELINE
parity targets).  Both the host-assembled operators (the oracle's inputs)
and the device-assembled ones (the benchmarked path) are checked.  The
oracle's exact inner is the reference with CHOLMOD replaced by SuperLU
(SURVEY §8c); the GPU's is the in-house nested-dissection Cholesky."""
import numpy as np
import pytest

from fullsize_util import StateChecker, load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["host", "device"])
def run(request):
    import paper_1711_08708_b200 as bd
    from paper_1711_08708_b200 import configs
    from paper_1711_08708_b200.precond import build_monodomain_matrix
    ref, states = load("cfg1_exact_oracle")
    if ref is None:
        pytest.skip("cfg1 oracle fixture not recorded")
    wl = configs.cfg1()
    mode = request.param
    sysm = bd.BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False,
                                   assembly=mode)
    km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers, assembly=mode)
    assert sysm.n == ref["n"] and sysm.n_heart == ref["m"]
    assert abs(np.abs(sysm.stiff_total.data).sum() / ref["checksum_S1"] - 1) <= 1e-12
    assert abs(np.abs(km.data).sum() / ref["checksum_Km"] - 1) <= 1e-12
    pre = bd.BlockLUPreconditioner(sysm, inner="exact", monodomain_matrix=km)
    state = bd.SimState.resting(sysm.n, sysm.n_heart, wl.ionic)
    pts = wl.mesh.vertices[: sysm.n_heart]
    chk = StateChecker(ref, states)
    iters, trace = [], []
    for k in range(len(ref["iters"])):
        state, st = bd.time_step(state, sysm, pre, wl.ionic, wl.protocol, wl.dt, tol=wl.tol,
                                 max_iter=20000, heart_points=pts)
        iters.append(st.iterations)
        u, v = state.u.cpu().numpy(), state.v.cpu().numpy()
        trace.append(v[wl.probes])
        chk.check(k + 1, u, v)
    print(f"cfg1 {mode}: worst projected rel-L2 {chk.worst_proj:.2e}, "
          f"worst subsample rel-L2 {chk.worst_sub:.2e}")
    return ref, iters, np.array(trace)


def test_cfg1_fullsize(run):
    ref, iters, trace = run
    assert len(iters) == 200
    assert np.max(np.abs(np.array(iters) - np.array(ref["iters"]))) <= 2
    rt = np.array(ref["trace"])
    assert np.max(np.abs(trace - rt) / np.maximum(np.abs(rt), 1.0)) <= 1e-6
