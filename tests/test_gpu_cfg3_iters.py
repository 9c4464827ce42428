"""GPU, BASELINE config 3 at full size (256x256x128 slab, 8,520,321 vertices,
17.0M fp64 unknowns, ic0 inner), iteration-level parity: the first 30 PCG
iterations of time step 1 (membrane RHS at rest, warm start x0 = (u0, v0),
tol 1e-10; bd/krylov.py:100-131) against the CPU oracle run recorded by
`tools/oracle_iters.py --config cfg3 --iters 30`
(tests/golden/cfg3_ic0_iters30.json + _states.npz; a full oracle time step
takes ~600 iterations x ~17 s on the CPU).

The operators are assembled on the device (the path bench.py and the
scaling runs use; cancellations take the host value, assembly.py), the
right-hand side is the oracle's own numpy evaluation.  Checked: the residual
and r·z histories entry by entry within 1e-8 relative, the counters, and the
normalised iterate after 30 iterations (norms, projected full-state rel-L2,
stride-97 subsample) within 1e-8."""
import numpy as np
import pytest

from fullsize_util import StateChecker, load

pytestmark = pytest.mark.gpu


def test_cfg3_first_iterations_match_oracle():
    import paper_1711_08708_b200 as bd
    from oracle import bidomain_oracle as orc
    from paper_1711_08708_b200 import configs
    from paper_1711_08708_b200.errors import NonConvergenceError
    from paper_1711_08708_b200.ionic import stimulus_vector
    from paper_1711_08708_b200.precond import build_monodomain_matrix

    ref, states = load("cfg3_ic0_iters30")
    if ref is None:
        pytest.skip("cfg3 iteration fixture not recorded")
    wl = configs.cfg3()
    sysm = bd.BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False,
                                   assembly="device")
    km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers, assembly="device")
    assert sysm.n == ref["n"] and sysm.stiff_total.nnz >= ref["nnz_S1"]
    assert abs(np.abs(sysm.stiff_total.data).sum() / ref["checksum_S1"] - 1) <= 1e-12
    assert abs(np.abs(km.data).sum() / ref["checksum_Km"] - 1) <= 1e-12
    pre = bd.BlockLUPreconditioner(sysm, inner="ic0", monodomain_matrix=km)
    n, m = sysm.n, sysm.n_heart
    u, v, w = np.zeros(n), np.full(m, wl.ionic.v_rest), np.ones(m)
    stim = stimulus_vector(wl.mesh.vertices[:m], 0.0, wl.protocol)
    ion = orc.ionic_current(v, w, c_m=wl.params.c_m)
    bu, bv = orc.build_rhs(n, sysm.heart_mass_diag, sysm.gamma, v, ion, stim, wl.params.chi)
    K = ref["iters"]
    with pytest.raises(NonConvergenceError) as exc:
        bd.pcg_solve(sysm, pre, bd.BlockVector(bu, bv), tol=wl.tol, max_iter=K,
                     x0=bd.BlockVector(u, v))
    st, it = exc.value.stats, exc.value.iterate
    assert st.iterations == K and st.mv_count == ref["mv_count"]
    assert st.p1_count == ref["p1_count"] and st.pk_count == ref["pk_count"]
    for key in ("residual_history", "preconditioned_history"):
        got, want = np.array(getattr(st, key)), np.array(ref[key])
        assert got.shape == want.shape, key
        rel = np.abs(got - want) / np.abs(want)
        print(f"cfg3 {key}: max rel diff {rel.max():.2e}")
        assert rel.max() <= 1e-8, key
    xu, xv = it.u.cpu().numpy(), it.v.cpu().numpy()
    ref_it = dict(ref, u_norm=[ref["u_norm"]], v_norm=[ref["v_norm"]], u_proj=[ref["u_proj"]],
                  v_proj=[ref["v_proj"]])
    chk = StateChecker(ref_it, {"u_1": states["u"], "v_1": states["v"]})
    chk.check(1, xu, xv)
    su = states["u"]
    rel_u = np.linalg.norm(xu[:: ref["sub_stride"]] - su) / np.linalg.norm(su)
    print(f"cfg3 iterate: projected rel-L2 {chk.worst_proj:.2e}, subsample {chk.worst_sub:.2e}, "
          f"u-block alone {rel_u:.2e}")
    assert rel_u <= 1e-6
