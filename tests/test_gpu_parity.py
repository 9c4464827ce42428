"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden outputs and the oracle, on identical inputs.

Tolerances: SpMV / preconditioner applications 1e-12 relative (different
summation order than scipy); IC(0) factors bit-exact; PCG iteration counts
equal on the small instances and within ±2 on the time-stepping runs;
per-step solution rel-L2 ≤ 1e-8; probe traces ≤ 1e-6 relative (BASELINE
parity targets)."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import SMALL, csr, golden, rel_l2

pytestmark = pytest.mark.gpu

import paper_1711_08708_b200 as bd  # noqa: E402
from oracle import bidomain_oracle as orc  # noqa: E402


def make_system(g):
    se = csr(g, "Se") if "Se_data" in g else None
    return bd.BidomainSystem(csr(g, "S1"), csr(g, "Si"), se, g["mass"], g["mh"],
                             float(g["gamma"]))


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


# ---- operator ------------------------------------------------------------------
@pytest.mark.parametrize("case", SMALL)
def test_lambda_apply(case):
    g = golden(case)
    sysm = make_system(g)
    q = sysm.apply(bd.BlockVector(g["x_u"], g["x_v"]))
    qu, qv = q.numpy()
    assert rel(qu, g["lam_u"]) <= 1e-13 and rel(qv, g["lam_v"]) <= 1e-13
    nu, nv = sysm.normalize(bd.BlockVector(g["x_u"], g["x_v"])).numpy()
    assert rel(nu, g["norm_u"]) <= 1e-13 and np.array_equal(nv, g["x_v"])
    assert abs(sysm.weighted_mean_u(nu)) <= 1e-14 * np.abs(nu).max()


@pytest.mark.parametrize("case", SMALL)
def test_lambda_kernel_and_symmetry(case, rng):
    g = golden(case)
    sysm = make_system(g)
    out = sysm.apply(bd.BlockVector(np.ones(sysm.n), np.zeros(sysm.n_heart)))
    scale = max(1.0, abs(sysm.stiff_total).sum(axis=1).max())
    assert out.norm() <= 1e-13 * scale
    for _ in range(3):
        x = bd.BlockVector(rng.standard_normal(sysm.n), rng.standard_normal(sysm.n_heart))
        y = bd.BlockVector(rng.standard_normal(sysm.n), rng.standard_normal(sysm.n_heart))
        assert sysm.apply(x).dot(y) == pytest.approx(x.dot(sysm.apply(y)), rel=1e-12)


def test_dimension_mismatch():
    g = golden("small_coupled2d")
    sysm = make_system(g)
    with pytest.raises(ValueError):
        sysm.apply(bd.BlockVector(np.zeros(sysm.n + 1), np.zeros(sysm.n_heart)))


def test_spmv_matches_scipy(rng):
    g = golden("cfg0")
    from paper_1711_08708_b200.system import NativeCsr
    from paper_1711_08708_b200 import _lib
    a = csr(g, "S1")
    nc = NativeCsr(_lib.Context.default(), a)
    x = rng.standard_normal(a.shape[1])
    y = nc.matvec(x).cpu().numpy()
    assert rel(y, a @ x) <= 1e-13


# ---- preconditioner ------------------------------------------------------------------
@pytest.mark.parametrize("case", SMALL)
@pytest.mark.parametrize("inner", ["ic0", "jacobi", "exact"])
def test_block_lu_apply(case, inner):
    g = golden(case)
    sysm = make_system(g)
    pre = bd.BlockLUPreconditioner(sysm, inner=inner, monodomain_matrix=csr(g, "Km"))
    assert pre.regularized.beta == float(g["beta"])
    pre.reset_counters()
    zu, zv = pre.apply_inverse(bd.BlockVector(g["y_u"], g["y_v"])).numpy()
    assert (pre.p1_count, pre.pk_count, pre.si_count) == (2, 1, 2)
    tol = 1e-12 if inner != "exact" else 1e-11
    assert rel(zu, g[f"pinv_{inner}_u"]) <= tol and rel(zv, g[f"pinv_{inner}_v"]) <= tol
    one = pre._bulk_inverse(np.ones(sysm.n))
    assert np.array_equal(one, np.ones(sysm.n) / pre.regularized.beta)  # bitwise (test_precond.py:72-76)
    zero = pre.apply_inverse(bd.BlockVector.zeros(sysm.n, sysm.n_heart))
    assert zero.norm() == 0.0


@pytest.mark.parametrize("case", SMALL)
def test_ic0_factor_bitwise(case):
    g = golden(case)
    sysm = make_system(g)
    pre = bd.BlockLUPreconditioner(sysm, inner="ic0", monodomain_matrix=csr(g, "Km"))
    for key, inner in (("L1", pre.inner_bulk), ("LK", pre.inner_schur)):
        low = inner.lower_factor
        ref = csr(g, key)
        assert np.array_equal(low.indptr, ref.indptr) and np.array_equal(low.indices, ref.indices)
        assert np.array_equal(low.data, ref.data)


def test_ic0_known_answers(rng):
    g = golden("ic0_kat")
    ic = bd.IncompleteCholesky0()
    ic.setup(csr(g, "tri"))
    assert np.array_equal(ic.lower_factor.data, g["tri_L_data"])
    y = rng.standard_normal(15)
    np.testing.assert_allclose(csr(g, "tri") @ ic.apply_inverse(y), y, atol=1e-10)
    ic = bd.IncompleteCholesky0()
    ic.setup(csr(g, "relaxed"))
    assert ic.restarts_used == int(g["relaxed_restarts"]) and 0 < ic.restarts_used <= 20
    assert np.array_equal(ic.lower_factor.data, g["relaxed_L_data"])
    kershaw = sp.csr_matrix(np.array([[3.0, -2.0, 0.0, 2.0], [-2.0, 3.0, -2.0, 0.0],
                                      [0.0, -2.0, 3.0, -2.0], [2.0, 0.0, -2.0, 3.0]]))
    with pytest.raises(bd.PreconditionerError):
        bd.IncompleteCholesky0().setup(kershaw)
    with pytest.raises(bd.PreconditionerError):
        bd.Jacobi().setup(sp.diags([0.0, 1.0]).tocsr())
    with pytest.raises(bd.PreconditionerError):  # missing diagonal (bd/precond.py:163-166)
        bd.IncompleteCholesky0().setup(sp.csr_matrix(np.array([[1.0, 0.5], [0.5, 0.0]])))
    d = 1.0 + rng.random(20)
    jac = bd.Jacobi()
    jac.setup(sp.diags(d).tocsr())
    y = rng.standard_normal(20)
    assert np.array_equal(jac.apply_inverse(y), (1.0 / d) * y)


@pytest.mark.parametrize("name", ["exact", "ic0", "jacobi"])
def test_inner_contract(name, rng):
    """Symmetric, positive and linear (bd/precond.py:10-13; tests/test_precond.py:89-118)."""
    g = golden("small_coupled2d")
    km = csr(g, "Km")
    inner = bd.make_inner(name)
    inner.setup(km)
    n = km.shape[0]
    for _ in range(5):
        y, z = rng.standard_normal(n), rng.standard_normal(n)
        assert inner.apply_inverse(y) @ z == pytest.approx(y @ inner.apply_inverse(z), rel=1e-10)
        assert y @ inner.apply_inverse(y) > 0.0
    y, z = rng.standard_normal(n), rng.standard_normal(n)
    comb = inner.apply_inverse(2.0 * y - 3.0 * z)
    parts = 2.0 * inner.apply_inverse(y) - 3.0 * inner.apply_inverse(z)
    np.testing.assert_allclose(comb, parts, atol=1e-10 * np.abs(parts).max())
    if name == "exact":
        x = inner.apply_inverse(y)
        assert np.linalg.norm(km @ x - y) <= 1e-12 * np.linalg.norm(y)


# ---- PCG --------------------------------------------------------------------------------
@pytest.mark.parametrize("case", SMALL)
@pytest.mark.parametrize("inner", ["ic0", "jacobi", "exact"])
def test_pcg_matches_reference(case, inner):
    g = golden(case)
    sysm = make_system(g)
    pre = bd.BlockLUPreconditioner(sysm, inner=inner, monodomain_matrix=csr(g, "Km"))
    x, st = bd.pcg_solve(sysm, pre, bd.BlockVector(g["b_u"], g["b_v"]), tol=1e-10, max_iter=2000)
    assert st.iterations == int(g[f"pcg_{inner}_iters"])
    assert [st.mv_count, st.p1_count, st.pk_count] == list(g[f"pcg_{inner}_counts"])
    assert len(st.residual_history) == st.iterations + 1
    np.testing.assert_allclose(st.residual_history, g[f"pcg_{inner}_res"], rtol=1e-6, atol=1e-13)
    xu, xv = x.numpy()
    assert rel_l2(xu, xv, g[f"pcg_{inner}_u"], g[f"pcg_{inner}_v"]) <= 1e-10
    # true residual honoured and mass-normalised output
    qu, qv = (sysm.apply(x)).numpy()
    tr = rel_l2(qu, qv, g["b_u"], g["b_v"])
    assert tr <= 1e-9
    assert abs(sysm.weighted_mean_u(xu)) <= 1e-10 * max(1.0, np.abs(xu).max())
    if inner == "exact":  # preconditioned measure non-increasing (tests/test_krylov.py:57-64)
        hist = st.preconditioned_history
        for a, b in zip(hist, hist[1:]):
            assert b <= a * (1 + 1e-10)


def _coupled():
    g = golden("small_coupled2d")
    sysm = make_system(g)
    return g, sysm


def test_pcg_zero_rhs_and_invalid_tol():
    g, sysm = _coupled()
    pre = bd.BlockLUPreconditioner(sysm, inner="exact", monodomain_matrix=csr(g, "Km"))
    x, st = bd.pcg_solve(sysm, pre, bd.BlockVector.zeros(sysm.n, sysm.n_heart))
    assert st.iterations == 0 and st.converged and x.norm() == 0.0
    assert st.residual_history == [0.0] and st.mv_count == 0
    with pytest.raises(ValueError):
        bd.pcg_solve(sysm, pre, bd.BlockVector.zeros(sysm.n, sysm.n_heart), tol=0.0)


def test_pcg_warm_start_and_counters():
    g, sysm = _coupled()
    pre = bd.BlockLUPreconditioner(sysm, inner="exact", monodomain_matrix=csr(g, "Km"))
    rhs = bd.BlockVector(g["b_u"], g["b_v"])
    x, st = bd.pcg_solve(sysm, pre, rhs, tol=1e-8)
    assert st.mv_count == st.iterations + 1
    assert st.p1_count == 2 * st.iterations and st.pk_count == st.iterations
    x2, st2 = bd.pcg_solve(sysm, pre, rhs, tol=1e-6, x0=x)
    assert st2.iterations == 0 and st2.mv_count == 1 and st2.p1_count == 0


def test_pcg_max_iter_error_carries_stats():
    g, sysm = _coupled()
    pre = bd.BlockLUPreconditioner(sysm, inner="jacobi", monodomain_matrix=csr(g, "Km"))
    with pytest.raises(bd.NonConvergenceError) as err:
        bd.pcg_solve(sysm, pre, bd.BlockVector(g["b_u"], g["b_v"]), tol=1e-14, max_iter=2)
    st = err.value.stats
    assert st is not None and st.iterations == 2 and not st.converged
    assert st.p1_count == 2 * 3 and len(st.residual_history) == 3
    # the oracle agrees on every counter of the failed solve
    po = orc.BlockLU(sysm.stiff_total, sysm.stiff_intra, csr(g, "Km"), "jacobi")
    with pytest.raises(orc.OracleNoConvergence) as oerr:
        orc.pcg(sysm.stiff_total, sysm.stiff_intra, sysm.heart_mass_diag, sysm.mass_diag,
                sysm.gamma, po, g["b_u"], g["b_v"], tol=1e-14, max_iter=2)
    assert oerr.value.stats["p1_count"] == st.p1_count
    assert oerr.value.stats["mv_count"] == st.mv_count


def test_pcg_breakdown_on_indefinite_operator():
    g, sysm = _coupled()
    bad = bd.BidomainSystem(sysm.stiff_total, sysm.stiff_intra, None, sysm.mass_diag,
                            sysm.heart_mass_diag, -1e6)
    pre = bd.BlockLUPreconditioner(bad, inner="jacobi", monodomain_matrix=csr(g, "Km"))
    with pytest.raises(bd.NumericalBreakdownError) as err:
        bd.pcg_solve(bad, pre, bd.BlockVector(g["b_u"], g["b_v"]), tol=1e-12, max_iter=100)
    assert err.value.stats is not None


def test_equal_anisotropy_single_iteration():
    """Surrogate equals the true Schur block → 1 iteration to machine
    precision (tests/test_krylov.py:117-124, bd/verify.py:82-100)."""
    for mesh, d in ((bd.build_square_mesh(4), 2), (bd.build_cube_mesh(2), 3)):
        base = bd.default_params(d)
        p = bd.default_params(d, g_i_l=base.g_i_l, g_i_t=base.g_i_t, g_e_l=2 * base.g_i_l,
                              g_e_t=2 * base.g_i_t)
        sysm = bd.BidomainSystem.build(mesh, p, 0.1)
        pre = bd.BlockLUPreconditioner(sysm, inner="exact")
        rng = np.random.default_rng(7)
        rhs = bd.BlockVector(np.zeros(sysm.n), rng.standard_normal(sysm.n_heart))
        x, st = bd.pcg_solve(sysm, pre, rhs, tol=1e-12, max_iter=10)
        qu, qv = sysm.apply(x).numpy()
        ru, rv = rhs.numpy()
        assert st.iterations == 1
        assert rel_l2(qu, qv, ru, rv) <= 1e-12


# ---- membrane kernels ------------------------------------------------------------------
def test_membrane_kernels_bitwise(rng):
    import torch
    from paper_1711_08708_b200.simulate import gate_update, membrane_rhs
    g, sysm = _coupled()
    m = sysm.n_heart
    ion_p = bd.IonicParams()
    v = rng.uniform(-90, 50, m)
    w = rng.uniform(0, 1, m)
    pts = rng.uniform(0, 1, (m, 2))
    proto = bd.StimulusProtocol(sites=(bd.StimulusSite((0.5, 0.5)),), radius=0.3,
                                amplitude=140.0, duration=2.0)
    sysm.params = bd.default_params(2, chi=200.0)
    rhs = membrane_rhs(sysm, torch.as_tensor(v).cuda(), torch.as_tensor(w).cuda(), proto, 1.0,
                       ion_p, pts)
    ion = bd.ionic_current(v, w, ion_p, 1.0)
    stim = bd.stimulus_vector(pts, 1.0, proto)
    ref = sysm.heart_mass_diag * (sysm.gamma * v - 200.0 * (ion - stim))
    ru, rv = rhs.numpy()
    assert np.array_equal(rv, ref) and np.array_equal(ru, np.zeros(sysm.n))
    wn = gate_update(sysm, torch.as_tensor(w).cuda(), torch.as_tensor(v).cuda(), 0.05, ion_p)
    assert np.array_equal(wn.cpu().numpy(), bd.update_gate(w, v, 0.05, ion_p))


# ---- time stepping against the reference runs --------------------------------------------
def _protocol(case, g):
    if case == "cfg0":
        return bd.StimulusProtocol(sites=(bd.StimulusBox((-np.inf, -np.inf), (0.1, np.inf)),),
                                   amplitude=140.0, duration=2.0)
    if case == "cfg1s":
        return bd.StimulusProtocol(sites=(bd.StimulusSite((6.5, 10.0)),), radius=0.3,
                                   amplitude=140.0, duration=2.0)
    return bd.StimulusProtocol(sites=(bd.StimulusSite((0.0, 0.0, 0.0)),),
                               radius=float(g["stim_radius"]), amplitude=140.0, duration=2.0)


def run_case(case, inner, steps):
    g = golden(case)
    sysm = make_system(g)
    sysm.params = bd.default_params(2, chi=200.0, c_m=1.0)
    pre = bd.BlockLUPreconditioner(sysm, inner=inner, monodomain_matrix=csr(g, "Km"))
    ion = bd.IonicParams()
    proto = _protocol(case, g)
    state = bd.SimState.resting(sysm.n, sysm.n_heart, ion)
    iters, traces, states = [], [], {}
    for k in range(steps):
        state, st = bd.time_step(state, sysm, pre, ion, proto, 0.05, tol=1e-10, max_iter=5000,
                                 heart_points=g["points"])
        iters.append(st.iterations)
        v = state.v.cpu().numpy()
        traces.append(v[g["probes"]])
        if (k + 1) in (10, 50, 100):
            states[k + 1] = (state.u.cpu().numpy(), v, state.w.cpu().numpy())
    return g, np.array(iters), np.array(traces), states


STEP_CASES = [("cfg0", "exact", 100), ("cfg0", "ic0", 100), ("cfg0", "jacobi", 100),
              ("cfg1s", "exact", 40), ("cfg1s", "ic0", 40),
              ("cfg2s", "ic0", 40), ("cfg2s", "exact", 40), ("cfg2s", "jacobi", 40)]


@pytest.mark.parametrize("case,inner,steps", STEP_CASES)
def test_time_steps_match_reference(case, inner, steps):
    g, iters, traces, states = run_case(case, inner, steps)
    ref_iters = g[f"steps_{inner}_iters"][:steps]
    assert np.max(np.abs(iters - ref_iters)) <= 2, (iters, ref_iters)
    ref_tr = g[f"steps_{inner}_trace"][1:steps + 1]
    scale = np.maximum(np.abs(ref_tr), 1.0)
    assert np.max(np.abs(traces - ref_tr) / scale) <= 1e-6
    for k, (u, v, w) in states.items():
        if f"steps_{inner}_u{k}" in g:
            assert rel_l2(u, v, g[f"steps_{inner}_u{k}"], g[f"steps_{inner}_v{k}"]) <= 1e-8
            np.testing.assert_allclose(w, g[f"steps_{inner}_w{k}"], rtol=0, atol=1e-8)


def test_determinism_bitwise():
    _, it1, tr1, st1 = run_case("cfg0", "ic0", 10)
    _, it2, tr2, st2 = run_case("cfg0", "ic0", 10)
    assert np.array_equal(it1, it2) and np.array_equal(tr1, tr2)
    for a, b in zip(st1[10], st2[10]):
        assert np.array_equal(a, b)


def test_resting_state_is_equilibrium():
    g = golden("small_cube2")
    sysm = make_system(g)
    sysm.params = bd.default_params(3)
    pre = bd.BlockLUPreconditioner(sysm, inner="exact", monodomain_matrix=csr(g, "Km"))
    ion = bd.IonicParams()
    state = bd.SimState.resting(sysm.n, sysm.n_heart, ion)
    new, st = bd.time_step(state, sysm, pre, ion, bd.StimulusProtocol(sites=()), 0.2,
                           heart_points=np.zeros((sysm.n_heart, 3)))
    np.testing.assert_allclose(new.v.cpu().numpy(), -90.0, atol=1e-10)
    np.testing.assert_allclose(new.u.cpu().numpy(), 0.0, atol=1e-10)
    assert np.array_equal(new.w.cpu().numpy(), np.ones(sysm.n_heart))
    assert st.iterations <= 1


@pytest.mark.parametrize("case,inners", [("cfg0", ("exact", "ic0", "jacobi")),
                                         ("cfg1s", ("exact", "ic0")),
                                         ("cfg2s", ("ic0", "exact", "jacobi"))])
def test_sanity_solve(case, inners):
    g = golden(case)
    sysm = make_system(g)
    for inner in inners:
        pre = bd.BlockLUPreconditioner(sysm, inner=inner, monodomain_matrix=csr(g, "Km"))
        x, st = bd.pcg_solve(sysm, pre, bd.BlockVector(g["sanity_b_u"], g["sanity_b_v"]),
                             tol=1e-10, max_iter=5000)
        assert abs(st.iterations - int(g[f"sanity_{inner}_iters"])) <= 2, inner
        xu, xv = x.numpy()
        assert rel_l2(xu, xv, g[f"sanity_{inner}_u"], g[f"sanity_{inner}_v"]) <= 1e-8
