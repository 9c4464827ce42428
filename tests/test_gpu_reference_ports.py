"""GPU: the reference's unit tests of the solve's building blocks, restated on
the sm_100a path (reference tests/test_krylov.py:27-135, tests/test_system.py:60-158,
tests/test_precond.py:17-215), same instances (the 8-cell 2D heart-in-torso
system, dt 0.05) and the same thresholds."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1711_08708_b200 as bd  # noqa: E402
from paper_1711_08708_b200.conductivity import default_params  # noqa: E402
from paper_1711_08708_b200.mesh import build_heart_torso_2d  # noqa: E402
from paper_1711_08708_b200.precond import build_monodomain_matrix, regularize_stiffness  # noqa: E402


@pytest.fixture(scope="module")
def mesh2d():
    return build_heart_torso_2d(8)


@pytest.fixture(scope="module")
def sys2d(mesh2d):
    return bd.BidomainSystem.build(mesh2d, default_params(2), dt=0.05)


@pytest.fixture(scope="module")
def pre_exact(sys2d):
    return bd.BlockLUPreconditioner(sys2d, inner="exact")


def _np(x):
    return x.numpy()


def true_residual(sysm, x, rhs):
    au, av = _np(sysm.apply(x))
    ru, rv = _np(rhs)
    return np.sqrt(np.sum((au - ru) ** 2) + np.sum((av - rv) ** 2)) / rhs.norm()


def range_rhs(sysm, rng):
    u = rng.standard_normal(sysm.n)
    u -= u.mean()
    return bd.BlockVector(u, rng.standard_normal(sysm.n_heart))


# ---- pcg (tests/test_krylov.py) --------------------------------------------------------
def test_tolerance_honored(sys2d, pre_exact, rng):
    for _ in range(3):
        rhs = range_rhs(sys2d, rng)
        x, st = bd.pcg_solve(sys2d, pre_exact, rhs, tol=1e-6)
        assert true_residual(sys2d, x, rhs) <= 1e-6 and st.final_residual <= 1e-6
    _, st = bd.pcg_solve(sys2d, pre_exact, range_rhs(sys2d, rng))  # default tolerance
    assert st.final_residual <= 1e-6


def test_histories(sys2d, pre_exact, rng):
    _, st = bd.pcg_solve(sys2d, pre_exact, range_rhs(sys2d, rng), tol=1e-10)
    assert len(st.residual_history) == st.iterations + 1
    assert all(np.isfinite(st.residual_history))
    _, st = bd.pcg_solve(sys2d, pre_exact, range_rhs(sys2d, rng), tol=1e-12)
    h = st.preconditioned_history
    assert all(cur <= prev * (1 + 1e-12) for prev, cur in zip(h, h[1:]))


def test_solution_normalised_and_kernel_quotient(sys2d, pre_exact, rng):
    rhs = range_rhs(sys2d, rng)
    x, _ = bd.pcg_solve(sys2d, pre_exact, rhs)
    xu, xv = _np(x)
    assert abs(sys2d.weighted_mean_u(x.u)) <= 1e-10 * max(1.0, np.abs(xu).max())
    ru, rv = _np(sys2d.normalize(bd.BlockVector(xu + 17.3, xv.copy())))
    np.testing.assert_allclose(ru, xu, atol=1e-10 * max(1, np.abs(xu).max()))
    np.testing.assert_array_equal(rv, xv)


def test_warm_start_and_counters(sys2d, rng):
    pre = bd.BlockLUPreconditioner(sys2d, inner="exact")
    rhs = range_rhs(sys2d, rng)
    x, st = bd.pcg_solve(sys2d, pre, rhs, tol=1e-8)
    assert st.mv_count == st.iterations + 1
    assert st.p1_count == 2 * st.iterations and st.pk_count == st.iterations
    _, st2 = bd.pcg_solve(sys2d, pre, rhs, tol=1e-6, x0=x)
    assert st2.iterations == 0


def test_counters_are_assignable(sys2d, rng):
    """p1_count / pk_count / si_count are plain attributes in the reference
    (bd/precond.py:272-279): assignment sticks and later applications add on."""
    pre = bd.BlockLUPreconditioner(sys2d, inner="jacobi")
    pre.p1_count, pre.pk_count, pre.si_count = 10, 20, 30
    assert (pre.p1_count, pre.pk_count, pre.si_count) == (10, 20, 30)
    pre.apply_inverse(range_rhs(sys2d, rng))
    assert (pre.p1_count, pre.pk_count, pre.si_count) == (12, 21, 32)
    _, st = bd.pcg_solve(sys2d, pre, range_rhs(sys2d, rng), tol=1e-8, max_iter=5000)
    assert st.p1_count == 2 * st.iterations and pre.p1_count == 12 + 2 * st.iterations
    pre.reset_counters()
    assert (pre.p1_count, pre.pk_count, pre.si_count) == (0, 0, 0)


def test_dump_residuals(sys2d, pre_exact, rng, tmp_path):
    _, st = bd.pcg_solve(sys2d, pre_exact, range_rhs(sys2d, rng))
    path = tmp_path / "residuals.csv"
    bd.dump_residuals(st, path)
    lines = path.read_text().strip().splitlines()
    assert lines[0] == "iter,rel_residual" and len(lines) == len(st.residual_history) + 1


# ---- operator, rhs, normalisation (tests/test_system.py) ------------------------------------
def test_quadratic_form_split_and_nonnegative(sys2d, rng):
    nh = sys2d.n_heart
    diff = (sys2d.stiff_total - sys2d.stiff_extra).tocsr()
    cols = [sys2d.apply(bd.BlockVector(*np.split(np.eye(sys2d.dof)[k], [sys2d.n]))).buf.cpu().numpy()
            for k in range(sys2d.dof)]
    lam_norm = np.linalg.norm(np.array(cols).T, np.inf)
    for _ in range(5):
        u, v = rng.standard_normal(sys2d.n), rng.standard_normal(nh)
        x = bd.BlockVector(u, v)
        quad = x.dot(sys2d.apply(x))
        padded = u.copy()
        padded[:nh] += v
        expected = (u @ (sys2d.stiff_extra @ u) + padded @ (diff @ padded)
                    + sys2d.gamma * (v @ (sys2d.heart_mass_diag * v)))
        assert quad == pytest.approx(expected, rel=1e-10)
    for _ in range(100):
        x = bd.BlockVector(rng.standard_normal(sys2d.n), rng.standard_normal(nh))
        assert x.dot(sys2d.apply(x)) >= -1e-12 * lam_norm * x.dot(x)


def test_build_rhs(sys2d, rng):
    nh = sys2d.n_heart
    z = np.zeros(nh)
    assert sys2d.build_rhs(z, z, z, chi=1500.0).norm() == 0.0
    v, cur = rng.standard_normal(nh), rng.standard_normal(nh)
    ru, rv = _np(sys2d.build_rhs(v, cur, cur, chi=1500.0))
    np.testing.assert_allclose(rv, sys2d.gamma * sys2d.heart_mass_diag * v)
    assert (ru == 0.0).all()
    v, ion, stim = (rng.standard_normal(nh) for _ in range(3))
    ru, rv = _np(sys2d.build_rhs(v, ion, stim, 1500.0))
    np.testing.assert_allclose(rv, sys2d.heart_mass_diag * (sys2d.gamma * v - 1500.0 * (ion - stim)),
                               rtol=1e-14)
    assert (ru == 0.0).all()
    with pytest.raises(ValueError):
        sys2d.build_rhs(np.zeros(3), np.zeros(3), np.zeros(3), chi=1500.0)


def test_normalize(sys2d, rng):
    m = sys2d.mass_diag
    u = rng.standard_normal(sys2d.n)
    u -= (m @ u) / m.sum()
    np.testing.assert_allclose(_np(sys2d.normalize(bd.BlockVector(u, np.zeros(sys2d.n_heart))))[0],
                               u, atol=1e-13)
    cu, _ = _np(sys2d.normalize(bd.BlockVector(3.7 * np.ones(sys2d.n), np.zeros(sys2d.n_heart))))
    np.testing.assert_allclose(cu, 0.0, atol=1e-14)
    for _ in range(5):
        u = rng.standard_normal(sys2d.n) * 40.0
        xu, _ = _np(sys2d.normalize(bd.BlockVector(u, np.zeros(sys2d.n_heart))))
        assert abs(m @ xu) <= 1e-12 * np.abs(m * u).sum()
    v = rng.standard_normal(sys2d.n_heart)
    _, xv = _np(sys2d.normalize(bd.BlockVector(rng.standard_normal(sys2d.n), v)))
    np.testing.assert_array_equal(xv, v)


# ---- preconditioner (tests/test_precond.py) ----------------------------------------------------
def test_monodomain_matrix(mesh2d, sys2d):
    km = build_monodomain_matrix(mesh2d, sys2d.params, sys2d.gamma)
    np.testing.assert_array_equal(km.indptr, sys2d.stiff_intra.indptr)
    np.testing.assert_array_equal(km.indices, sys2d.stiff_intra.indices)
    np.testing.assert_allclose(km @ np.ones(sys2d.n_heart), sys2d.gamma * sys2d.heart_mass_diag,
                               atol=1e-12 * sys2d.gamma * sys2d.heart_mass_diag.max())
    np.linalg.cholesky(km.toarray())
    with pytest.raises(ValueError):
        build_monodomain_matrix(mesh2d, default_params(2), 0.0)
    assert regularize_stiffness(sys2d.stiff_total).beta == pytest.approx(
        sys2d.stiff_total.diagonal().mean())


def test_block_preconditioner_properties(sys2d, rng):
    pre = bd.BlockLUPreconditioner(sys2d, inner="exact")
    assert pre.apply_inverse(bd.BlockVector.zeros(sys2d.n, sys2d.n_heart)).norm() == 0.0
    pre.reset_counters()
    pre.apply_inverse(bd.BlockVector(rng.standard_normal(sys2d.n), rng.standard_normal(sys2d.n_heart)))
    assert (pre.p1_count, pre.pk_count, pre.si_count) == (2, 1, 2)
    for _ in range(5):
        y, z = range_rhs(sys2d, rng), range_rhs(sys2d, rng)
        assert pre.apply_inverse(y).dot(z) == pytest.approx(y.dot(pre.apply_inverse(z)), rel=1e-9)
