"""Data formats and the study harness on either side of the solve: VTK
round trips and the activation CSV (reference tests/test_cli.py:71-107),
growth rates / slopes (tests/test_bench.py:14-48) on the CPU; the scaling
study and the device-timed calibration (tests/test_bench.py:51-115) on the GPU."""
import hashlib

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_1711_08708_b200.assembly import assemble_stiffness
from paper_1711_08708_b200.conductivity import TensorField, default_params
from paper_1711_08708_b200.mesh import build_cube_mesh, build_heart_torso_2d
from paper_1711_08708_b200.study import growth_rate, least_squares_slope
from paper_1711_08708_b200.vtkio import (read_mesh_vtk, write_activation_csv, write_fields_vtk,
                                         write_mesh_vtk)


# ---- CPU: formats -----------------------------------------------------------------
def _digest(mat):
    h = hashlib.sha256()
    for a in (mat.indptr, mat.indices, mat.data):
        h.update(a.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("mesh_fn", [lambda: build_heart_torso_2d(8), lambda: build_cube_mesh(3)])
def test_vtk_mesh_roundtrip_bit_identical(tmp_path, mesh_fn):
    mesh = mesh_fn()
    path = tmp_path / "mesh.vtk"
    write_mesh_vtk(mesh, path)
    back = read_mesh_vtk(path)
    assert back.dim == mesh.dim and back.heart_vertex_count == mesh.heart_vertex_count
    np.testing.assert_array_equal(back.elements, mesh.elements)
    np.testing.assert_array_equal(back.tags, mesh.tags)
    np.testing.assert_array_equal(back.vertices, mesh.vertices)
    p = default_params(mesh.dim)
    assert _digest(assemble_stiffness(mesh, TensorField(p, mesh.dim, "bar1"))) == \
        _digest(assemble_stiffness(back, TensorField(p, mesh.dim, "bar1")))


def test_vtk_fields_file(tmp_path):
    mesh = build_heart_torso_2d(4)
    path = tmp_path / "fields.vtk"
    u = np.linspace(-1, 1, mesh.vertex_count)
    v = np.linspace(-90, 50, mesh.heart_vertex_count)
    write_fields_vtk(mesh, path, u, v)
    back = read_mesh_vtk(path)
    np.testing.assert_array_equal(back.elements, mesh.elements)
    text = path.read_text()
    assert "POINT_DATA" in text and "SCALARS v double 1" in text
    tok = text.split()
    k = tok.index("u")
    got_u = np.asarray(tok[k + 5: k + 5 + mesh.vertex_count], dtype=float)
    np.testing.assert_array_equal(got_u, u)  # 17 significant digits: exact
    k = tok.index("v", k)
    got_v = np.asarray(tok[k + 5: k + 5 + mesh.vertex_count], dtype=float)
    np.testing.assert_array_equal(got_v[: mesh.heart_vertex_count], v)
    assert np.isnan(got_v[mesh.heart_vertex_count:]).all()


def test_activation_csv(tmp_path):
    mesh = build_cube_mesh(2)
    phi = np.full(mesh.heart_vertex_count, np.nan)
    phi[0], phi[3] = 0.0, 1.25
    path = tmp_path / "activation.csv"
    write_activation_csv(mesh, phi, path)
    lines = path.read_text().splitlines()
    assert lines[0] == "vertex_id,x,y,z,phi_ms"
    assert len(lines) == mesh.heart_vertex_count + 1
    assert lines[4].split(",")[-1] == "1.25" and lines[2].split(",")[-1] == "nan"


# ---- CPU: growth rates (reference KATs) -----------------------------------------------
def test_growth_rate_reference_pairs():
    assert growth_rate(1.73, 6.32, 143053, 344408) == pytest.approx(1.47, abs=0.01)
    assert growth_rate(4.34, 8.75, 344408, 684112) == pytest.approx(1.02, abs=0.01)
    assert growth_rate(2.0, 4.0, 1000, 2000) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        growth_rate(0.0, 1.0, 10, 20)
    with pytest.raises(ValueError):
        growth_rate(1.0, 1.0, 20, 10)


@given(cost=st.floats(1e-3, 1e3), factor=st.floats(1.1, 8.0), dof=st.integers(10, 10 ** 7))
@settings(max_examples=100, deadline=None)
def test_proportional_cost_is_exactly_one(cost, factor, dof):
    dof2 = int(dof * factor)
    if dof2 > dof:
        assert growth_rate(cost, cost * dof2 / dof, dof, dof2) == pytest.approx(1.0, abs=1e-9)


def test_least_squares_slope_on_powerlaw():
    dofs = np.array([1e3, 1e4, 1e5])
    assert least_squares_slope(dofs, 3.0 * dofs ** 1.25) == pytest.approx(1.25, abs=1e-12)


# ---- GPU: study harness ----------------------------------------------------------------
@pytest.fixture(scope="module")
def small_study():
    from paper_1711_08708_b200.study import BenchConfig, run_scaling_study

    return run_scaling_study(BenchConfig(series=(4, 8), dim=3, dt_coarsest=0.4, t_end=2.0,
                                         calibration_trials=10))


@pytest.mark.gpu
def test_scaling_study(small_study, tmp_path):
    from paper_1711_08708_b200.study import save_study

    recs = small_study.records
    assert len(recs) == 2 and recs[1].dof > recs[0].dof
    assert np.isfinite(recs[1].r_iter) and np.isfinite(recs[1].r_cpu)
    for r in recs:
        assert 1.0 <= r.iter_avg <= 10.0
        assert r.mv_equivalent > 0.0
    written = save_study(small_study, tmp_path)
    lines = (tmp_path / "scaling.csv").read_text().strip().splitlines()
    assert tmp_path / "scaling.csv" in written
    assert lines[0] == "n,dof,iter_avg,cpu_avg_s,r_iter,r_cpu" and len(lines) == 3
    assert (tmp_path / "calibration.csv").exists()
    res = list(tmp_path.glob("residuals_*.csv"))
    assert res and all(p.read_text().splitlines()[0] == "iter,rel_residual" for p in res)


@pytest.mark.gpu
def test_series_too_short():
    from paper_1711_08708_b200.study import BenchConfig, run_scaling_study

    with pytest.raises(ValueError):
        run_scaling_study(BenchConfig(series=(8,)))


@pytest.mark.gpu
def test_calibration():
    import paper_1711_08708_b200 as bd
    from paper_1711_08708_b200.study import calibrate_costs

    mesh = build_cube_mesh(8)
    system = bd.BidomainSystem.build(mesh, default_params(3), dt=0.2)
    pre = bd.BlockLUPreconditioner(system, inner="exact")
    with pytest.raises(ValueError):
        calibrate_costs(system, pre, trials=3)
    rng = np.random.default_rng(5)
    a = calibrate_costs(system, pre, trials=15, rng=rng)
    b = calibrate_costs(system, pre, trials=15, rng=rng)
    assert a > 0 and abs(a - b) <= 0.3 * max(a, b)
    small = bd.BidomainSystem.build(build_cube_mesh(4), default_params(3), dt=0.2)
    assert calibrate_costs(small, bd.BlockLUPreconditioner(small, inner="jacobi"), trials=10) > 0
