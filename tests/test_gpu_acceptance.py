"""GPU: the reference's acceptance criteria that exercise the solve
(tests/test_acceptance.py: 6 scaling-study iteration counts, 7 almost-linear
cost, 9 physiology, 10 per-step normalisation), run end to end on the sm_100a
path with the reference's own thresholds.  Criterion 5 (equal-anisotropy
single iteration) is tests/test_gpu_parity.py::test_equal_anisotropy_single_iteration;
criterion 8 (growth-rate formula) is tests/test_io_study.py."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1711_08708_b200 as bd  # noqa: E402
from paper_1711_08708_b200.conductivity import default_params  # noqa: E402
from paper_1711_08708_b200.ionic import IonicParams, default_protocol  # noqa: E402
from paper_1711_08708_b200.mesh import build_cube_mesh  # noqa: E402
from paper_1711_08708_b200.simulate import SimulationSetup  # noqa: E402
from paper_1711_08708_b200.study import BenchConfig, run_scaling_study  # noqa: E402


@pytest.fixture(scope="module")
def scaling_study():
    return run_scaling_study(BenchConfig(series=(8, 16, 32), dim=3, dt_coarsest=0.2, t_end=10.0,
                                         tol=1e-6, inner="exact"))


@pytest.fixture(scope="module")
def cube16_run():
    mesh = build_cube_mesh(16)
    system = bd.BidomainSystem.build(mesh, default_params(3), dt=0.1)
    precond = bd.BlockLUPreconditioner(system, inner="exact")
    setup = SimulationSetup(mesh=mesh, system=system, precond=precond, ionic=IonicParams(),
                            protocol=default_protocol(3), dt=0.1, t_end=200.0, tol=1e-6,
                            stop_when_activated=True)
    return mesh, bd.run_simulation(setup)


def test_criterion_6_scaling_iterations(scaling_study):
    recs = scaling_study.records
    assert all(1.0 <= r.iter_avg <= 10.0 for r in recs), [r.iter_avg for r in recs]
    assert recs[-1].iter_avg / recs[0].iter_avg <= 2.0


def test_criterion_7_almost_linear_cost(scaling_study):
    assert scaling_study.slope_iter_dof <= 1.3, scaling_study.slope_iter_dof


def test_criterion_9_physiology(cube16_run):
    mesh, result = cube16_run
    phi = result.activation.phi
    assert np.isfinite(phi).all()
    pts = mesh.vertices
    on_plane = np.isclose(pts[:, 2], 0.5)
    dist = np.linalg.norm(pts[on_plane, :2] - 0.5, axis=1)
    plane_phi = phi[on_plane]
    bins = np.digitize(dist, np.linspace(0.0, dist.max() + 1e-9, 6))
    means = [plane_phi[bins == b].mean() for b in range(1, 6) if (bins == b).any()]
    assert all(a < b for a, b in zip(means, means[1:])), means

    def phi_at(target):
        return phi[int(np.argmin(((pts - target) ** 2).sum(axis=1)))]

    assert phi_at((0.8125, 0.5, 0.5)) < phi_at((0.5, 0.8125, 0.5))  # faster along the fibres


def test_criterion_10_normalization_every_step(cube16_run):
    _, result = cube16_run
    assert result.n_steps > 0 and float(result.u_mean_ratios.max()) <= 1e-10
