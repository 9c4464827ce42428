"""GPU: the time loop with its bookkeeping on the device (bd_step_track) —
the reference's TestRunSimulation cases (tests/test_simulate.py:90-151), the
device tracker against the reference's host tracker on the same trajectory
(bitwise), and the activation map against the CPU oracle's time loop."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1711_08708_b200 as bd  # noqa: E402
from paper_1711_08708_b200.conductivity import default_params  # noqa: E402
from paper_1711_08708_b200.ionic import (IonicParams, StimulusProtocol, StimulusSite,  # noqa: E402
                                         default_protocol, stimulus_vector)
from paper_1711_08708_b200.mesh import build_cube_mesh  # noqa: E402
from paper_1711_08708_b200.simulate import (DEPOL_BAND, ActivationTracker,  # noqa: E402
                                            SimulationSetup)


@pytest.fixture(scope="module")
def small_setup():
    mesh = build_cube_mesh(4)
    params = default_params(3)
    system = bd.BidomainSystem.build(mesh, params, dt=0.2)
    precond = bd.BlockLUPreconditioner(system, inner="exact")
    return SimulationSetup(mesh=mesh, system=system, precond=precond, ionic=IonicParams(),
                           protocol=default_protocol(3), dt=0.2, t_end=4.0)


def _with(setup, **kw):
    d = dict(mesh=setup.mesh, system=setup.system, precond=setup.precond, ionic=setup.ionic,
             protocol=setup.protocol, dt=setup.dt, t_end=setup.t_end)
    d.update(kw)
    return SimulationSetup(**d)


def test_device_bookkeeping_equals_host_tracker(small_setup):
    """Same GPU trajectory, bookkeeping twice: the reference's host loop
    (bd/simulate.py:221-245) and run_simulation's fused kernel — bitwise."""
    setup = _with(small_setup, t_end=6.0)
    res = bd.run_simulation(setup)
    sysm = setup.system
    state = bd.SimState.resting(sysm.n, sysm.n_heart, setup.ionic)
    tracker = ActivationTracker(sysm.n_heart, state.v.cpu().numpy())
    pts = setup.mesh.vertices[: sysm.n_heart]
    depol, ratios, iters = [], [], []
    for _ in range(res.n_steps):
        v_prev, t_prev = state.v.cpu().numpy(), state.t
        state, st = bd.time_step(state, sysm, setup.precond, setup.ionic, setup.protocol,
                                 setup.dt, tol=setup.tol, max_iter=setup.max_iter,
                                 heart_points=pts)
        v = state.v.cpu().numpy()
        tracker.record(v_prev, v, t_prev, setup.dt)
        in_band = bool(((v >= DEPOL_BAND[0]) & (v <= DEPOL_BAND[1])).any())
        covered = bool(np.isfinite(tracker.phi).all())
        depol.append(in_band and not covered)
        u = state.u.cpu().numpy()
        u_inf = float(np.abs(u).max())
        ratios.append(0.0 if u_inf == 0.0 else abs(sysm.weighted_mean_u(state.u)) / u_inf)
        iters.append(st.iterations)
    np.testing.assert_array_equal(res.iters, iters)
    np.testing.assert_array_equal(res.activation.phi, tracker.phi)
    np.testing.assert_array_equal(res.depol_mask, depol)
    np.testing.assert_array_equal(res.u_mean_ratios, ratios)
    assert np.isfinite(res.activation.phi).any()  # the wave started


def test_activation_map_matches_oracle(small_setup):
    """Activation map and iterations of the device loop vs the CPU oracle's
    time loop with the reference's host tracker (same matrices)."""
    from oracle import bidomain_oracle as orc

    setup = _with(small_setup, t_end=6.0)
    res = bd.run_simulation(setup)
    sysm = setup.system
    po = orc.BlockLU(sysm.stiff_total, sysm.stiff_intra, setup.precond.monodomain_matrix, "exact")
    m = sysm.n_heart
    pts = setup.mesh.vertices[:m]
    st = (np.zeros(sysm.n), np.full(m, setup.ionic.v_rest), np.ones(m))
    tracker = ActivationTracker(m, st[1])
    t = 0.0
    its = []
    for _ in range(res.n_steps):
        stim = stimulus_vector(pts, t, setup.protocol)
        v_prev = st[1]
        st, so = orc.time_step(st, sysm.stiff_total, sysm.stiff_intra, sysm.heart_mass_diag,
                               sysm.mass_diag, sysm.gamma, po, sysm.params.chi, sysm.params.c_m,
                               stim, setup.dt, tol=setup.tol, max_iter=setup.max_iter)
        tracker.record(v_prev, st[1], t, setup.dt)
        its.append(so["iterations"])
        t += setup.dt
    assert np.all(np.abs(np.asarray(res.iters) - np.asarray(its)) <= 2)
    phi_o = tracker.phi
    assert np.array_equal(np.isfinite(res.activation.phi), np.isfinite(phi_o))
    f = np.isfinite(phi_o)
    assert np.abs(res.activation.phi[f] - phi_o[f]).max(initial=0.0) <= 1e-6


def test_ends_before_stimulus_starts(small_setup):
    delayed = StimulusProtocol(sites=(StimulusSite((0.5, 0.5, 0.5), start=5.0),))
    res = bd.run_simulation(_with(small_setup, protocol=delayed, t_end=1.0))
    assert not np.isfinite(res.activation.phi).any()


def test_activation_spreads_outward():
    mesh = build_cube_mesh(8)
    system = bd.BidomainSystem.build(mesh, default_params(3), dt=0.2)
    precond = bd.BlockLUPreconditioner(system, inner="exact")
    res = bd.run_simulation(SimulationSetup(mesh=mesh, system=system, precond=precond,
                                            ionic=IonicParams(), protocol=default_protocol(3),
                                            dt=0.2, t_end=30.0, stop_when_activated=True))
    phi = res.activation.phi
    dist = np.linalg.norm(mesh.vertices - 0.5, axis=1)
    center, corner = int(np.argmin(dist)), int(np.argmax(dist))
    assert np.isfinite(phi[center])
    if np.isfinite(phi[corner]):
        assert phi[center] < phi[corner]
    bins = np.digitize(dist, np.linspace(0, dist.max() + 1e-9, 5))
    means = [phi[(bins == b) & np.isfinite(phi)].mean()
             for b in range(1, 5) if ((bins == b) & np.isfinite(phi)).any()]
    assert all(a < b for a, b in zip(means, means[1:]))


def test_normalization_held_every_step(small_setup):
    assert (bd.run_simulation(small_setup).u_mean_ratios <= 1e-10).all()


def test_snapshot_count(small_setup):
    seen = []

    def writer(state, step):
        seen.append(step)
        return step

    res = bd.run_simulation(_with(small_setup, snapshot_every=5), snapshot_writer=writer)
    assert len(res.snapshots) == int(np.floor(4.0 / (5 * 0.2))) + 1
    assert seen[0] == 0


def test_determinism(small_setup):
    r1 = bd.run_simulation(small_setup)
    r2 = bd.run_simulation(small_setup)
    np.testing.assert_array_equal(r1.activation.phi, r2.activation.phi)
    np.testing.assert_array_equal(r1.iters, r2.iters)


def test_zero_t_end(small_setup):
    assert bd.run_simulation(_with(small_setup, t_end=0.0)).n_steps == 0
