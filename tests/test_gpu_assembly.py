"""GPU: P1 assembly on the device (bd_assemble_p1) against
the host assembly that is bit-identical to the reference
(tests/test_host.py::test_builders_and_assembly_bit_identical_to_reference).

Same sparsity pattern (explicit zeros kept, as the reference's COO -> CSR)
and the SAME values, bit for bit, at the entries whose contributions cancel
in exact arithmetic (exact zeros and the reference's ~1e-32 rounding
residues), so the zero-dropping CSR adds of grounding and K_m give the
host's IC(0) patterns; entries within 1e-13 of the row scale (different summation order); lumped
masses within 1e-13 relative; deterministic run to run; a time step on the
device-assembled system within the BASELINE parity tolerances of the host one."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1711_08708_b200 as bd  # noqa: E402
from paper_1711_08708_b200 import configs  # noqa: E402
from paper_1711_08708_b200.assembly import (DeviceAssembler, Space, assemble_stiffness,  # noqa: E402
                                            lumped_mass_diagonal)
from paper_1711_08708_b200.conductivity import TensorField, default_params  # noqa: E402
from paper_1711_08708_b200.errors import AssemblyError  # noqa: E402
from paper_1711_08708_b200.mesh import build_cube_mesh  # noqa: E402
from paper_1711_08708_b200.precond import build_monodomain_matrix  # noqa: E402

CASES = {
    "cube4": lambda: (build_cube_mesh(4), default_params(3), None),
    "cfg0_16": lambda: (lambda w: (w.mesh, w.params, w.fibers))(configs.cfg0(16)),
    "cfg1_64": lambda: (lambda w: (w.mesh, w.params, w.fibers))(configs.cfg1(64)),
    "cfg2_8": lambda: (lambda w: (w.mesh, w.params, w.fibers))(configs.cfg2((8, 8, 4))),
    "cfg4_12": lambda: (lambda w: (w.mesh, w.params, w.fibers))(configs.cfg4(12)),
    "cfg2_32": lambda: (lambda w: (w.mesh, w.params, w.fibers))(configs.cfg2((32, 32, 16))),
    "cfg4_24": lambda: (lambda w: (w.mesh, w.params, w.fibers))(configs.cfg4(24)),
}


def _same(dev, host):
    assert dev.shape == host.shape
    np.testing.assert_array_equal(dev.indptr, host.indptr)
    np.testing.assert_array_equal(dev.indices, host.indices)
    scale = np.repeat(np.maximum(abs(host).max(axis=1).toarray().ravel(), 1e-300),
                      np.diff(host.indptr))
    assert (np.abs(dev.data - host.data) <= 1e-13 * scale).all()
    # exact-arithmetic cancellations: the same exact zeros and the same
    # rounding residues, bit for bit, so the zero-dropping adds agree
    np.testing.assert_array_equal(dev.data == 0.0, host.data == 0.0)
    tiny = np.abs(host.data) <= 1e-10 * scale
    np.testing.assert_array_equal(dev.data[tiny], host.data[tiny])


@pytest.mark.parametrize("case", sorted(CASES))
def test_device_blocks_match_host(case):
    mesh, params, fibers = CASES[case]()
    da = DeviceAssembler(mesh, params, fibers)
    d = mesh.dim
    for kind, space in (("bar1", Space.FULL), ("bar_e", Space.FULL), ("intra", Space.HEART_ONLY),
                        ("mono", Space.HEART_ONLY)):
        host = assemble_stiffness(mesh, TensorField(params, d, kind, fibers), space)
        _same(da.stiffness(kind), host)
    for space in (Space.FULL, Space.HEART_ONLY):
        np.testing.assert_allclose(da.lumped_mass(space), lumped_mass_diagonal(mesh, space),
                                   rtol=1e-13, atol=0)
    km_h = build_monodomain_matrix(mesh, params, 4000.0, fibers)
    km_d = build_monodomain_matrix(mesh, params, 4000.0, fibers, assembly="device")
    _same(km_d, km_h)
    # the grounded S_1 (the bulk IC(0) input) has the host's pattern
    from paper_1711_08708_b200.precond import regularize_stiffness
    g_h = regularize_stiffness(assemble_stiffness(mesh, TensorField(params, d, "bar1", fibers)))
    g_d = regularize_stiffness(da.stiffness("bar1"))
    _same(g_d.grounded(), g_h.grounded())


def test_device_assembly_deterministic():
    mesh, params, fibers = CASES["cfg2_8"]()
    a = DeviceAssembler(mesh, params, fibers).stiffness("bar1")
    b = DeviceAssembler(mesh, params, fibers).stiffness("bar1")
    assert np.array_equal(a.data, b.data) and np.array_equal(a.indices, b.indices)


def test_degenerate_element_raises():
    mesh = build_cube_mesh(2)
    mesh.elements[0, [1, 2]] = mesh.elements[0, [2, 1]]  # inverted tet
    with pytest.raises(AssemblyError):
        DeviceAssembler(mesh, default_params(3)).stiffness("bar1")


def test_time_step_on_device_assembled_system():
    wl = configs.cfg2((16, 16, 8))
    out = {}
    for mode in ("host", "device"):
        sysm = bd.BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers,
                                       with_extra=False, assembly=mode)
        km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers, assembly=mode)
        pre = bd.BlockLUPreconditioner(sysm, inner="ic0", monodomain_matrix=km)
        st = bd.SimState.resting(sysm.n, sysm.n_heart, wl.ionic)
        its = []
        for _ in range(5):
            st, s = bd.time_step(st, sysm, pre, wl.ionic, wl.protocol, wl.dt, tol=1e-10,
                                 max_iter=5000)
            its.append(s.iterations)
        out[mode] = (its, st.u.cpu().numpy(), st.v.cpu().numpy())
    (ih, uh, vh), (idv, ud, vd) = out["host"], out["device"]
    assert np.all(np.abs(np.asarray(ih) - np.asarray(idv)) <= 2)
    rel = np.sqrt(np.sum((ud - uh) ** 2) + np.sum((vd - vh) ** 2)) / np.sqrt(
        np.sum(uh ** 2) + np.sum(vh ** 2))
    assert rel <= 1e-8


@pytest.mark.parametrize("ortho", [True, False])
def test_transmural_tensors_on_device(ortho):
    """Heart tensors of the transmural-rotation model evaluated on the device
    (bd_tensors_transmural) vs the host TensorField (cos/sin to the last ulps)."""
    wl = configs.cfg2((6, 6, 4))
    params = wl.params if ortho else default_params(3)
    da = DeviceAssembler(wl.mesh, params, wl.fibers)
    tf = TensorField(params, 3, "bar1", wl.fibers)
    hi, he = tf._heart_tensors(wl.mesh.vertices[da.el_h].mean(axis=1))
    for dev, host in ((da.intra, hi), (da.extra, he)):
        assert np.abs(dev - host).max() <= 1e-14 * np.abs(host).max()


def test_row_blocked_assembly_identical(monkeypatch):
    """Meshes too large for one device pass are assembled in row blocks
    (BD_ASSEMBLY_MAX_PAIRS); each block sees every element touching its rows
    in the global element order, so the result equals the one-pass assembly
    bit for bit (values, pattern, masses)."""
    wl = configs.cfg4(20)
    one = DeviceAssembler(wl.mesh, wl.params, wl.fibers)
    ref = {k: one.stiffness(k) for k in ("bar1", "intra", "mono")}
    mref = {s: one.lumped_mass(s) for s in (Space.FULL, Space.HEART_ONLY)}
    monkeypatch.setenv("BD_ASSEMBLY_MAX_PAIRS", "20000")
    blk = DeviceAssembler(wl.mesh, wl.params, wl.fibers)
    for k, a in ref.items():
        b = blk.stiffness(k)
        np.testing.assert_array_equal(a.indptr, b.indptr)
        np.testing.assert_array_equal(a.indices, b.indices)
        np.testing.assert_array_equal(a.data.view(np.int64), b.data.view(np.int64))
    for s, m in mref.items():
        np.testing.assert_array_equal(m.view(np.int64), blk.lumped_mass(s).view(np.int64))
