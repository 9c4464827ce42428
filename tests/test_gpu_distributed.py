"""GPU: the sharded driver with the native backend (sm_100a SpMV and inner
solves) over NCCL at world size 1 reproduces the single-GPU solve."""
import os
import socket

import numpy as np
import pytest

from conftest import csr, golden, rel_l2

pytestmark = pytest.mark.gpu


def test_distributed_native_backend_nccl_world1():
    import torch
    import torch.distributed as dist
    from oracle import bidomain_oracle as orc
    from paper_1711_08708_b200 import distributed as D

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = golden("cfg2s")
        S1, Si, Km = csr(g, "S1"), csr(g, "Si"), csr(g, "Km")
        beta, grounded = orc.regularize(S1)
        part = D.rcb_partition(g["points"], 1)
        lp = D.build_local(S1, Si, g["mass"], g["mh"], g["gamma"], grounded, Km, part, 0, 1)
        comm = D.Comm(dist, torch.device("cuda", 0))
        dsys = D.DistributedSystem(lp, comm, D.NativeBackend())
        for inner in ("jacobi", "ic0"):
            pre = D.DistributedBlockLU(dsys, inner, beta)
            b = torch.as_tensor(np.concatenate([g["sanity_b_u"][lp.owned],
                                                g["sanity_b_v"][lp.owned[: lp.m_own]]])).cuda()
            x, st = D.distributed_pcg(dsys, pre, b, tol=1e-10, max_iter=5000)
            x = x.cpu().numpy()
            xu = np.zeros(lp.n_own)
            xv = np.zeros(lp.m_own)
            xu[lp.owned] = x[: lp.n_own]
            xv[lp.owned[: lp.m_own]] = x[lp.n_own:]
            assert abs(st["iterations"] - int(g[f"sanity_{inner}_iters"])) <= 2, inner
            assert rel_l2(xu, xv, g[f"sanity_{inner}_u"], g[f"sanity_{inner}_v"]) <= 1e-8
    finally:
        dist.destroy_process_group()


def test_sharded_time_step_world1_matches_single_gpu():
    """DistributedSimulation at world size 1 (NCCL) = the single-GPU time step:
    with one block, block-Jacobi IC(0) is the full IC(0)."""
    import torch
    import torch.distributed as dist
    import paper_1711_08708_b200 as bd
    from paper_1711_08708_b200 import configs
    from paper_1711_08708_b200 import distributed as D

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        wl = configs.cfg2((12, 12, 6), steps=5)
        part = D.rcb_partition(wl.mesh.vertices, 1)
        sim = D.DistributedSimulation(wl, part, 0, 1, dist, torch.device("cuda", 0))
        state = sim.resting()
        sysm = bd.BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers)
        pre = bd.BlockLUPreconditioner(sysm, inner="ic0")
        ref = bd.SimState.resting(sysm.n, sysm.n_heart, wl.ionic)
        lp = sim.lp
        for _ in range(5):
            state, st = sim.step(state)
            ref, rst = bd.time_step(ref, sysm, pre, wl.ionic, wl.protocol, wl.dt, tol=wl.tol,
                                    max_iter=20000)
            assert abs(st["iterations"] - rst.iterations) <= 1
            u = np.zeros(lp.n_own)
            u[lp.owned] = state[0].cpu().numpy()
            v = np.zeros(lp.m_own)
            v[lp.owned[: lp.m_own]] = state[1].cpu().numpy()
            assert rel_l2(u, v, ref.u.cpu().numpy(), ref.v.cpu().numpy()) <= 1e-9
    finally:
        dist.destroy_process_group()


def test_local_device_assembly_matches_global():
    """Per-rank assembly ON THE DEVICE (local mesh of the touching elements)
    reproduces the rows of the global host-assembled matrices (3 ranks, the
    heart-in-torso mesh with heart and torso ghosts), to rounding."""
    import numpy as np
    import paper_1711_08708_b200.distributed as D
    from paper_1711_08708_b200 import configs
    from paper_1711_08708_b200.precond import build_monodomain_matrix, regularize_stiffness
    from paper_1711_08708_b200.system import BidomainSystem
    wl = configs.cfg1(32)
    sysm = BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False)
    km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers)
    reg = regularize_stiffness(sysm.stiff_total)
    part = D.rcb_partition(wl.mesh.vertices, 3)
    tot = float(sysm.stiff_total.diagonal().sum())
    for r in range(3):
        ref = D.build_local(sysm.stiff_total, sysm.stiff_intra, sysm.mass_diag,
                            sysm.heart_mass_diag, sysm.gamma, reg.grounded(), km, part, r, 3)
        loc = D.build_local_from_mesh(wl.mesh, wl.params, wl.fibers, wl.dt, part, r, 3,
                                      comm_allreduce=lambda v: [tot], assembly="device")
        assert np.array_equal(ref.owned, loc.owned) and np.array_equal(ref.ghosts, loc.ghosts)
        for a, b in ((ref.S1, loc.S1), (ref.Si, loc.Si), (ref.bulk_block, loc.bulk_block),
                     (ref.schur_block, loc.schur_block)):
            assert a.shape == b.shape
            np.testing.assert_allclose(a.toarray(), b.toarray(), rtol=0,
                                       atol=1e-13 * max(1.0, np.abs(a.data).max()))
        np.testing.assert_allclose(loc.mass, ref.mass, rtol=1e-13)
        np.testing.assert_allclose(loc.heart_mass, ref.heart_mass, rtol=1e-13)
