"""GPU: the sharded driver's native path (NativeShard: bd_shard_* kernels,
sm_100a SpMV and block-Jacobi inner solves; ShardSolver: halos, the four
all-reduces, the CUDA-graph loop).

* world size 1 over NCCL: equals the single-GPU solve / time step;
* world size 2 with BOTH ranks on cuda:0 (this pool has one GPU per box):
  the native kernels of two real sub-blocks with real halos, the halos and
  partial sums staged through host memory over gloo (HostStagedComm, test
  only; no kernel ever waits on the other rank's kernels), against the
  oracle and the single-GPU path: jacobi shards exactly (iterations +-2,
  rel-L2 1e-8), block-Jacobi IC(0) changes the preconditioner (solution
  1e-8 at tol 1e-10, iterations reported and bounded)."""
import os
import socket

import numpy as np
import pytest

from conftest import csr, golden, rel_l2

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _nccl1():
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    return dist


def test_native_shard_nccl_world1():
    import torch
    from oracle import bidomain_oracle as orc
    from paper_1711_08708_b200 import distributed as D

    dist = _nccl1()
    try:
        g = golden("cfg2s")
        S1, Si, Km = csr(g, "S1"), csr(g, "Si"), csr(g, "Km")
        beta, grounded = orc.regularize(S1)
        part = D.rcb_partition(g["points"], 1)
        lp = D.build_local(S1, Si, g["mass"], g["mh"], g["gamma"], grounded, Km, part, 0, 1)
        comm = D.Comm(dist, torch.device("cuda", 0))
        for inner in ("jacobi", "ic0"):
            solver = D.ShardSolver(lp, comm, D.NativeShard(lp, inner))
            b = torch.as_tensor(np.concatenate([g["sanity_b_u"][lp.owned],
                                                g["sanity_b_v"][lp.owned[: lp.m_own]]])).cuda()
            for graph in (False, True):
                x, st = solver.solve(b, tol=1e-10, max_iter=5000, graph=graph)
                x = x.cpu().numpy()
                xu, xv = np.zeros(lp.n_own), np.zeros(lp.m_own)
                xu[lp.owned] = x[: lp.n_own]
                xv[lp.owned[: lp.m_own]] = x[lp.n_own:]
                assert abs(st["iterations"] - int(g[f"sanity_{inner}_iters"])) <= 2, inner
                assert len(st["residual_history"]) == st["iterations"] + 1
                assert rel_l2(xu, xv, g[f"sanity_{inner}_u"], g[f"sanity_{inner}_v"]) <= 1e-8
            # zero right-hand side: no iteration, x = 0 (bd/krylov.py:69-72)
            x0, st0 = solver.solve(b * 0.0, tol=1e-10, max_iter=50)
            assert st0["iterations"] == 0 and float(x0.abs().max()) == 0.0
    finally:
        dist.destroy_process_group()


def test_sharded_time_step_world1_matches_single_gpu():
    """DistributedSimulation at world size 1 (NCCL, graph-captured loop) = the
    single-GPU time step: with one block, block-Jacobi IC(0) is the full IC(0)."""
    import torch
    import paper_1711_08708_b200 as bd
    from paper_1711_08708_b200 import configs
    from paper_1711_08708_b200 import distributed as D

    dist = _nccl1()
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
        assert st["graph"], st.get("graph_error")
    finally:
        dist.destroy_process_group()


# ---- two ranks on one GPU -------------------------------------------------------------
def _host_staged_comm(D, dist, device):
    return D.HostStagedComm(dist, device)


def _problem(name):
    from oracle import bidomain_oracle as orc
    if name == "slab":
        g = golden("cfg2s")
        S1, Si, Km = csr(g, "S1"), csr(g, "Si"), csr(g, "Km")
        return dict(S1=S1, Si=Si, Km=Km, mass=g["mass"], mh=g["mh"], gamma=float(g["gamma"]),
                    pts=g["points"], bu=g["sanity_b_u"], bv=g["sanity_b_v"],
                    grounded=orc.regularize(S1)[1])
    from paper_1711_08708_b200 import configs
    from paper_1711_08708_b200.precond import build_monodomain_matrix
    from paper_1711_08708_b200.system import BidomainSystem
    wl = configs.cfg4(14)  # 3D heart-in-torso box: heart and torso ghosts
    sysm = BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False)
    km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers)
    bu, bv = configs.sanity_rhs(sysm.n, sysm.n_heart, seed=5)
    return dict(S1=sysm.stiff_total, Si=sysm.stiff_intra, Km=km, mass=sysm.mass_diag,
                mh=sysm.heart_mass_diag, gamma=sysm.gamma, pts=wl.mesh.vertices, bu=bu, bv=bv,
                grounded=orc.regularize(sysm.stiff_total)[1])


def _worker(rank, world, port, name, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_08708_b200 import distributed as D
        P = _problem(name)
        part = D.rcb_partition(P["pts"], world)
        lp = D.build_local(P["S1"], P["Si"], P["mass"], P["mh"], P["gamma"], P["grounded"],
                           P["Km"], part, rank, world)
        lp.coords = np.ascontiguousarray(P["pts"][lp.owned], dtype=float)
        comm = _host_staged_comm(D, dist, torch.device("cuda", 0))
        b = torch.as_tensor(np.concatenate([P["bu"][lp.owned],
                                            P["bv"][lp.owned[: lp.m_own]]])).cuda()
        out = {"owned": lp.owned, "m_own": lp.m_own, "ghosts": lp.ghosts.size,
               "heart_ghosts": lp.m_ghost}
        for inner in ("jacobi", "ic0"):
            solver = D.ShardSolver(lp, comm, D.NativeShard(lp, inner))
            x, st = solver.solve(b, tol=1e-10, max_iter=20000)
            out[f"x_{inner}"] = x.cpu().numpy()
            out[f"it_{inner}"] = st["iterations"]
            out[f"res_{inner}"] = np.array(st["residual_history"])
        np.savez(os.path.join(out_dir, f"{name}{rank}.npz"), **out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["slab", "torso"])
def test_native_shard_world2_on_one_gpu(name, tmp_path):
    import torch.multiprocessing as mp
    from oracle import bidomain_oracle as orc
    world = 2
    mp.spawn(_worker, args=(world, _port(), name, str(tmp_path)), nprocs=world, join=True)
    P = _problem(name)
    n, m = P["S1"].shape[0], P["Si"].shape[0]
    parts = [dict(np.load(tmp_path / f"{name}{r}.npz")) for r in range(world)]
    assert all(int(p["ghosts"]) > 0 for p in parts)
    if name == "torso":
        assert all(int(p["ghosts"]) > int(p["heart_ghosts"]) for p in parts)
    for inner in ("jacobi", "ic0"):
        xu, xv = np.zeros(n), np.zeros(m)
        for p in parts:
            own, mo = p["owned"], int(p["m_own"])
            xu[own] = p[f"x_{inner}"][: own.size]
            xv[own[:mo]] = p[f"x_{inner}"][own.size:]
        assert int(parts[0][f"it_{inner}"]) == int(parts[1][f"it_{inner}"])
        np.testing.assert_array_equal(parts[0][f"res_{inner}"], parts[1][f"res_{inner}"])
        pre = orc.BlockLU(P["S1"], P["Si"], P["Km"], inner)
        (ru, rv), st = orc.pcg(P["S1"], P["Si"], P["mh"], P["mass"], P["gamma"], pre, P["bu"],
                               P["bv"], tol=1e-10, max_iter=20000)
        it = int(parts[0][f"it_{inner}"])
        print(f"{name} {inner}: world-2 iterations {it}, 1-GPU oracle {st['iterations']}")
        assert rel_l2(xu, xv, ru, rv) <= 1e-8, inner
        if inner == "jacobi":
            assert abs(it - st["iterations"]) <= 2
        else:
            assert it <= 3 * st["iterations"]


def test_local_device_assembly_matches_global():
    """Per-rank assembly ON THE DEVICE (local mesh of the touching elements)
    reproduces the rows of the global host-assembled matrices (3 ranks, the
    heart-in-torso mesh with heart and torso ghosts), to rounding."""
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
