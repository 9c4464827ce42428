"""CPU (gloo, world size 2): the sharded path's host logic — RCB partition,
heart-first local numbering with ghosts grouped by owner, the halo plan, the
four all-reduces per iteration and the block-Jacobi PCG loop of
ShardSolver — against the single-process oracle on the golden config-2
slab.  The rank-local kernels run in TorchShard, the CPU restatement of the
native bd_shard_* kernels (the product path is NativeShard; its GPU tests are
tests/test_gpu_distributed.py)."""
import os
import socket

import numpy as np
import pytest

from conftest import REPO, csr, golden

from paper_1711_08708_b200 import distributed as D


def test_rcb_partition_balanced_boxes():
    g = golden("cfg2s")
    pts = g["points"]
    for parts in (2, 3, 4, 8):
        part = D.rcb_partition(pts, parts)
        counts = np.bincount(part, minlength=parts)
        assert counts.sum() == pts.shape[0] and counts.max() - counts.min() <= 1


def test_local_problems_cover_and_halo_consistent():
    g = golden("cfg2s")
    S1, Si, Km = csr(g, "S1"), csr(g, "Si"), csr(g, "Km")
    from oracle import bidomain_oracle as orc
    beta, grounded = orc.regularize(S1)
    part = D.rcb_partition(g["points"], 3)
    lps = [D.build_local(S1, Si, g["mass"], g["mh"], g["gamma"], grounded, Km, part, r, 3)
           for r in range(3)]
    owned = np.concatenate([lp.owned for lp in lps])
    assert np.array_equal(np.sort(owned), np.arange(S1.shape[0]))
    for lp in lps:
        # heart-first locally; ghosts owned by someone else; halo lists match pairwise
        assert (lp.owned[: lp.m_own] < lp.m_global).all() and (lp.owned[lp.m_own:] >= lp.m_global).all()
        assert (part[lp.ghosts] != lp.rank).all()
        for q, idx in lp.send.items():
            peer = lps[q]
            assert np.array_equal(lp.owned[idx], peer.ghosts[peer.recv[lp.rank]])
    # local Λ rows reproduce the global operator
    rng = np.random.default_rng(0)
    u, v = rng.standard_normal(S1.shape[0]), rng.standard_normal(Si.shape[0])
    top, bot = orc.lambda_apply(S1, Si, g["mh"], float(g["gamma"]), u, v)
    for lp in lps:
        ext = np.concatenate([lp.owned, lp.ghosts])
        hext = np.concatenate([lp.owned[: lp.m_own], lp.ghosts[: lp.m_ghost]])
        t = lp.S1 @ u[ext]
        t[: lp.m_own] += lp.Si @ v[hext]
        np.testing.assert_allclose(t, top[lp.owned], rtol=1e-13, atol=1e-13 * np.abs(top).max())


def _worker(rank, world, port, inner, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import bidomain_oracle as orc
        g = golden("cfg2s")
        S1, Si, Km = csr(g, "S1"), csr(g, "Si"), csr(g, "Km")
        beta, grounded = orc.regularize(S1)
        part = D.rcb_partition(g["points"], world)
        lp = D.build_local(S1, Si, g["mass"], g["mh"], g["gamma"], grounded, Km, part, rank, world)
        comm = D.Comm(dist, torch.device("cpu"))
        solver = D.ShardSolver(lp, comm, D.TorchShard(lp, D._cpu_inner(inner)))
        bu, bv = g["sanity_b_u"], g["sanity_b_v"]
        b = torch.as_tensor(np.concatenate([bu[lp.owned], bv[lp.owned[: lp.m_own]]]))
        x, st = solver.solve(b, tol=1e-10, max_iter=5000)
        # the four all-reduces of an iteration leave the residual history of
        # the recursive residual on every rank identical
        assert len(st["residual_history"]) == st["iterations"] + 1
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), x=x.numpy(), owned=lp.owned,
                 m_own=lp.m_own, iters=st["iterations"])
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("inner", ["jacobi", "ic0"])
def test_distributed_pcg_gloo_world2(inner, tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), inner, str(tmp_path)), nprocs=world, join=True)
    g = golden("cfg2s")
    n, m = g["mass"].size, g["mh"].size
    xu, xv = np.zeros(n), np.zeros(m)
    iters = []
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        own, mo = d["owned"], int(d["m_own"])
        xu[own] = d["x"][: own.size]
        xv[own[:mo]] = d["x"][own.size:]
        iters.append(int(d["iters"]))
    assert iters[0] == iters[1]
    ref_u, ref_v = g[f"sanity_{inner}_u"], g[f"sanity_{inner}_v"]
    rel = np.sqrt(np.sum((xu - ref_u) ** 2) + np.sum((xv - ref_v) ** 2)) / np.sqrt(
        np.sum(ref_u ** 2) + np.sum(ref_v ** 2))
    assert rel <= 1e-8
    if inner == "jacobi":  # block-Jacobi of a diagonal is the diagonal: shards exactly
        assert abs(iters[0] - int(g["sanity_jacobi_iters"])) <= 2
    else:  # block-Jacobi IC(0) changes the preconditioner: report, bounded
        assert iters[0] <= 3 * int(g["sanity_ic0_iters"])


def _torso_problem():
    """Heart-in-torso 2D mesh (heart-first numbering, torso AND heart ghosts)."""
    from oracle import bidomain_oracle as orc
    from paper_1711_08708_b200 import configs
    from paper_1711_08708_b200.precond import build_monodomain_matrix
    from paper_1711_08708_b200.system import BidomainSystem
    wl = configs.cfg1(40)
    sysm = BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False)
    km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers)
    beta, grounded = orc.regularize(sysm.stiff_total)
    bu, bv = configs.sanity_rhs(sysm.n, sysm.n_heart, seed=3)
    return wl, sysm, km, grounded, bu, bv


def _torso_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl, sysm, km, grounded, bu, bv = _torso_problem()
        part = D.rcb_partition(wl.mesh.vertices, world)
        lp = D.build_local(sysm.stiff_total, sysm.stiff_intra, sysm.mass_diag,
                           sysm.heart_mass_diag, sysm.gamma, grounded, km, part, rank, world)
        assert lp.m_ghost < lp.ghosts.size  # torso ghosts present
        solver = D.ShardSolver(lp, D.Comm(dist, torch.device("cpu")),
                               D.TorchShard(lp, D._cpu_inner("jacobi")))
        b = torch.as_tensor(np.concatenate([bu[lp.owned], bv[lp.owned[: lp.m_own]]]))
        x, st = solver.solve(b, tol=1e-10, max_iter=20000)
        np.savez(os.path.join(out_dir, f"t{rank}.npz"), x=x.numpy(), owned=lp.owned,
                 m_own=lp.m_own, iters=st["iterations"])
    finally:
        dist.destroy_process_group()


def test_distributed_pcg_gloo_world2_heart_in_torso(tmp_path):
    """World size 2 on a heart-in-torso mesh: the S_i products read only the
    heart ghosts, Λ the heart and torso ghosts; jacobi shards exactly, so the
    sharded solve equals the oracle's (iterations +-2, rel-L2 1e-8)."""
    import torch.multiprocessing as mp
    from oracle import bidomain_oracle as orc
    world = 2
    mp.spawn(_torso_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    wl, sysm, km, grounded, bu, bv = _torso_problem()
    pre = orc.BlockLU(sysm.stiff_total, sysm.stiff_intra, km, "jacobi")
    (ru, rv), st = orc.pcg(sysm.stiff_total, sysm.stiff_intra, sysm.heart_mass_diag,
                           sysm.mass_diag, sysm.gamma, pre, bu, bv, tol=1e-10, max_iter=20000)
    xu, xv = np.zeros(sysm.n), np.zeros(sysm.n_heart)
    iters = []
    for r in range(world):
        d = np.load(tmp_path / f"t{r}.npz")
        own, mo = d["owned"], int(d["m_own"])
        xu[own] = d["x"][: own.size]
        xv[own[:mo]] = d["x"][own.size:]
        iters.append(int(d["iters"]))
    assert iters[0] == iters[1] and abs(iters[0] - st["iterations"]) <= 2
    rel = np.sqrt(np.sum((xu - ru) ** 2) + np.sum((xv - rv) ** 2)) / np.sqrt(
        np.sum(ru ** 2) + np.sum(rv ** 2))
    assert rel <= 1e-8


def test_local_assembly_matches_global():
    """Per-rank assembly from the touching elements reproduces the rows of the
    global matrices and the global halo plan."""
    from paper_1711_08708_b200 import configs
    from paper_1711_08708_b200.precond import build_monodomain_matrix, regularize_stiffness
    from paper_1711_08708_b200.system import BidomainSystem
    wl = configs.cfg1(32)  # heart-in-torso: heart-first numbering, torso and heart ghosts
    sysm = BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers, with_extra=False)
    km = build_monodomain_matrix(wl.mesh, wl.params, sysm.gamma, wl.fibers)
    reg = regularize_stiffness(sysm.stiff_total)
    part = D.rcb_partition(wl.mesh.vertices, 3)
    for r in range(3):
        ref = D.build_local(sysm.stiff_total, sysm.stiff_intra, sysm.mass_diag,
                            sysm.heart_mass_diag, sysm.gamma, reg.grounded(), km, part, r, 3)
        tot = float(sysm.stiff_total.diagonal().sum())  # stands in for the all_reduce
        loc = D.build_local_from_mesh(wl.mesh, wl.params, wl.fibers, wl.dt, part, r, 3,
                                      comm_allreduce=lambda v: [tot])
        assert np.array_equal(ref.owned, loc.owned) and np.array_equal(ref.ghosts, loc.ghosts)
        assert loc.beta == pytest.approx(reg.beta, rel=1e-14)
        for a, b in ((ref.S1, loc.S1), (ref.Si, loc.Si), (ref.bulk_block, loc.bulk_block),
                     (ref.schur_block, loc.schur_block)):
            assert a.shape == b.shape
            np.testing.assert_allclose(a.toarray(), b.toarray(), rtol=0,
                                       atol=1e-13 * max(1.0, np.abs(a.data).max()))
        np.testing.assert_allclose(loc.mass, ref.mass, rtol=1e-14)
        np.testing.assert_allclose(loc.heart_mass, ref.heart_mass, rtol=1e-14)
        for q in ref.send:
            assert np.array_equal(ref.send[q], loc.send[q])
        for q in ref.recv:
            assert np.array_equal(ref.recv[q], loc.recv[q])
        for q in ref.send_heart:
            assert np.array_equal(ref.send_heart[q], loc.send_heart[q])
