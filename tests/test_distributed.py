"""CPU (gloo, world size 2): the sharded path's host logic — RCB partition,
heart-first local numbering, one-layer halo plan, distributed Λ and the
distributed block-Jacobi PCG — against the single-process oracle on the
golden config-2 slab.  Local compute uses a scipy test double for the
backend (the product backend is paper_1711_08708_b200.distributed.NativeBackend)."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from conftest import REPO, csr, golden

from paper_1711_08708_b200 import distributed as D


class ScipyBackend:
    """Test double: local SpMV and block inner solves with scipy on CPU tensors."""

    def matrix(self, a):
        return sp.csr_matrix(a)

    def spmv(self, a, x):
        import torch
        return torch.as_tensor(a @ x.numpy())

    def inner(self, kind, a, coords=None):
        from oracle import bidomain_oracle as orc
        return orc.make_inner(kind, a)

    def inner_apply(self, p, y):
        import torch
        return torch.as_tensor(p.apply(y.numpy()))


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
        dsys = D.DistributedSystem(lp, comm, ScipyBackend())
        pre = D.DistributedBlockLU(dsys, inner, beta)
        bu, bv = g["sanity_b_u"], g["sanity_b_v"]
        b = torch.as_tensor(np.concatenate([bu[lp.owned], bv[lp.owned[: lp.m_own]]]))
        x, st = D.distributed_pcg(dsys, pre, b, tol=1e-10, max_iter=5000)
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


def test_weak_scaling_grids():
    """bench.py --mode sharded refines the cfg2 slab so every rank keeps a
    cfg2-sized part; 8 ranks is exactly BASELINE config 3 (256x256x128)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(REPO, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    base = (128, 128, 64)
    assert b.weak_cells(base, 1) == base
    assert b.weak_cells(base, 8) == (256, 256, 128)
    for w in (1, 2, 4, 8, 16):
        c = b.weak_cells(base, w)
        assert c[0] * c[1] * c[2] == w * base[0] * base[1] * base[2]
