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
