"""PCG iterations per time step of the mesh-partitioned solve at N ranks
(block-Jacobi inners: the preconditioner changes with the partition), next to
the 1-GPU count, on ONE GPU: N processes share cuda:0, each runs its rank's
native kernels (NativeShard), and the halos / partial sums travel through host
memory over gloo (distributed.HostStagedComm).  Timings here are not
multi-GPU timings (the ranks time-share one GPU and the host stages every
exchange); the iteration counts are exactly those of an N-GPU run.

  python tools/sharded_iters.py --workload cfg2 --ranks 1,2,4,8 --steps 3
"""
import argparse
import json
import os
import socket
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, workload, steps, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_08708_b200 import configs
        from paper_1711_08708_b200 import distributed as D
        wl = configs.BUILDERS[workload]()
        part = D.rcb_partition(wl.mesh.vertices, world)
        dev = torch.device("cuda", 0)
        comm = D.HostStagedComm(dist, dev)
        t0 = time.perf_counter()
        sim = D.DistributedSimulation(wl, part, rank, world, dist, dev, comm=comm)
        setup = time.perf_counter() - t0
        st = sim.resting()
        its = []
        for _ in range(steps):
            st, s = sim.step(st)
            its.append(s["iterations"])
        if rank == 0:
            with open(out, "w") as fh:
                json.dump({"workload": workload, "ranks": world, "iters": its,
                           "n_own_rank0": sim.lp.n_own, "ghosts_rank0": int(sim.lp.ghosts.size),
                           "setup_s_rank0": round(setup, 1)}, fh)
    finally:
        dist.destroy_process_group()


def main():
    import torch.multiprocessing as mp
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--ranks", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    res = []
    for w in [int(x) for x in a.ranks.split(",")]:
        out = f"/tmp/sharded_iters_{w}.json"
        mp.spawn(worker, args=(w, _port(), a.workload, a.steps, out), nprocs=w, join=True)
        rec = json.load(open(out))
        print(json.dumps(rec), flush=True)
        res.append(rec)


if __name__ == "__main__":
    main()
