"""Two (or more) PROCESSES on the one GPU, peer-linked through CUDA IPC handles: the multi-process form of the
in-kernel exchange (one process per GPU on a node; here the processes time-share one device, so this checks the
IPC mapping, the system-scope signalling and the host protocol -- not speed).  gloo carries the host plumbing.
    python tools/ipc_two_process.py [case] [world]"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def worker(rank, world, name, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2604_23175_b200 as G
    from paper_2604_23175_b200.distributed import DistributedEstimator
    from conftest import build_case
    net, ms, part, g = build_case(name)
    est = DistributedEstimator(net, ms, part, device=0, exchange="peer")
    est.engine.plan  # noqa: B018
    try:
        assert est.linked
        res = []
        for _ in range(2):
            st, rep = est.estimate()
            res.append((st, rep))
        if rank == 0:
            ref, rref = G.solve_multiarea(net, ms, part)
            for st, rep in res:
                assert rep.iterations == rref.iterations == int(g["iterations"]) and rep.converged
                assert np.array_equal(st.va, ref.va) and np.array_equal(st.vm, ref.vm), "state differs from the single-plan solve"
                assert rep.objective == rref.objective
            print(f"ipc ok: {name} world={world} iterations={rep.iterations} J={rep.objective!r} "
                  f"launches/solve={est.launches_per_solve} solve_s={est.last_gpu_s:.4f}", flush=True)
    finally:
        est.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "ieee118_k6"
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    mp.spawn(worker, args=(world, name, 20000 + os.getpid() % 20000, None), nprocs=world, join=True)
