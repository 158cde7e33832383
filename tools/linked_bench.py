"""Peer-linked rank plans side by side on the ONE GPU (debug / evidence; not a bench value): the same grid solved
by 1, 2, 4 ... rank plans that split the device's resident CTAs between them and exchange inside their persistent
kernels.  Shows what the in-kernel exchange protocol costs relative to the single plan (the hardware is the same
296 CTA slots in every row; on a node every rank has a whole GPU).
    python tools/linked_bench.py [workload] [worlds ...]"""
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2604_23175_b200 as G
from paper_2604_23175_b200.distributed import CudaEngine, area_work_estimate, assign_areas

name = sys.argv[1] if len(sys.argv) > 1 else "pegase9241_k16"
worlds = [int(v) for v in sys.argv[2:]] or [1, 2, 4]
net, ms, part = bench.build_workload(name)
bord, maps = G.build_variable_maps(net, part)
cfg = G.SolverConfig()
flat = G.StateVector.flat_start(net)
single = G.MultiAreaEstimator(net, ms, part, maps=(bord, maps), config=cfg)
for _ in range(3):
    ref, rref = single.estimate()
t = []
for _ in range(10):
    single.estimate(); t.append(single.last_gpu_s)
print(f"{name}: single plan (296 CTAs, fenced counters, fused state update)  {np.median(t) * 1e3:.3f} ms per solve, {rref.iterations} iterations")
single.close()
for world in worlds:
    if world < 2:
        continue
    area_rank = assign_areas(area_work_estimate(maps), world)
    engines = [CudaEngine(net, ms, part, bord, maps, cfg, r, world, area_rank, 0, max_ctas=296 // world) for r in range(world)]
    infos = [e.peer_info() for e in engines]
    for e in engines:
        e.peer_link(infos)
    times = []
    for rep_i in range(13):
        for e in engines:
            e.load_state(flat.va, flat.vm)
            e.solve_prepare()
        out = [None] * world
        def work(k):
            out[k] = engines[k].solve_linked(cfg)
        th = [threading.Thread(target=work, args=(k,)) for k in range(world)]
        t0 = time.perf_counter()
        [x.start() for x in th]; [x.join() for x in th]
        wall = time.perf_counter() - t0
        if rep_i >= 3:
            times.append((max(r.gpu_s for r in out), wall))
    state = engines[0].state.clone()
    for r in range(1, world):
        m = engines[r].owned_mask
        state[:, m] = engines[r].state[:, m]
    o = state.cpu().numpy()
    same = np.array_equal(o[0], ref.va) and np.array_equal(o[1], ref.vm)
    print(f"{name}: {world} linked rank plans x {296 // world} CTAs  {np.median([a for a, _ in times]) * 1e3:.3f} ms per solve (max over ranks, CUDA events), "
          f"host wall {np.median([b for _, b in times]) * 1e3:.3f} ms; iterations {out[0].iterations}; state bit-identical to the single plan: {same}")
    for e in engines:
        e.close()
