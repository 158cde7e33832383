"""Per-item timeline of the persistent dataflow kernel (debug; numbers here are not bench values).

Arms gse_debug_trace, runs one warm solve and prints, per iteration: when each item class
started / ended, how long items waited on dependencies vs. executed, and the critical chain.
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2604_23175_b200 as G
from paper_2604_23175_b200 import _native

name = sys.argv[1] if len(sys.argv) > 1 else "pegase9241_k16"
net, ms, part = bench.build_workload(name)
est = G.MultiAreaEstimator(net, ms, part)
for _ in range(3):
    est.estimate()
L = _native.lib()
L.gse_debug_trace.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
L.gse_solve_layout.argtypes = [C.c_void_p, C.c_void_p]
lay = np.zeros(8, dtype=np.int32)
L.gse_solve_layout(est.plan._h, lay.ctypes.data_as(C.c_void_p))
n_eval, n_acc, n_task, n_bwd, n_upd, grid, smem, persistent = (int(v) for v in lay)
per_it = L.gse_debug_trace(est.plan._h, 1, None, 0)
state, rep = est.estimate()
tr = np.zeros(per_it * 16 * 8, dtype=np.uint64)
L.gse_debug_trace(est.plan._h, 0, tr.ctypes.data_as(C.c_void_p), tr.size)
tr = tr.reshape(-1, 8).astype(np.int64)
print(f"{name}: persistent={persistent} grid={grid} smem={smem} items/it={per_it} "
      f"(eval {n_eval}, acc {n_acc}, front {n_task}, bwd {n_bwd}, upd {n_upd}); iterations={rep.iterations} "
      f"gpu_s={est.last_gpu_s*1e3:.3f} ms")
t0 = tr[0, 0]
bounds = np.cumsum([0, n_eval, n_acc, n_task, n_bwd, n_upd])
names = ["eval", "acc", "front", "bwd", "upd"]
for it in range(rep.iterations):
    blk = tr[it * per_it:(it + 1) * per_it]
    print(f"-- iteration {it}: starts {(blk[:, 0].min() - t0) / 1e3:8.1f} us, ends {(blk[:, 3].max() - t0) / 1e3:8.1f} us")
    for k, nm in enumerate(names):
        b = blk[bounds[k]:bounds[k + 1]]
        if not len(b):
            continue
        pull, ready, end = b[:, 0], np.maximum(np.maximum(b[:, 1], b[:, 2]), b[:, 0]), b[:, 3]
        print(f"   {nm:5s} n={len(b):5d} first pull {(pull.min() - t0) / 1e3:8.1f}  last end {(end.max() - t0) / 1e3:8.1f}  "
              f"wait mean {np.mean(ready - pull) / 1e3:6.2f} max {np.max(ready - pull) / 1e3:6.2f}  "
              f"exec mean {np.mean(end - ready) / 1e3:6.2f} max {np.max(end - ready) / 1e3:6.2f} us")
    if it == 1:
        b = blk[bounds[1]:bounds[2]]
        rdy = np.maximum(b[:, 2], b[:, 0])
        print(f"   acc detail (mean us): gather {np.mean(b[:,5]-rdy)/1e3:.2f}  tma wait {np.mean(b[:,6]-b[:,5])/1e3:.2f}  "
              f"contributions {np.mean(b[:,7]-b[:,6])/1e3:.2f}  signal {np.mean(b[:,3]-b[:,7])/1e3:.2f}")
    if it == 1 or rep.iterations == 1:
        # front tasks: end time by position in the list (level order) -- the wavefront
        b = blk[bounds[2]:bounds[3]]
        step = max(1, len(b) // 40)
        print("   front wavefront (task idx: pull, ready, end in us rel. to iteration start):")
        s0 = blk[:, 0].min()
        for i in range(0, len(b), step):
            print(f"     {i:5d}: {(b[i,0]-s0)/1e3:7.1f} {(max(b[i,1],b[i,2],b[i,0])-s0)/1e3:7.1f} {(b[i,3]-s0)/1e3:7.1f}  sm {b[i,4] & 0xffff}")
        b = blk[bounds[3]:bounds[4]]
        step = max(1, len(b) // 25)
        print("   backward wavefront:")
        for i in range(0, len(b), step):
            print(f"     {i:5d}: {(b[i,0]-s0)/1e3:7.1f} {(max(b[i,2],b[i,0])-s0)/1e3:7.1f} {(b[i,3]-s0)/1e3:7.1f}")
