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
tr = np.zeros(per_it * 16 * 32, dtype=np.uint64)
L.gse_debug_trace(est.plan._h, 0, tr.ctypes.data_as(C.c_void_p), tr.size)
tr = tr.reshape(-1, 32).astype(np.int64)
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
        b = blk[bounds[0]:bounds[1]]
        ex = (b[:, 3] - b[:, 0]) / 1e3
        q = len(ex) // 8 or 1
        print("   eval exec by item index (mean us per eighth: flow units first, then injection, then VM): "
              + " ".join(f"{ex[i:i + q].mean():.1f}" for i in range(0, len(ex), q)))
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
        # per front: when its children were ready, when panels / updates finished
        fr = {}
        for i in range(len(b)):
            kind = int(b[i, 6] & 0xff); f = int((b[i, 6] >> 8) & 0xffffff); pv = int(b[i, 7] & 0xffff); u1 = int((b[i, 7] >> 16) & 0xffff)
            nchild = int((b[i, 7] >> 32) & 0xffff)
            d = fr.setdefault(f, dict(p=pv, u1=u1, kinds=set(), n=0, ready=[], pend=[], uend=[], nchild=0, pull=[], pready=[]))
            d["kinds"].add(kind); d["n"] += 1; d["nchild"] = max(d["nchild"], nchild)
            d["pull"].append(b[i, 0] - s0)
            d["ready"].append(max(b[i, 1], b[i, 2], b[i, 0]) - s0)
            (d["pend"] if kind == 1 else d["uend"]).append(b[i, 3] - s0)
            if kind == 2: d["pready"].append(b[i, 5] - s0)
        print("   fronts by completion (front: p u1 tasks kinds nchild | children ready(max)  panels end(max)  panel-wait end(max)  all end(max)  last pull):")
        items = sorted(fr.items(), key=lambda kv: max(kv[1]["uend"] or kv[1]["pend"]))
        for f, d in items[-45:]:
            print(f"     {f:5d}: {d['p']:3d} {d['u1']:4d} {d['n']:4d} {sorted(d['kinds'])} {d['nchild']:3d} | {max(d['ready'])/1e3:7.1f} "
                  f"{(max(d['pend']) if d['pend'] else 0)/1e3:7.1f} {(max(d['pready']) if d['pready'] else 0)/1e3:7.1f} {max(d['uend'] or d['pend'])/1e3:7.1f} {max(d['pull'])/1e3:7.1f}")
        # phase breakdown (us) of the tasks on the critical chain: stamps 8.. = start, zero, orig, gather end, panel end,
        # update end, store end, inv-map built
        print("   task phases (front kind ci cj | zero orig invmap [child wait] gather panel [panel wait+load] update store signal):")
        for f, d in items[-14:]:
            for i in range(len(b)):
                if int((b[i, 6] >> 8) & 0xffffff) != f: continue
                kind = int(b[i, 6] & 0xff); ci = int((b[i, 6] >> 32) & 0xffff); cj = int((b[i, 6] >> 48) & 0xffff)
                if ci > 1 or cj > 0 and kind != 2: continue
                st = b[i, 8:16]
                cw = max(b[i, 2], st[7]) if b[i, 2] else st[7]
                pw = b[i, 5] if kind == 2 else st[4]
                print(f"     {f:5d} k{kind} {ci},{cj} | {(st[1]-st[0])/1e3:5.1f} {(st[2]-st[1])/1e3:5.1f} {(st[7]-st[2])/1e3:5.1f} [{(cw-st[7])/1e3:5.1f}] "
                      f"{(st[3]-cw)/1e3:5.1f} {(st[4]-st[3])/1e3:5.1f} [{(pw-st[4])/1e3:5.1f}] {(st[5]-pw)/1e3:5.1f} {(st[6]-st[5])/1e3:5.1f} {(b[i,3]-st[6])/1e3:5.1f}"
                      + ("   panel cyc: diagupd %d - %d factor %d publish %d barrier %d tile solve %d tail %d" % tuple(b[i, 16:23]) if kind != 2 else ""))
        b = blk[bounds[3]:bounds[4]]
        step = max(1, len(b) // 25)
        print("   backward wavefront:")
        for i in range(0, len(b), step):
            print(f"     {i:5d}: {(b[i,0]-s0)/1e3:7.1f} {(max(b[i,2],b[i,0])-s0)/1e3:7.1f} {(b[i,3]-s0)/1e3:7.1f}")
        if os.environ.get("GSE_TRACE_HIST"):
            # where the CTA time of the front tasks goes: by (pivots, update rows) class -- tasks, CTA-time from ready to
            # end, and its phases (gather, panel, update, signal)
            bf = blk[bounds[2]:bounds[3]]
            cls = {}
            for i in range(len(bf)):
                pv = int(bf[i, 7] & 0xffff); u1 = int((bf[i, 7] >> 16) & 0xffff); nchild = int((bf[i, 7] >> 32) & 0xffff)
                st = bf[i, 8:16]
                rdy = max(bf[i, 1], bf[i, 2], bf[i, 0])
                cw = max(bf[i, 2], st[7]) if bf[i, 2] else st[7]
                key = (min(pv // 16 * 16, 64), 0 if u1 <= 32 else 1 if u1 <= 96 else 2 if u1 <= 256 else 3)
                d = cls.setdefault(key, np.zeros(8))
                d += [1, (bf[i, 3] - rdy) / 1e3, (bf[i, 3] - bf[i, 0]) / 1e3, (st[3] - cw) / 1e3, (st[4] - st[3]) / 1e3,
                      (st[5] - st[4]) / 1e3, (bf[i, 3] - st[5]) / 1e3, (st[7] - st[0]) / 1e3]
            print("   front tasks by class (p>=, u class 0:<=32 1:<=96 2:<=256 3:more | tasks  exec-us total  held-us total | mean gather panel update signal prep):")
            for key in sorted(cls):
                d = cls[key]; n = d[0]
                print(f"     p>={key[0]:2d} u{key[1]} | {int(n):6d} {d[1]:10.0f} {d[2]:10.0f} | {d[3]/n:5.1f} {d[4]/n:5.1f} {d[5]/n:5.1f} {d[6]/n:5.1f} {d[7]/n:5.1f}")
            bb = blk[bounds[3]:bounds[4]]
            print(f"   backward tasks: n={len(bb)} exec total {np.sum(bb[:,3]-np.maximum(bb[:,2],bb[:,0]))/1e3:.0f} us  held total {np.sum(bb[:,3]-bb[:,0])/1e3:.0f} us")
        if os.environ.get("GSE_TRACE_FRONT"):
            # every task of one front: tile, SM, when it was ready / ended, its phases; and which other front task shared its SM
            want = int(os.environ["GSE_TRACE_FRONT"])
            bf = blk[bounds[2]:bounds[3]]
            s0 = blk[:, 0].min()
            rows = []
            for i in range(len(bf)):
                f = int((bf[i, 6] >> 8) & 0xffffff)
                rdy = max(bf[i, 1], bf[i, 2], bf[i, 0])
                rows.append((f, int((bf[i, 6] >> 32) & 0xffff), int((bf[i, 6] >> 48) & 0xffff), int(bf[i, 4] & 0xffff), rdy - s0, bf[i, 3] - s0, bf[i, 8:16], bf[i, 24:27]))
            print(f"   tasks of front {want} (ci cj sm | ready end exec | gather panel update | tasks of other fronts busy on the same SM meanwhile):")
            for f, ci, cj, sm, rdy, end, st, sub in rows:
                if f != want: continue
                mates = [(g, a, b) for g, a, b, sm2, r2, e2, _, _ in rows if sm2 == sm and not (g == f and a == ci and b == cj) and r2 < end and e2 > rdy]
                cw = st[7]
                print(f"     {ci:2d},{cj:2d} sm {sm:3d} | {rdy/1e3:7.1f} {end/1e3:7.1f} {(end-rdy)/1e3:5.1f} | {(st[3]-max(cw, rdy+s0))/1e3:5.1f} {(st[4]-st[3])/1e3:5.1f} {(st[5]-st[4])/1e3:5.1f} | {mates[:3]}"
                      + (f"  last child: ready->start {(sub[0]-(rdy+s0))/1e3:4.1f} panel {(sub[1]-sub[0])/1e3:4.1f} tile {(sub[2]-sub[1])/1e3:4.1f} ->gather end {(st[3]-sub[2])/1e3:4.1f}" if sub[0] else ""))
