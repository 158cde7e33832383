"""Warm per-launch device times of one GN iteration (CUDA events around every launch)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2604_23175_b200 as G
from paper_2604_23175_b200 import _native

name = sys.argv[1] if len(sys.argv) > 1 else "pegase9241_k16"
net, ms, part = bench.build_workload(name)
est = G.MultiAreaEstimator(net, ms, part)
for _ in range(3):
    est.estimate()
L = _native.lib()
L.gse_profile_iteration.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, _native.i32p, _native.i32p, _native.i32p, _native.f64p]
est._load_flat_start(); est.torch.cuda.synchronize()
va, vm = est._ptrs()
N = 512
kind = np.zeros(N, np.int32); ph = np.zeros(N, np.int32); ct = np.zeros(N, np.int32); us = np.zeros(N)
best = None
for rep in range(5):
    est._load_flat_start(); est.torch.cuda.synchronize()
    n = L.gse_profile_iteration(est.plan._h, va, vm, N, kind.ctypes.data_as(_native.i32p), ph.ctypes.data_as(_native.i32p), ct.ctypes.data_as(_native.i32p), us.ctypes.data_as(_native.f64p))
    best = us[:n].copy() if best is None else np.minimum(best, us[:n])
names = ["eval", "accumulate", "front", "backward", "update"]
print(f"{name}: {n} launches, sum {best.sum():.1f} us (min over 5 reps, each launch bracketed by events)")
for i in range(n):
    print(f"{i:3d} {names[kind[i]]:10s} phase {ph[i]} ctas {ct[i]:5d} {best[i]:8.2f} us")
for k in range(5):
    sel = kind[:n] == k
    if sel.any():
        print(f"{names[k]:10s} launches {sel.sum():3d} total {best[sel].sum():8.1f} us")

# ---- per-task phase clocks of the front kernel -------------------------------------------------
L.gse_debug_task_clocks.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
nt = L.gse_debug_task_clocks(est.plan._h, 1, None, 0)
est._load_flat_start(); est.torch.cuda.synchronize()
L.gse_profile_iteration(est.plan._h, va, vm, N, kind.ctypes.data_as(_native.i32p), ph.ctypes.data_as(_native.i32p), ct.ctypes.data_as(_native.i32p), us.ctypes.data_as(_native.f64p))
clk = np.zeros(nt * 32, dtype=np.int64)
L.gse_debug_task_clocks(est.plan._h, 0, clk.ctypes.data_as(C.c_void_p), nt * 32)
clk = clk.reshape(nt, 32)
d = np.diff(clk[:, :7], axis=1)   # zero, orig, children, panel, dmma, store
labels = ["zero", "orig", "extend-add", "panel", "dmma", "Lstore"]
# tasks are laid out launch by launch in the same order as the front launches above
pos = 0
print("per-launch front task phases (globaltimer ns, max over the launch's CTAs of total; phases of that slowest CTA)")
for i in range(n):
    if kind[i] != 2:
        continue
    blk = d[pos:pos + ct[i]]
    tot = blk.sum(axis=1)
    w = int(np.argmax(tot))
    print(f"launch {i:2d} ctas {ct[i]:4d} slowest {tot[w]:7d} ns: " + " ".join(f"{l}={v}" for l, v in zip(labels, blk[w])) + f" | median total {int(np.median(tot))}")
    row = clk[pos + w]
    if row[24] > 0:
        print("      last panel block: diag-dmma=%d load-d=%d factor=%d publish=%d sync1=%d trsm=%d sync2=%d" % tuple(int(row[k + 1] - row[k]) for k in range(24, 31)))
    if ct[i] <= 8 or i in (3, 17):
        row = clk[pos + w]
        ch = [(int(row[8 + 2 * c] - (row[7] if c == 0 else row[7 + 2 * c])), int(row[9 + 2 * c] - row[8 + 2 * c])) for c in range(12) if row[8 + 2 * c] > 0 and row[9 + 2 * c] >= row[8 + 2 * c]]
        print(f"      stage0={int(row[7] - row[2])} children (add, wait+sync): {ch}")
    pos += ct[i]
