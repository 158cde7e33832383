"""Soak test of the persistent kernel's hand-offs: N flat-start solves per workload on one plan, every result compared
bit for bit with the first one (a stale read through a hand-off would show up as a different iterate sooner or later).
    python tools/soak.py [n_small] [n_large]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2604_23175_b200 as G

n_small = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
n_large = int(sys.argv[2]) if len(sys.argv) > 2 else 300
for name, n in (("pegase2869_k8", n_small), ("pegase9241_k16", n_small), ("activsg10k_k32", n_small), ("tiled101k_k128", n_large)):
    net, ms, part = bench.build_workload(name)
    est = G.MultiAreaEstimator(net, ms, part)
    ref, rep0 = est.estimate()
    bad, t0 = 0, time.perf_counter()
    for k in range(n):
        st, rep = est.estimate()
        if rep.iterations != rep0.iterations or rep.objective != rep0.objective or not (np.array_equal(st.va, ref.va) and np.array_equal(st.vm, ref.vm)):
            bad += 1
    print(f"{name}: {n} solves, {bad} differ from the first (iterations {rep0.iterations}, J {rep0.objective!r}), {time.perf_counter() - t0:.1f} s", flush=True)
    est.close()

# varied data: fresh noise every solve, the persistent kernel against the level-launch path on the same plan family
rng = np.random.default_rng(1)
for name, n in (("pegase2869_k8", 300), ("pegase9241_k16", 300)):
    net, ms, part = bench.build_workload(name)
    a = G.MultiAreaEstimator(net, ms, part)
    b = G.MultiAreaEstimator(net, ms, part, config=G.SolverConfig(profile_phases=True))
    bad = 0
    for k in range(n):
        z = ms.z + rng.normal(0.0, 1.0, ms.m) / np.sqrt(ms.weight)
        ms2 = ms.with_values(z) if hasattr(ms, "with_values") else None
        if ms2 is None:
            import dataclasses
            ms2 = dataclasses.replace(ms, z=z)
        a.update_measurements(ms2); b.update_measurements(ms2)
        sa, ra = a.estimate(); sb, rb = b.estimate()
        if ra.iterations != rb.iterations or not (np.array_equal(sa.va, sb.va) and np.array_equal(sa.vm, sb.vm)):
            bad += 1
    print(f"{name}: {n} noisy scans, persistent vs level-launch path: {bad} differ", flush=True)
    a.close(); b.close()
