"""Cold path: where the plan build spends its time (GSE_DEBUG_TIME=1 prints the C++ sections)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GSE_DEBUG_TIME", "1")
import torch
import bench
import paper_2604_23175_b200 as G
name = sys.argv[1] if len(sys.argv) > 1 else "pegase9241_k16"
net, ms, part = bench.build_workload(name)
torch.zeros(1, device="cuda"); torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    maps = G.build_variable_maps(net, part)
    t1 = time.perf_counter()
    est = G.MultiAreaEstimator(net, ms, part, maps=maps)
    t2 = time.perf_counter()
    st, rp = est.estimate()
    t3 = time.perf_counter()
    est.close()
    print(f"{name} rep {rep}: maps {t1 - t0:.3f} s, estimator {t2 - t1:.3f} s, first solve {t3 - t2:.4f} s "
          f"(iterations {rp.iterations})", flush=True)
