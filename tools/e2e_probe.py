import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import bench, torch
import paper_2604_23175_b200 as G
net, ms, part = bench.build_workload("pegase9241_k16")
est = G.MultiAreaEstimator(net, ms, part)
zv, wv = est.pinned_inputs(); zv[:] = ms.z; wv[:] = ms.weight
for _ in range(5): est.update_from_pinned(); est.estimate()
N = 200
t_copy = t_est = t_all = 0.0
for _ in range(N):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); est.update_from_pinned(); torch.cuda.synchronize(); t1 = time.perf_counter()
    est.estimate(); t2 = time.perf_counter()
    t_copy += t1 - t0; t_est += t2 - t1
for _ in range(N):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); est.update_from_pinned(); est.estimate(); t_all += time.perf_counter() - t0
print(f"copy+sync {t_copy/N*1e6:.1f} us   estimate {t_est/N*1e6:.1f} us (gpu_s {est.last_gpu_s*1e6:.1f})   both, no sync between {t_all/N*1e6:.1f} us")
