"""cProfile of the host side of one end-to-end step (update_measurements + estimate)."""
import cProfile, pstats, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2604_23175_b200 as G
net, ms, part = bench.build_workload(sys.argv[1] if len(sys.argv) > 1 else "pegase9241_k16")
est = G.MultiAreaEstimator(net, ms, part)
for _ in range(5):
    est.update_measurements(ms); est.estimate()
pr = cProfile.Profile(); pr.enable()
for _ in range(200):
    est.update_measurements(ms); est.estimate()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
