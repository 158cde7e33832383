"""Two warm solves of a named workload (for ncu captures; numbers printed here are not bench values)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2604_23175_b200 as G

name = sys.argv[1] if len(sys.argv) > 1 else "pegase9241_k16"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
net, ms, part = bench.build_workload(name)
est = G.MultiAreaEstimator(net, ms, part)
for _ in range(n):
    state, rep = est.estimate()
print(name, rep.iterations, rep.objective, est.plan.stats())
