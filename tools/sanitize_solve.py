"""One persistent-kernel solve and one level-path solve of a golden case (run under compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from conftest import build_case
import paper_2604_23175_b200 as G
name = sys.argv[1] if len(sys.argv) > 1 else "ieee118_k6"
net, ms, part, g = build_case(name)
a, ra = G.solve_multiarea(net, ms, part)
b, rb = G.solve_multiarea(net, ms, part, config=G.SolverConfig(profile_phases=True))
assert ra.iterations == int(g["iterations"]) and np.array_equal(a.va, b.va) and np.array_equal(a.vm, b.vm)
print(name, "ok", ra.iterations, ra.objective)
