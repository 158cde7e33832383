"""Debug helper: phase outputs vs the oracle for one case, printing max errors."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from conftest import build_case
import paper_2604_23175_b200 as G
from paper_2604_23175_b200._native import Plan, NativeError
from oracle.mase_oracle import Oracle

def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / (1.0 + np.abs(b)))) if a.size else 0.0

name = sys.argv[1]
net, ms, part, g = build_case(name)
bord, maps = G.build_variable_maps(net, part)
orc = Oracle(net, ms, part.area_of_bus)
for rep in range(2):
    plan = Plan(net, ms, part, bord, maps)
    st = np.stack([np.zeros(net.n_bus), np.ones(net.n_bus)]); st[0, net.slack] = net.buses[net.slack].va_true
    st = torch.from_numpy(st).cuda()
    va0, vm0 = st[0].cpu().numpy().copy(), st[1].cpu().numpy().copy()
    orc.local(va0, vm0)
    plan.phase_assemble(st[0].data_ptr(), st[1].data_ptr())
    try:
        plan.phase_condense()
    except NativeError as e:
        print("condense failed:", e)
    worst = []
    for a in range(part.k):
        s_b, b_hat = plan.area_schur(a); os_b, ob_hat = orc.schur(a)
        worst.append((rel(s_b, os_b), rel(b_hat, ob_hat)))
    print(rep, "schur errs per area:", ["%.1e/%.1e" % w for w in worst])
    if bord.n_gamma:
        orc.boundary()
        try:
            plan.phase_boundary()
        except NativeError as e:
            print("boundary failed:", e)
        s_g, b_g, dx = plan.boundary_system(); og, obg, odx = orc.boundary_system()
        print(rep, "S_gamma", rel(s_g, og), "b_gamma", rel(b_g, obg), "dx_gamma", rel(dx, odx))
    dinf = plan.phase_recover(st[0].data_ptr(), st[1].data_ptr())
    va1, vm1 = va0.copy(), vm0.copy()
    odinf = orc.recover(va1, vm1)
    print(rep, "delta_inf", dinf, odinf, "interior delta errs", ["%.1e" % rel(plan.area_delta(a), orc.interior_delta(a)) for a in range(part.k)])
    plan.close()
