"""Current-magnitude measurement template (MeasurementType.IF / IT): a north_star template the reference does not
have (its enum ends at QT, reference measurement.py:27-34) -- PARITY UNPINNED.  What can be checked is: the analytic
gradient against finite differences, the three independent restatements against each other (host scalar formulas in
complex arithmetic, the C oracle in rectangular arithmetic, the device / host-interpreter template in the
trigonometric |I|^2 form), and the estimator property noiseless -> truth.  The default measurement sets stay the
reference's seven types."""

import numpy as np
import pytest

from conftest import build_case


@pytest.fixture(scope="module")
def G():
    import paper_2604_23175_b200 as G
    return G


def _with_currents(G, net, seed=0, noiseless=False, min_current=0.1):
    """The reference's seven row types plus ammeter rows (IF / IT) on the loaded branches: |I| has a kink at zero,
    so a magnitude reading of a (nearly) idle branch cannot be fitted smoothly -- Gauss-Newton then hovers around
    the kink; such rows are left out, as a real measurement plan would."""
    types = G.measurement.REFERENCE_TYPES + (G.MeasurementType.IF, G.MeasurementType.IT)
    ms = G.generate_measurements(net, G.MeasurementConfig(types=types, seed=seed))
    exact = G.measurement.eval_h_all(ms, G.StateVector.truth(net))
    keep = (ms.mtype < int(G.MeasurementType.IF)) | (exact >= min_current)
    z = exact if noiseless else ms.z
    sigma = np.full(ms.m, 0.01) if noiseless else ms.sigma
    return G.make_measurement_set(net, ms.mtype[keep], ms.target[keep], z[keep], sigma[keep])


def test_defaults_stay_the_reference_types(G):
    net, ms, part, g = build_case("ieee14_k2")
    assert ms.m == 3 * net.n_bus + 4 * net.n_branch and int(ms.mtype.max()) == int(G.MeasurementType.QT)
    assert G.measurement.type_from_label("if") == G.MeasurementType.IF and G.MeasurementType.IT.is_branch
    with_i = _with_currents(G, net, min_current=0.0)
    assert with_i.m == ms.m + 2 * net.n_branch
    # the shared rows are generated from the same stream positions only for the first seven types' prefix
    assert np.array_equal(with_i.mtype[:ms.m], ms.mtype) and np.array_equal(with_i.target[:ms.m], ms.target)


def test_gradient_matches_finite_differences(G):
    net, ms, part, g = build_case("ieee118_k3")
    rng = np.random.default_rng(5)
    va = rng.uniform(-0.2, 0.2, net.n_bus)
    vm = rng.uniform(0.9, 1.1, net.n_bus)
    st = G.StateVector(va=va, vm=vm)
    worst = 0.0
    for t in (G.MeasurementType.IF, G.MeasurementType.IT):
        for e in range(0, net.n_branch, 7):
            h0 = G.eval_h(net, t, e, st)
            assert h0 > 0.0
            for (bus, quant), val in G.eval_row_gradient(net, t, e, st):
                step = 1e-6
                up, dn = st.copy(), st.copy()
                arr_u = up.va if quant == "va" else up.vm
                arr_d = dn.va if quant == "va" else dn.vm
                arr_u[bus] += step
                arr_d[bus] -= step
                fd = (G.eval_h(net, t, e, up) - G.eval_h(net, t, e, dn)) / (2 * step)
                worst = max(worst, abs(fd - val) / (1.0 + abs(val)))
    assert worst < 1e-7, worst


def test_vanishing_current_has_no_gradient(G):
    # flat start on a branch without charging or tap: i = 0, the row contributes nothing to that iteration
    net = G.BusBranchNetwork.from_components(
        [G.Bus(id=1, is_slack=True), G.Bus(id=2)], [G.Branch(from_bus=0, to_bus=1, r=0.01, x=0.1, b_charging=0.0)])
    st = G.StateVector.flat_start(net)
    assert G.eval_h(net, G.MeasurementType.IF, 0, st) == 0.0
    assert all(v == 0.0 for _, v in G.eval_row_gradient(net, G.MeasurementType.IF, 0, st))


@pytest.mark.parametrize("name", ["ieee14_k2", "ieee118_k6"])
def test_oracle_and_host_interpreter_agree_and_recover_truth(G, name):
    """C oracle (rectangular arithmetic) vs the device program on the host interpreter (the CUDA template's
    formulas): same iteration count, states within 1e-9; noiseless rows -> the true state."""
    from hostsim import HostSim
    from oracle.mase_oracle import Oracle
    net, _, part, g = build_case(name)
    bord, maps = G.build_variable_maps(net, part)
    ms = _with_currents(G, net, seed=3)
    ref = Oracle(net, ms, part.area_of_bus).solve()
    assert ref["converged"]
    sim = HostSim(net, ms, part, bord, maps)
    va, vm, it, conv, deltas = sim.solve(tol=1e-6)
    assert conv and it == ref["iterations"]
    assert max(np.max(np.abs(va - ref["va"])), np.max(np.abs(vm - ref["vm"]))) < 1e-9
    # the current rows carry information: the estimate differs from the one without them
    base = Oracle(net, build_case(name)[1], part.area_of_bus).solve()
    assert np.max(np.abs(base["vm"] - ref["vm"])) > 1e-7
    exact = _with_currents(G, net, noiseless=True)
    tr = Oracle(net, exact, part.area_of_bus).solve()
    va_true = np.array([b.va_true for b in net.buses]); vm_true = np.array([b.vm_true for b in net.buses])
    assert tr["converged"] and np.max(np.abs(tr["va"] - va_true)) < 1e-8 and np.max(np.abs(tr["vm"] - vm_true)) < 1e-8
    assert tr["objective"] < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["ieee14_k2", "ieee118_k6", "pegase2869_k8"])
def test_device_solve_with_current_rows_matches_the_oracle(G, name):
    from oracle.mase_oracle import Oracle
    net, _, part, g = build_case(name)
    ms = _with_currents(G, net, seed=3)
    ref = Oracle(net, ms, part.area_of_bus).solve()
    est, rep = G.solve_multiarea(net, ms, part)
    assert rep.converged and rep.iterations == ref["iterations"]
    assert np.max(np.abs(est.va - ref["va"])) < 1e-8 and np.max(np.abs(est.vm - ref["vm"]) / ref["vm"]) < 1e-8
    assert abs(rep.objective - ref["objective"]) <= 1e-10 * ref["objective"]
    lvl, rl = G.solve_multiarea(net, ms, part, config=G.SolverConfig(profile_phases=True))
    assert np.array_equal(lvl.va, est.va) and np.array_equal(lvl.vm, est.vm) and rl.objective == rep.objective


@pytest.mark.gpu
def test_device_template_matches_scalar_formulas_with_current_rows(G):
    """H^T W H / H^T W r of the device templates vs the host scalar formulas row by row (the test of the seven
    reference types, tests/test_gpu_parity.py, with IF / IT rows in the set)."""
    net, _, part, _ = build_case("ieee118_k3")
    ms = _with_currents(G, net, seed=1)
    bord, maps = G.build_variable_maps(net, part)
    rng = np.random.default_rng(3)
    va = rng.uniform(-0.15, 0.15, net.n_bus)
    va[net.slack] = net.buses[net.slack].va_true
    vm = rng.uniform(0.9, 1.1, net.n_bus)
    st = G.StateVector(va=va, vm=vm)
    for vmap in maps:
        lb_ang = vmap.local_boundary_angle_buses()
        x_i = vmap.gather_interior(va, vm)
        x_b = np.concatenate([va[lb_ang], vm[vmap.local_boundary_buses]])
        blk = G.fused_accumulate(vmap, ms, x_i, x_b)
        n_i, n_b = vmap.n_interior, vmap.n_boundary
        gfull, gabs = np.zeros((n_i + n_b, n_i + n_b)), np.zeros((n_i + n_b, n_i + n_b))
        bfull, babs = np.zeros(n_i + n_b), np.zeros(n_i + n_b)
        for r in range(ms.m):
            if int(ms.owner_bus[r]) not in vmap.owned_buses:
                continue
            grad = G.eval_row_gradient(net, ms.mtype[r], ms.target[r], st)
            idx = [vmap.local_index(b, q) for (b, q), _ in grad]
            val = np.array([v for _, v in grad])
            res = ms.z[r] - G.eval_h(net, ms.mtype[r], ms.target[r], st)
            gfull[np.ix_(idx, idx)] += ms.weight[r] * np.outer(val, val)
            gabs[np.ix_(idx, idx)] += ms.weight[r] * np.abs(np.outer(val, val))
            bfull[idx] += ms.weight[r] * res * val
            babs[idx] += ms.weight[r] * np.abs(res * val)
        scale = 1.0 + gabs
        assert np.max(np.abs(blk.g_ii.toarray() - gfull[:n_i, :n_i]) / scale[:n_i, :n_i]) < 1e-11
        assert np.max(np.abs(blk.g_ib.toarray() - gfull[:n_i, n_i:]) / scale[:n_i, n_i:]) < 1e-11
        assert np.max(np.abs(blk.g_bb - gfull[n_i:, n_i:]) / scale[n_i:, n_i:]) < 1e-11
        assert np.max(np.abs(blk.b_i - bfull[:n_i]) / (1.0 + babs[:n_i]), initial=0.0) < 1e-11
        assert np.max(np.abs(blk.b_b - bfull[n_i:]) / (1.0 + babs[n_i:]), initial=0.0) < 1e-11
