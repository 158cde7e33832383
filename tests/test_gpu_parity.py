"""Parity of the CUDA path (through the C ABI) against the CPU oracle and the reference-
generated golden fixtures.  Needs a B200: run with ``pytest -m gpu``.

Tolerances (BASELINE.json north_star / reference tests):
  * same GN iteration count as the reference;
  * final vm, va within 1e-8 relative; J(x) within 1e-10 relative;
  * normal-equation blocks within 5e-13 * (1 + |v|)   (reference test_assembly.py:25,131-146);
  * Schur blocks / boundary system / increments within 1e-9 (reference test_linalg.py:205-219).
"""

import numpy as np
import pytest

from conftest import BIG_CASES, SMALL_CASES, build_case, make_path4

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / (1.0 + np.abs(b)))) if a.size else 0.0


def _state_err(va, vm, gva, gvm):
    return max(float(np.max(np.abs(va - gva) / np.maximum(np.abs(gva), 1.0))),
               float(np.max(np.abs(vm - gvm) / np.abs(gvm))))


@pytest.fixture(scope="module")
def G():
    import paper_2604_23175_b200 as G
    return G


def _device_state(net):
    import torch
    st = np.stack([np.zeros(net.n_bus), np.ones(net.n_bus)])
    st[0, net.slack] = net.buses[net.slack].va_true
    return torch.from_numpy(st).cuda()


@pytest.mark.parametrize("boundary", ["dense", "sparse"])
@pytest.mark.parametrize("name", SMALL_CASES + BIG_CASES)
def test_solve_matches_reference_golden(G, name, boundary):
    net, ms, part, g = build_case(name)
    tol = 1e-10 if name == "path4_slack_boundary" else 1e-6
    est, rep = G.solve_multiarea(net, ms, part, config=G.SolverConfig(convergence_tol=tol, boundary=boundary))
    assert rep.iterations == int(g["iterations"])
    assert rep.converged == bool(g["converged"])
    assert rep.n_gamma == int(g["n_gamma"])
    assert _state_err(est.va, est.vm, g["va"], g["vm"]) < 1e-8
    jref = float(g["objective"])
    assert abs(rep.objective - jref) <= 1e-10 * max(jref, 1e-20) + 1e-25
    assert rep.weighted_residual_norm == pytest.approx(np.sqrt(rep.objective))


@pytest.mark.parametrize("name", ["ieee14_k2", "ieee118_k6", "rand300_k3_maskpf", "pegase2869_k8"])
def test_lockstep_with_oracle(G, name):
    """Every iterate equals the oracle's (same inputs) -- reference test_solver.py:122-168."""
    from oracle.mase_oracle import Oracle
    net, ms, part, _ = build_case(name)
    ref = Oracle(net, ms, part.area_of_bus).solve(trace=True)
    trace = []
    est, rep = G.solve_multiarea(net, ms, part, on_iteration=lambda it, s, d: trace.append((s, d)))
    assert rep.iterations == ref["iterations"] == len(trace)
    for i, (s, d) in enumerate(trace):
        assert np.max(np.abs(s.va - ref["trace_va"][i])) < 1e-9
        assert np.max(np.abs(s.vm - ref["trace_vm"][i])) < 1e-9
        if ref["deltas"][i] > 1e-5:
            assert d == pytest.approx(ref["deltas"][i], rel=1e-6)
    assert abs(rep.objective - ref["objective"]) <= 1e-10 * ref["objective"]


@pytest.mark.parametrize("boundary_mode", [1, 2])
@pytest.mark.parametrize("name", SMALL_CASES + ["pegase2869_k8"])
def test_phase_outputs_match_oracle(G, name, boundary_mode):
    """Blocks, Schur blocks, boundary system and increments of the first iteration
    (boundary factored as the dense chain and as the block-sparse tree)."""
    from oracle.mase_oracle import Oracle
    from paper_2604_23175_b200._native import Plan
    net, ms, part, g = build_case(name)
    bord, maps = G.build_variable_maps(net, part)
    orc = Oracle(net, ms, part.area_of_bus)
    plan = Plan(net, ms, part, bord, maps, boundary_mode=boundary_mode)
    st = _device_state(net)
    va0, vm0 = st[0].cpu().numpy().copy(), st[1].cpu().numpy().copy()
    orc.local(va0, vm0)
    plan.phase_assemble(st[0].data_ptr(), st[1].data_ptr())
    for a in range(part.k):
        ob = orc.blocks(a)
        ii_ptr, ii_idx, ib_ptr, ib_idx = plan.area_pattern(a)
        assert np.array_equal(ii_ptr, ob["ii_ptr"]) and np.array_equal(ii_idx, ob["ii_idx"])
        assert np.array_equal(ib_ptr, ob["ib_ptr"]) and np.array_equal(ib_idx, ob["ib_idx"])
        data_ii, data_ib, g_bb, b_i, b_b = plan.area_blocks(a)
        for mine, key in ((data_ii, "data_ii"), (data_ib, "data_ib"), (g_bb, "g_bb"),
                          (b_i, "b_i"), (b_b, "b_b")):
            assert _rel(mine, ob[key]) < 5e-13, (a, key)
            if f"a{a}_{key}" in g:   # and directly against the reference's values
                assert _rel(mine, g[f"a{a}_{key}"]) < 5e-13, (a, key)
    plan.phase_condense()
    for a in range(part.k):
        s_b, b_hat = plan.area_schur(a)
        os_b, ob_hat = orc.schur(a)
        assert _rel(s_b, os_b) < 1e-9 and _rel(b_hat, ob_hat) < 1e-9
        assert np.array_equal(s_b, s_b.T)
    if bord.n_gamma:
        orc.boundary()
        plan.phase_boundary()
        s_g, b_g, dx = plan.boundary_system()
        og, obg, odx = orc.boundary_system()
        assert _rel(s_g, og) < 1e-9 and _rel(b_g, obg) < 1e-9 and _rel(dx, odx) < 1e-9
        if "s_gamma" in g:
            assert _rel(s_g, g["s_gamma"]) < 1e-9 and _rel(dx, g["dx_gamma"]) < 1e-9
    dinf = plan.phase_recover(st[0].data_ptr(), st[1].data_ptr())
    odinf = orc.recover(va0, vm0)
    assert dinf == pytest.approx(odinf, rel=1e-8)
    for a in range(part.k):
        assert _rel(plan.area_delta(a), orc.interior_delta(a)) < 1e-9
    assert np.max(np.abs(st[0].cpu().numpy() - va0)) < 1e-9
    assert np.max(np.abs(st[1].cpu().numpy() - vm0)) < 1e-9
    # objective kernel vs oracle at the updated state
    j = plan.objective(st[0].data_ptr(), st[1].data_ptr())
    assert j == pytest.approx(orc.objective(va0, vm0), rel=1e-10)
    plan.close()


@pytest.mark.parametrize("boundary_mode", [1, 2])
@pytest.mark.parametrize("name", ["pegase9241_k16", "activsg10k_k32"])
def test_phase_fingerprints_match_reference_at_headline_sizes(G, name, boundary_mode):
    """BASELINE configs[2] / configs[3]: first-iteration phase outputs against the fingerprints
    make_golden.py stored from the unmodified reference (fused_accumulate -> schur_condense ->
    assemble_boundary -> dense_cholesky_solve at the flat start), then the per-iteration stacked norms
    of the reference's own solve (reference test_solver.py:122-168 at the headline sizes)."""
    from paper_2604_23175_b200._native import Plan
    net, ms, part, g = build_case(name)
    bord, maps = G.build_variable_maps(net, part)
    assert bord.n_gamma == int(g["n_gamma"])
    plan = Plan(net, ms, part, bord, maps, boundary_mode=boundary_mode)
    st = _device_state(net)
    plan.phase_assemble(st[0].data_ptr(), st[1].data_ptr())
    for a in range(part.k):
        n_i, n_b, nnz_ii, nnz_ib = (int(v) for v in g[f"a{a}_dims"])
        assert np.array_equal(maps[a].boundary_selector, g[f"a{a}_sel"])
        ii_ptr, ii_idx, ib_ptr, ib_idx = plan.area_pattern(a)
        assert (len(ii_ptr) - 1, len(ii_idx), len(ib_idx)) == (n_i, nnz_ii, nnz_ib)
        data_ii, data_ib, g_bb, b_i, b_b = plan.area_blocks(a)
        sums = g[f"a{a}_sum_ii"]          # order-sensitive at 1e-16, compared at 1e-12 (make_golden.py)
        assert abs(data_ii.sum() - sums[0]) <= 1e-12 * sums[1] and abs(np.abs(data_ii).sum() - sums[1]) <= 1e-12 * sums[1]
        assert _rel(b_i, g[f"a{a}_b_i"]) < 5e-13 and _rel(b_b, g[f"a{a}_b_b"]) < 5e-13, a
    plan.phase_condense()
    for a in range(part.k):
        s_b, b_hat = plan.area_schur(a)
        assert _rel(np.diag(s_b), g[f"a{a}_sb_diag"]) < 1e-9 and _rel(b_hat, g[f"a{a}_b_hat"]) < 1e-9, a
    plan.phase_boundary()
    s_g, b_g, dx = plan.boundary_system()
    assert _rel(np.diag(s_g), g["s_gamma_diag"]) < 1e-9
    assert _rel(b_g, g["b_gamma"]) < 1e-9 and _rel(dx, g["dx_gamma"]) < 1e-9
    plan.close()
    # the reference's per-iteration norms, through the persistent kernel (last_deltas) and the callback loop
    trace = []
    est, rep = G.solve_multiarea(net, ms, part, config=G.SolverConfig(boundary={1: "dense", 2: "sparse"}[boundary_mode]),
                                 on_iteration=lambda it, s, d: trace.append(d))
    ref_d = g["deltas"]
    assert rep.iterations == len(ref_d) == len(trace)
    assert np.allclose(trace, ref_d, rtol=1e-6, atol=1e-12)
    warm = G.MultiAreaEstimator(net, ms, part, config=G.SolverConfig(boundary={1: "dense", 2: "sparse"}[boundary_mode]))
    est2, rep2 = warm.estimate()
    assert np.allclose(warm.last_deltas[:rep2.iterations], ref_d, rtol=1e-6, atol=1e-12)
    assert np.array_equal(est2.va, est.va) and np.array_equal(est2.vm, est.vm)
    warm.close()


def _single_area(G, net):
    part = G.partition_network(net, 1)
    _, maps = G.build_variable_maps(net, part)
    return maps[0]


def test_fused_accumulate_hand_example(G):
    # reference test_assembly.py:66-76: one VM row, sigma 0.5 -> g_ii = [[4]], b_i = [0.8]
    net = G.BusBranchNetwork.from_components([G.Bus(id=1, is_slack=True)], [])
    ms = G.make_measurement_set(net, [int(G.MeasurementType.VM)], [0], z=[1.2], sigma=[0.5])
    vmap = _single_area(G, net)
    blocks = G.fused_accumulate(vmap, ms, np.ones(1), np.zeros(0))
    assert blocks.g_ii.toarray() == pytest.approx(np.array([[4.0]]))
    assert blocks.b_i == pytest.approx(np.array([0.8]))
    assert blocks.g_ib.shape == (1, 0) and blocks.g_bb.shape == (0, 0)


def test_fused_accumulate_masking_and_determinism(G):
    # reference test_assembly.py:79-87,200-216,242-252
    net = make_path4()
    ms = G.generate_measurements(net)
    vmap = _single_area(G, net)
    rng = np.random.default_rng(1)
    x_i = np.concatenate([rng.uniform(-0.15, 0.15, 3), rng.uniform(0.9, 1.1, 4)])
    pat = G.build_patterns(vmap, ms)
    b1 = G.fused_accumulate(vmap, ms, x_i, np.zeros(0), pattern=pat)
    b2 = G.fused_accumulate(vmap, ms, x_i, np.zeros(0), pattern=pat)
    assert np.array_equal(b1.g_ii.data, b2.g_ii.data) and np.array_equal(b1.b_i, b2.b_i)
    assert np.max(np.abs(b1.g_ii.toarray() - b1.g_ii.toarray().T)) < 1e-12 * np.max(np.abs(b1.g_ii.data))
    zero = G.fused_accumulate(vmap, G.apply_mask(ms, np.ones(ms.m, dtype=bool)), x_i, np.zeros(0), pattern=pat)
    assert np.all(zero.g_ii.data == 0.0) and np.all(zero.b_i == 0.0)
    # masked == deleted
    fam = G.MeasurementType.PF
    masked = G.fused_accumulate(vmap, G.apply_mask(ms, fam), x_i, np.zeros(0), pattern=pat)
    keep = ms.mtype != int(fam)
    trimmed = G.make_measurement_set(net, ms.mtype[keep], ms.target[keep], ms.z[keep], ms.sigma[keep])
    deleted = G.fused_accumulate(vmap, trimmed, x_i, np.zeros(0))
    assert _rel(masked.g_ii.toarray(), deleted.g_ii.toarray()) < 5e-13
    assert _rel(masked.b_i, deleted.b_i) < 5e-13


def test_templates_match_scalar_formulas(G):
    """Device templates vs the scalar per-row formulas (reference test_assembly.py:255-280):
    H^T W H and H^T W r rebuilt row by row on the host from eval_row_gradient / eval_h."""
    net, ms, part, _ = build_case("ieee118_k3")
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
        gfull = np.zeros((n_i + n_b, n_i + n_b))
        gabs = np.zeros((n_i + n_b, n_i + n_b))   # sum of |terms|: the scale rounding errors live on
        bfull = np.zeros(n_i + n_b)
        babs = np.zeros(n_i + n_b)
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
        assert np.max(np.abs(blk.g_ii.toarray() - gfull[:n_i, :n_i]) / scale[:n_i, :n_i]) < 1e-12
        assert np.max(np.abs(blk.g_ib.toarray() - gfull[:n_i, n_i:]) / scale[:n_i, n_i:]) < 1e-12
        assert np.max(np.abs(blk.g_bb - gfull[n_i:, n_i:]) / scale[n_i:, n_i:]) < 1e-12
        assert np.max(np.abs(blk.b_i - bfull[:n_i]) / (1.0 + babs[:n_i]), initial=0.0) < 1e-12
        assert np.max(np.abs(blk.b_b - bfull[n_i:]) / (1.0 + babs[n_i:]), initial=0.0) < 1e-12


def test_bitwise_repeatable_and_warm_path(G):
    # reference test_solver.py:314-322 + the warm estimator
    net, ms, part, g = build_case("ieee118_k6")
    e1, r1 = G.solve_multiarea(net, ms, part)
    e2, r2 = G.solve_multiarea(net, ms, part)
    assert np.array_equal(e1.va, e2.va) and np.array_equal(e1.vm, e2.vm)
    assert r1.objective == r2.objective and r1.iterations == r2.iterations
    est = G.MultiAreaEstimator(net, ms, part)
    e3, r3 = est.estimate()
    e4, r4 = est.estimate()
    assert np.array_equal(e3.va, e1.va) and np.array_equal(e4.vm, e1.vm)
    # masking = weight refresh on the same plan == a fresh solve of the masked set
    masked = G.apply_mask(ms, G.MeasurementType.QT)
    est.update_measurements(masked)
    e5, r5 = est.estimate()
    e6, r6 = G.solve_multiarea(net, masked, part)
    assert np.array_equal(e5.va, e6.va) and r5.iterations == r6.iterations
    est.close()


def test_dense_backend_agrees_with_sparse(G):
    net, ms, part, g = build_case("rand120_k4")
    es, rs = G.solve_multiarea(net, ms, part, config=G.SolverConfig(backend="sparse"))
    ed, rd = G.solve_multiarea(net, ms, part, config=G.SolverConfig(backend="dense"))
    assert rs.iterations == rd.iterations
    assert max(np.max(np.abs(es.va - ed.va)), np.max(np.abs(es.vm - ed.vm))) < 1e-9


def test_iteration_cap_and_report(G):
    net, ms, part, g = build_case("ieee14_k2")
    est, rep = G.solve_multiarea(net, ms, part, config=G.SolverConfig(max_outer_iterations=1))
    assert not rep.converged and rep.iterations == 1
    assert np.all(np.isfinite(est.va)) and np.all(np.isfinite(est.vm))
    _, rep = G.solve_multiarea(net, ms, part, config=G.SolverConfig(profile_phases=True))
    doc = rep.to_dict()
    assert doc["method"] == "multiarea"
    for phase in ("assembly", "local_condense", "boundary_assemble", "boundary_solve", "recovery"):
        assert phase in doc["timings"] and doc["timings"][phase] > 0.0
    assert sum(v for k, v in doc["timings"].items() if k != "total") <= doc["timings"]["total"]


def test_centralized_k1_and_every_bus_its_own_area(G):
    from oracle.mase_oracle import Oracle
    net, ms, part, g = build_case("ieee14_k1")
    ec, rc = G.solve_centralized(net, ms)
    assert rc.method == "centralized" and rc.n_gamma == 0 and rc.iterations == int(g["iterations"])
    assert _state_err(ec.va, ec.vm, g["va"], g["vm"]) < 1e-8
    net, ms, part, g = build_case("ieee14_k14")   # n_i = 0 everywhere
    em, rm = G.solve_multiarea(net, ms, part)
    assert rm.iterations == int(g["iterations"]) and _state_err(em.va, em.vm, g["va"], g["vm"]) < 1e-8


@pytest.mark.parametrize("name", ["ieee14_centralized_refined", "ieee118_centralized_refined"])
def test_centralized_with_iterative_refinement_matches_reference(G, name):
    """SolverConfig(iterative_refinement=True) -- read by solve_centralized only (reference
    solver.py:181-183): same iteration count, per-iteration norms and iterates as the reference's run."""
    net, ms, part, g = build_case(name)
    trace = []
    est, rep = G.solve_centralized(net, ms, config=G.SolverConfig(iterative_refinement=True),
                                   on_iteration=lambda it, s, d: trace.append((s, d)))
    assert rep.method == "centralized" and rep.n_gamma == 0
    assert rep.iterations == int(g["iterations"]) and rep.converged == bool(g["converged"])
    assert _state_err(est.va, est.vm, g["va"], g["vm"]) < 1e-8          # north_star tolerance
    assert abs(rep.objective - float(g["objective"])) <= 1e-10 * float(g["objective"])
    for (s, d), va, vm, dref in zip(trace, g["trace_va"], g["trace_vm"], g["deltas"]):
        assert _state_err(s.va, s.vm, va, vm) < 1e-9 and abs(d - dref) <= 1e-9 * (1 + dref)
    assert set(rep.timings) == {"assembly", "local_condense", "boundary_assemble", "boundary_solve", "recovery", "total"}
    # and the plain centralized solve agrees with it to rounding (the refinement only polishes)
    plain, rplain = G.solve_centralized(net, ms)
    assert rplain.iterations == rep.iterations and _state_err(plain.va, plain.vm, est.va, est.vm) < 1e-10


def test_unobservable_raises_solver_error(G):
    # reference test_solver.py:335-342
    net, ms, part, _ = build_case("ieee14_k2")
    vm_only = G.apply_mask(ms, lambda t, tg: t != G.MeasurementType.VM)
    with pytest.raises(G.SolverError, match="unobservable|not positive definite"):
        G.solve_centralized(net, vm_only)
    with pytest.raises(G.SolverError, match="area"):
        G.solve_multiarea(net, vm_only, part)


def test_noiseless_recovers_truth(G):
    # reference test_solver.py:80-92
    net, _, part, _ = build_case("ieee14_k3")
    ms = G.generate_measurements(net, G.MeasurementConfig(sigma_vm=0.0, sigma_power=0.0))
    est, rep = G.solve_multiarea(net, ms, part, config=G.SolverConfig(convergence_tol=1e-10))
    truth = G.StateVector.truth(net)
    assert rep.converged
    assert max(np.max(np.abs(est.va - truth.va)), np.max(np.abs(est.vm - truth.vm))) < 1e-8
    assert rep.objective < 1e-16 * ms.m


def test_weight_scaling_property_full_size(G):
    """Size-independent property at the BASELINE size: scaling every weight by c leaves the
    estimate unchanged (to rounding) and scales J by c."""
    net, ms, part, g = build_case("pegase9241_k16")
    est = G.MultiAreaEstimator(net, ms, part)
    e1, r1 = est.estimate()
    from dataclasses import replace
    est.update_measurements(replace(ms, weight=ms.weight * 4.0))
    e2, r2 = est.estimate()
    est.close()
    assert r1.iterations == r2.iterations == int(g["iterations"])
    assert max(np.max(np.abs(e1.va - e2.va)), np.max(np.abs(e1.vm - e2.vm))) < 1e-10
    assert r2.objective == pytest.approx(4.0 * r1.objective, rel=1e-10)


@pytest.mark.parametrize("name,inner", [("ieee118_k6_inner2", 2), ("rand120_k4_inner3", 3)])
def test_inner_gn_steps_match_reference_golden(G, name, inner):
    """SolverConfig.inner_gn_steps > 1 (reference solver.py:253-260): same iteration count, per-iteration
    stacked norms, iterates, final state and J as the reference run stored in the fixture."""
    net, ms, part, g = build_case(name)
    trace = []
    est, rep = G.solve_multiarea(net, ms, part, config=G.SolverConfig(inner_gn_steps=inner),
                                 on_iteration=lambda it, s, d: trace.append((s, d)))
    assert rep.iterations == int(g["iterations"]) and rep.converged == bool(g["converged"])
    assert np.allclose([d for _, d in trace], g["deltas"], rtol=1e-6, atol=1e-12)
    for (s, _), va, vm in zip(trace, g["trace_va"], g["trace_vm"]):
        assert np.max(np.abs(s.va - va)) < 1e-9 and np.max(np.abs(s.vm - vm)) < 1e-9
    assert _state_err(est.va, est.vm, g["va"], g["vm"]) < 1e-8
    assert abs(rep.objective - float(g["objective"])) <= 1e-10 * float(g["objective"])
    # without the callback the same loop runs (inner steps are host-sequenced): identical result
    est2, rep2 = G.solve_multiarea(net, ms, part, config=G.SolverConfig(inner_gn_steps=inner))
    assert rep2.iterations == rep.iterations and np.array_equal(est2.va, est.va) and np.array_equal(est2.vm, est.vm)


def test_fused_matches_explicit_jacobian_path(G):
    """reference test_assembly.py:90-140: ``explicit_assemble`` materialises H (here: the template values the device
    kernel wrote, read back through gse_area_templates) and forms the blocks by sparse triple products on the host;
    ``fused_accumulate`` must agree, which isolates the device accumulation program.  The triplets also reproduce
    the scalar per-row gradients."""
    net, ms, part, _ = build_case("ieee118_k3")
    bord, maps = G.build_variable_maps(net, part)
    rng = np.random.default_rng(11)
    va = rng.uniform(-0.15, 0.15, net.n_bus)
    va[net.slack] = net.buses[net.slack].va_true
    vm = rng.uniform(0.9, 1.1, net.n_bus)
    st = G.StateVector(va=va, vm=vm)
    for vmap in maps:
        lb_ang = vmap.local_boundary_angle_buses()
        x_i = vmap.gather_interior(va, vm)
        x_b = np.concatenate([va[lb_ang], vm[vmap.local_boundary_buses]])
        pat = G.build_patterns(vmap, ms)
        fused = G.fused_accumulate(vmap, ms, x_i, x_b, pattern=pat)
        trip, expl = G.explicit_assemble(vmap, ms, x_i, x_b, pattern=pat)
        assert isinstance(trip, G.JacobianTriplets) and trip.n_cols == vmap.n_interior + vmap.n_boundary
        h = trip.to_csr()
        assert h.shape == (len(pat.row_ids), trip.n_cols)
        scale = 1.0 + (abs(h).T @ (abs(h).multiply(trip.weights[:, None]))).toarray()
        n_i = vmap.n_interior
        assert np.max(np.abs(fused.g_ii.toarray() - expl.g_ii.toarray()) / scale[:n_i, :n_i]) < 1e-12
        assert np.max(np.abs(fused.g_ib.toarray() - expl.g_ib.toarray()) / scale[:n_i, n_i:], initial=0.0) < 1e-12
        assert np.max(np.abs(fused.g_bb - expl.g_bb) / scale[n_i:, n_i:], initial=0.0) < 1e-12
        bscale = 1.0 + np.asarray(abs(h).T @ np.abs(trip.weights * trip.residuals)).ravel()
        assert np.max(np.abs(fused.b_i - expl.b_i) / bscale[:n_i]) < 1e-12
        assert np.max(np.abs(fused.b_b - expl.b_b) / bscale[n_i:], initial=0.0) < 1e-12
        # a few rows against the scalar formulas
        for k in range(0, len(pat.row_ids), 37):
            r = int(pat.row_ids[k])
            grad = G.eval_row_gradient(net, ms.mtype[r], ms.target[r], st)
            dense_row = np.zeros(trip.n_cols)
            for (b, q), v in grad:
                dense_row[vmap.local_index(b, q)] += v
            assert np.max(np.abs(h[k].toarray().ravel() - dense_row)) < 1e-12 * (1.0 + np.max(np.abs(dense_row)))
            assert trip.residuals[k] == pytest.approx(ms.z[r] - G.eval_h(net, ms.mtype[r], ms.target[r], st), rel=1e-12, abs=1e-14)
