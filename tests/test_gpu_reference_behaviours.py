"""The reference's own behavioural tests of the solve path, run against the device solvers: the cases of reference
tests/test_solver.py, test_assembly.py and test_linalg.py that the golden-fixture suites do not already replay
(each test names the reference test it mirrors).  Needs a B200: ``pytest -m gpu``."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import make_path4

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import paper_2604_23175_b200 as G
    return G


@pytest.fixture(scope="module")
def net14(G):
    import os
    return G.load_case(os.path.join(os.path.dirname(G.__file__), "cases", "ieee14.m"))


@pytest.fixture(scope="module")
def net118(G):
    import os
    return G.load_case(os.path.join(os.path.dirname(G.__file__), "cases", "ieee118.m"))


def _diff(a, b):
    return max(np.max(np.abs(a.va - b.va)), np.max(np.abs(a.vm - b.vm)))


def _lockstep(G, net, ms, part):
    """Per-iteration iterates of the centralized and the multi-area device solves (reference run_lockstep)."""
    tc, tm = [], []
    _, rc = G.solve_centralized(net, ms, on_iteration=lambda t, s, d: tc.append(s))
    _, rm = G.solve_multiarea(net, ms, part, on_iteration=lambda t, s, d: tm.append(s))
    assert len(tc) == len(tm) and rc.iterations == rm.iterations
    return max(_diff(a, b) for a, b in zip(tc, tm)), rc, rm


# ---- objective (reference test_solver.py:41-73) -------------------------------------------------------------

def test_objective_zero_at_truth_and_single_row(G):
    net = make_path4()
    ms = G.generate_measurements(net, G.MeasurementConfig(sigma_vm=0.0, sigma_power=0.0))
    assert G.objective(ms, G.StateVector.truth(net)) < 1e-20
    one = G.BusBranchNetwork.from_components([G.Bus(id=1, is_slack=True)], [])
    row = G.make_measurement_set(one, [int(G.MeasurementType.VM)], [0], z=[1.0], sigma=[0.5])
    st = G.StateVector.flat_start(one)
    st.vm[0] = 0.0
    assert G.objective(row, st) == pytest.approx(4.0)            # z = 1, h = 0, w = 4


def test_objective_ignores_masked_rows(G, net14):
    ms = G.generate_measurements(net14)
    st = G.StateVector.flat_start(net14)
    masked = G.apply_mask(ms, G.MeasurementType.PINJ)
    keep = ms.mtype != int(G.MeasurementType.PINJ)
    trimmed = G.make_measurement_set(net14, ms.mtype[keep], ms.target[keep], ms.z[keep], ms.sigma[keep])
    assert G.objective(masked, st) == pytest.approx(G.objective(trimmed, st), rel=1e-13)


# ---- fixed points and toy problems (reference test_solver.py:80-118) -----------------------------------------

@pytest.mark.parametrize("method", ["centralized", "multiarea"])
def test_noiseless_recovers_truth_ieee14(G, net14, method):
    ms = G.generate_measurements(net14, G.MeasurementConfig(sigma_vm=0.0, sigma_power=0.0))
    cfg = G.SolverConfig(convergence_tol=1e-10)
    if method == "centralized":
        est, rep = G.solve_centralized(net14, ms, cfg)
    else:
        est, rep = G.solve_multiarea(net14, ms, G.partition_network(net14, 3, seed=0), config=cfg)
    assert rep.converged and _diff(est, G.StateVector.truth(net14)) < 1e-8
    assert rep.objective < 1e-16 * ms.m


def test_linear_toy_single_iteration_exact(G):
    # a magnitude-only problem is linear: the first GN step lands exactly, the follow-up update is exactly zero
    net = G.BusBranchNetwork.from_components([G.Bus(id=1, is_slack=True)], [])
    ms = G.make_measurement_set(net, [int(G.MeasurementType.VM)], [0], z=[1.013], sigma=[0.01])
    states = []
    est, rep = G.solve_centralized(net, ms, G.SolverConfig(), on_iteration=lambda t, s, d: states.append((s, d)))
    assert rep.converged
    assert states[0][0].vm[0] == pytest.approx(1.013, abs=1e-15)
    assert states[-1][1] == 0.0 or states[-1][1] < 1e-15


# ---- lockstep equivalence of the two formulations on the device (reference test_solver.py:122-168) -----------

def test_lockstep_ieee14_k2_k3(G, net14):
    ms = G.generate_measurements(net14, G.MeasurementConfig(seed=2))
    for k in (2, 3):
        worst, rc, rm = _lockstep(G, net14, ms, G.partition_network(net14, k, seed=0))
        assert worst < 1e-9
        assert rm.objective == pytest.approx(rc.objective, rel=1e-10)


def test_lockstep_random_net_with_taps_and_shifts(G):
    from paper_2604_23175_b200 import synth
    net = synth.random_network(40, seed=77)
    ms = G.generate_measurements(net, G.MeasurementConfig(seed=3))
    worst, _, _ = _lockstep(G, net, ms, G.partition_network(net, 3, seed=0))
    assert worst < 1e-9


def test_lockstep_every_bus_its_own_area_and_two_bus_all_boundary(G):
    from paper_2604_23175_b200 import synth
    path4 = make_path4()
    ms = G.generate_measurements(path4, G.MeasurementConfig(seed=0))
    worst, _, rm = _lockstep(G, path4, ms, G.load_partition(path4, [0, 1, 2, 3]))
    assert rm.n_gamma == 2 * 4 - 1 and worst < 1e-11          # k = n_bus: all interiors empty
    two = synth.random_network(2, seed=0, extra_frac=0.0)
    ms2 = G.generate_measurements(two, G.MeasurementConfig(seed=1))
    worst, _, rm = _lockstep(G, two, ms2, G.load_partition(two, [0, 1]))
    assert rm.n_gamma == 3 and worst < 1e-11


def test_observable_without_magnitude_rows(G, net14):
    full = G.generate_measurements(net14, G.MeasurementConfig(seed=3))
    keep = full.mtype != int(G.MeasurementType.VM)
    sub = G.make_measurement_set(net14, full.mtype[keep], full.target[keep], full.z[keep], full.sigma[keep])
    _, rc = G.solve_centralized(net14, sub)
    _, rm = G.solve_multiarea(net14, sub, G.partition_network(net14, 3, seed=0))
    assert rc.converged and rm.converged
    assert rm.objective == pytest.approx(rc.objective, rel=1e-9)


def test_multiarea_noisy_matches_centralized_objective(G, net118):
    ms = G.generate_measurements(net118, G.MeasurementConfig(seed=0))
    _, rc = G.solve_centralized(net118, ms)
    _, rm = G.solve_multiarea(net118, ms, G.partition_network(net118, 6, seed=0))
    assert rc.converged and rm.converged
    assert rm.objective == pytest.approx(rc.objective, rel=1e-6)


def test_inner_gn_steps_variant_reaches_the_same_optimum(G, net14):
    ms = G.generate_measurements(net14, G.MeasurementConfig(seed=4))
    est, rep = G.solve_multiarea(net14, ms, G.partition_network(net14, 2, seed=0), config=G.SolverConfig(inner_gn_steps=3))
    ref, _ = G.solve_centralized(net14, ms)
    assert rep.converged and _diff(est, ref) < 1e-6


# ---- convergence semantics and reporting (reference test_solver.py:270-330) -----------------------------------

def test_converged_iff_final_delta_below_tol_and_objective_decreases(G, net14, net118):
    ms = G.generate_measurements(net118, G.MeasurementConfig(seed=8))
    deltas = []
    _, rep = G.solve_centralized(net118, ms, G.SolverConfig(), on_iteration=lambda t, s, d: deltas.append(d))
    assert rep.converged == (deltas[-1] < G.SolverConfig().convergence_tol)
    for net, seed in ((net14, 0), (net118, 1)):
        ms = G.generate_measurements(net, G.MeasurementConfig(seed=seed))
        objs = []
        G.solve_centralized(net, ms, G.SolverConfig(), on_iteration=lambda t, s, d: objs.append(G.objective(ms, s)))
        assert all(b < a for a, b in zip(objs, objs[1:]))


def test_report_fields_and_json(G, net14):
    ms = G.generate_measurements(net14)
    part = G.partition_network(net14, 2, seed=0)
    _, rep = G.solve_multiarea(net14, ms, part)
    doc = rep.to_dict()
    assert doc["method"] == "multiarea"
    assert doc["n_gamma"] == 2 * len(part.boundary_buses) - (1 if net14.slack in part.boundary_buses else 0)
    for phase in ("assembly", "local_condense", "boundary_assemble", "boundary_solve", "recovery"):
        assert phase in doc["timings"]
    assert sum(v for k, v in doc["timings"].items() if k != "total") <= doc["timings"]["total"]
    assert doc["objective"] >= 0.0 and doc["weighted_residual_norm"] == pytest.approx(np.sqrt(doc["objective"]))


def test_parallel_mode_matches_deterministic(G, net118):
    # (the device path has one mode: every reduction order is fixed; the flag must not change a bit)
    ms = G.generate_measurements(net118, G.MeasurementConfig(seed=10))
    part = G.partition_network(net118, 4, seed=0)
    est_d, rep_d = G.solve_multiarea(net118, ms, part, config=G.SolverConfig(deterministic=True))
    est_p, rep_p = G.solve_multiarea(net118, ms, part, config=G.SolverConfig(deterministic=False))
    assert np.array_equal(est_d.va, est_p.va) and np.array_equal(est_d.vm, est_p.vm) and rep_d.iterations == rep_p.iterations


def test_unobservable_system_raises_in_both_formulations(G, net14):
    ms = G.generate_measurements(net14)
    vm_only = G.apply_mask(ms, lambda t, tg: t != G.MeasurementType.VM)
    with pytest.raises(G.SolverError, match="unobservable|not positive definite"):
        G.solve_centralized(net14, vm_only)
    with pytest.raises(G.SolverError, match="area"):
        G.solve_multiarea(net14, vm_only, G.partition_network(net14, 2, seed=0))


# ---- assembly (reference test_assembly.py:79-216) ---------------------------------------------------------------

def _single_area(G, net):
    part = G.partition_network(net, 1)
    return G.build_variable_maps(net, part)[1][0]


def test_vm_only_identity_and_noiseless_rhs_vanishes(G):
    net = make_path4()
    vmap = _single_area(G, net)
    truth = G.StateVector.truth(net)
    x_i = vmap.gather_interior(truth.va, truth.vm)
    ms = G.generate_measurements(net, G.MeasurementConfig(sigma_vm=0.0, sigma_power=0.0))
    blk = G.fused_accumulate(vmap, ms, x_i, np.zeros(0))
    assert np.max(np.abs(blk.b_i)) < 1e-9 * np.max(np.abs(blk.g_ii.data))      # z = h(x_true): H^T W r = 0
    vm_rows = ms.mtype == int(G.MeasurementType.VM)
    only = G.make_measurement_set(net, ms.mtype[vm_rows], ms.target[vm_rows], ms.z[vm_rows], np.full(int(vm_rows.sum()), 0.5))
    g = G.fused_accumulate(vmap, only, x_i, np.zeros(0)).g_ii.toarray()
    na = len(vmap.interior_angle_buses)
    assert np.all(g[:na] == 0.0) and np.array_equal(g[na:, na:], 4.0 * np.eye(net.n_bus))


def test_additivity_of_disjoint_subsets_and_pattern_reuse(G, net14):
    ms = G.generate_measurements(net14, G.MeasurementConfig(seed=2))
    vmap = _single_area(G, net14)
    rng = np.random.default_rng(4)
    x_i = np.concatenate([rng.uniform(-0.1, 0.1, len(vmap.interior_angle_buses)), rng.uniform(0.95, 1.05, net14.n_bus)])
    pat = G.build_patterns(vmap, ms)
    full = G.fused_accumulate(vmap, ms, x_i, np.zeros(0), pattern=pat)
    fresh = G.fused_accumulate(vmap, ms, x_i, np.zeros(0))
    assert np.array_equal(full.g_ii.data, fresh.g_ii.data) and np.array_equal(full.b_i, fresh.b_i)
    half = np.arange(ms.m) % 2 == 0
    a = G.fused_accumulate(vmap, G.apply_mask(ms, half), x_i, np.zeros(0), pattern=pat)
    b = G.fused_accumulate(vmap, G.apply_mask(ms, ~half), x_i, np.zeros(0), pattern=pat)
    scale = 1.0 + np.abs(full.g_ii.toarray())
    assert np.max(np.abs(a.g_ii.toarray() + b.g_ii.toarray() - full.g_ii.toarray()) / scale) < 1e-12
    assert np.max(np.abs(a.b_i + b.b_i - full.b_i) / (1.0 + np.abs(full.b_i))) < 1e-10
    # the analysed pattern covers the numeric support
    sup = full.g_ii.toarray() != 0.0
    assert np.all(pat.gii_pattern().toarray()[sup] != 0.0)


# ---- linear algebra (reference test_linalg.py:60-260) ------------------------------------------------------------

def _solve_check(G, a, rng, tol=1e-9):
    cache = G.symbolic_analyze(a)
    G.numeric_refactor(cache, a)
    b = rng.standard_normal(a.shape[0])
    x = cache.solve(b)
    assert np.max(np.abs(a @ x - b)) < tol * (1.0 + np.max(np.abs(b)))
    return cache


def test_diagonal_tridiagonal_and_arrow_patterns(G):
    rng = np.random.default_rng(0)
    n = 80
    _solve_check(G, sp.diags(rng.uniform(1.0, 2.0, n)).tocsr(), rng).close()
    tri = sp.diags([np.full(n - 1, -1.0), np.full(n, 2.5), np.full(n - 1, -1.0)], [-1, 0, 1]).tocsr()
    _solve_check(G, tri, rng).close()
    arrow = sp.lil_matrix((n, n))
    arrow.setdiag(4.0 + np.arange(n) * 0.01)
    arrow[0, 1:] = 0.1
    arrow[1:, 0] = 0.1
    _solve_check(G, sp.csr_matrix(arrow), rng).close()


def test_refactor_zero_values_fails_and_symbolic_reuse_and_projection(G):
    rng = np.random.default_rng(3)
    n = 70
    tri = sp.diags([np.full(n - 1, -1.0), np.full(n, 2.5), np.full(n - 1, -1.0)], [-1, 0, 1]).tocsr()
    cache = G.symbolic_analyze(tri)
    with pytest.raises(G.NotPositiveDefiniteError):
        G.numeric_refactor(cache, np.zeros(tri.nnz))
    with pytest.raises(RuntimeError):
        cache.solve(np.ones(n))                                   # no valid factor after the failure
    for scale in (1.0, 3.0, 0.25):                                # symbolic reuse across value updates
        G.numeric_refactor(cache, tri.data * scale)
        b = rng.standard_normal(n)
        assert np.max(np.abs(scale * (tri @ cache.solve(b)) - b)) < 1e-10 * (1.0 + np.max(np.abs(b)))
    diag_only = sp.diags(np.full(n, 3.0)).tocsr()                  # a matrix with a sub-pattern projects onto it
    G.numeric_refactor(cache, diag_only)
    assert np.allclose(cache.solve(np.full(n, 6.0)), 2.0, rtol=0, atol=1e-13)
    outside = sp.lil_matrix((n, n))
    outside.setdiag(3.0)
    outside[0, n - 1] = outside[n - 1, 0] = 0.5
    with pytest.raises(ValueError):
        G.numeric_refactor(cache, sp.csr_matrix(outside))
    cache.close()


def test_schur_decoupled_blocks_spd_propagation_and_zero_boundary_delta(G):
    rng = np.random.default_rng(5)
    n_i, n_b = 90, 7
    m = sp.random(n_i, n_i, density=0.04, random_state=np.random.RandomState(5), format="csr")
    g_ii = sp.csr_matrix(m + m.T + sp.eye(n_i) * (1.0 + abs(m).sum(axis=1).max() * 2))
    g_ii.sort_indices()
    cache = G.symbolic_analyze(g_ii)
    G.numeric_refactor(cache, g_ii.data)
    b_i, b_b = rng.standard_normal(n_i), rng.standard_normal(n_b)
    # decoupled: G_ib = 0 -> S_b = G_bb, b_hat = b_b
    g_bb = np.diag(rng.uniform(2.0, 3.0, n_b))
    res = G.schur_condense(cache, sp.csr_matrix((n_i, n_b)), g_bb, b_i, b_b)
    assert np.allclose(res.s_b, g_bb, rtol=0, atol=1e-14) and np.allclose(res.b_hat, b_b, rtol=0, atol=1e-14)
    # coupled: S_b of an SPD matrix stays SPD; zero boundary delta recovers the plain interior solve
    g_ib = sp.random(n_i, n_b, density=0.1, random_state=np.random.RandomState(6), format="csr") * 0.3
    full = np.block([[g_ii.toarray(), g_ib.toarray()], [g_ib.toarray().T, g_bb + 2.0 * np.eye(n_b)]])
    assert np.min(np.linalg.eigvalsh(full)) > 0
    res = G.schur_condense(cache, g_ib, g_bb + 2.0 * np.eye(n_b), b_i, b_b)
    assert np.min(np.linalg.eigvalsh(res.s_b)) > 0 and np.allclose(res.s_b, res.s_b.T, rtol=0, atol=1e-13)
    dx = G.interior_recover(cache, g_ib, b_i, np.zeros(n_b))
    assert np.max(np.abs(dx - np.linalg.solve(g_ii.toarray(), b_i))) < 1e-10
    cache.close()


def test_iterative_refinement_pass_and_stats(G):
    rng = np.random.default_rng(9)
    n = 150
    m = sp.random(n, n, density=0.03, random_state=np.random.RandomState(9), format="csr")
    a = sp.csr_matrix(m + m.T + sp.eye(n) * (1.0 + abs(m).sum(axis=1).max()))
    a.sort_indices()
    cache = G.symbolic_analyze(a)
    G.numeric_refactor(cache, a.data)
    b = rng.standard_normal(n)
    x0, x1 = cache.solve(b), cache.solve(b, refine_with=a)
    assert np.max(np.abs(a @ x1 - b)) <= np.max(np.abs(a @ x0 - b)) * 1.5 + 1e-15
    st = cache.stats()
    assert st["n"] == n and st["pattern_nnz"] == a.nnz and st["mode"] == "sparse"
    small = G.symbolic_analyze(sp.eye(10, format="csr"))
    assert small.mode == "dense"                                   # dense fallback below the threshold
    small.close(); cache.close()
