"""Pin the CPU oracle (oracle/mase_oracle.c) against fixtures generated from the
unmodified reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import BIG_CASES, SMALL_CASES, build_case
from oracle.mase_oracle import Oracle, OracleError, dense_cholesky_solve


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / (1.0 + np.abs(b)))) if a.size else 0.0


@pytest.mark.parametrize("name", SMALL_CASES + ["pegase2869_k8"])
def test_blocks_schur_boundary_match_reference(name):
    net, ms, part, g = build_case(name)
    assert np.array_equal(ms.z, g["z"]) and np.array_equal(ms.weight, g["weight"])
    orc = Oracle(net, ms, part.area_of_bus)
    assert orc.n_gamma == int(g["n_gamma"])
    st_va = np.zeros(net.n_bus)
    st_va[net.slack] = net.buses[net.slack].va_true
    st_vm = np.ones(net.n_bus)
    orc.local(st_va, st_vm)
    for a in range(part.k):
        d, blk = orc.dims(a), orc.blocks(a)
        assert [d["n_i"], d["n_b"], d["nnz_ii"], d["nnz_ib"]] == list(g[f"a{a}_dims"])
        assert np.array_equal(orc.selector(a), g[f"a{a}_sel"])
        assert np.array_equal(blk["ii_ptr"], g[f"a{a}_ii_ptr"])
        assert np.array_equal(blk["ii_idx"], g[f"a{a}_ii_idx"])
        assert np.array_equal(blk["ib_idx"], g[f"a{a}_ib_idx"])
        # the accumulation order is restated exactly: bit-identical blocks
        for key in ("data_ii", "data_ib", "g_bb", "b_i", "b_b"):
            assert _rel(blk[key], g[f"a{a}_{key}"]) <= 1e-14, (a, key)
        s_b, b_hat = orc.schur(a)
        assert _rel(s_b, g[f"a{a}_s_b"]) < 1e-9
        assert _rel(b_hat, g[f"a{a}_b_hat"]) < 1e-9
    if orc.n_gamma:
        orc.boundary()
        s_g, b_g, dx = orc.boundary_system()
        assert _rel(s_g, g["s_gamma"]) < 1e-9
        assert _rel(b_g, g["b_gamma"]) < 1e-9
        assert _rel(dx, g["dx_gamma"]) < 1e-9


@pytest.mark.parametrize("name", SMALL_CASES + BIG_CASES)
def test_solve_matches_reference(name):
    net, ms, part, g = build_case(name)
    zs = g["z_sum"]
    assert abs(ms.z.sum() - zs[0]) <= 1e-9 * max(1.0, abs(zs[1]))
    tol = 1e-10 if name == "path4_slack_boundary" else 1e-6
    res = Oracle(net, ms, part.area_of_bus).solve(tol=tol, trace=True)
    assert res["iterations"] == int(g["iterations"])
    assert res["converged"] == bool(g["converged"])
    assert np.max(np.abs(res["va"] - g["va"])) < 1e-9
    assert np.max(np.abs(res["vm"] - g["vm"]) / g["vm"]) < 1e-9
    jref = float(g["objective"])
    assert abs(res["objective"] - jref) <= 1e-10 * max(jref, 1e-20) + 1e-25
    big = g["deltas"] > 1e-5
    assert np.allclose(res["deltas"][big], g["deltas"][big], rtol=1e-6)
    if "trace_va" in g:
        assert np.max(np.abs(res["trace_va"] - g["trace_va"])) < 1e-9
        assert np.max(np.abs(res["trace_vm"] - g["trace_vm"])) < 1e-9


@pytest.mark.parametrize("name,inner", [("ieee118_k6_inner2", 2), ("rand120_k4_inner3", 3)])
def test_inner_gn_steps_match_reference(name, inner):
    # SolverConfig.inner_gn_steps > 1 (reference solver.py:253-260)
    net, ms, part, g = build_case(name)
    res = Oracle(net, ms, part.area_of_bus).solve(trace=True, inner=inner)
    assert res["iterations"] == int(g["iterations"]) and res["converged"] == bool(g["converged"])
    assert np.allclose(res["deltas"], g["deltas"], rtol=1e-6, atol=1e-12)
    assert np.max(np.abs(res["trace_va"] - g["trace_va"])) < 1e-9
    assert np.max(np.abs(res["trace_vm"] - g["trace_vm"])) < 1e-9
    assert abs(res["objective"] - float(g["objective"])) <= 1e-10 * float(g["objective"])


def test_reference_hand_values_dense_solve():
    # reference tests/test_linalg.py:42-50: [[4,2],[2,3]] x = [2,1] -> [0.5, 0]; pivot 1 of [[1,2],[2,1]]
    x = dense_cholesky_solve(np.array([[4.0, 2.0], [2.0, 3.0]]), np.array([2.0, 1.0]))
    assert np.allclose(x, [0.5, 0.0], atol=1e-15)
    with pytest.raises(OracleError) as exc:
        dense_cholesky_solve(np.array([[1.0, 2.0], [2.0, 1.0]]), np.array([1.0, 1.0]))
    assert exc.value.pivot == 1


def test_unobservable_area_reports_area():
    # reference tests/test_solver.py:335-342: mask everything an area owns
    import paper_2604_23175_b200 as G
    net, ms, part, _ = build_case("ieee14_k2")
    owned = part.area_of_bus[ms.owner_bus] == 1
    ms2 = G.apply_mask(ms, owned)
    with pytest.raises(OracleError) as exc:
        Oracle(net, ms2, part.area_of_bus).solve()
    assert exc.value.kind == 1 and exc.value.area == 1


@pytest.mark.parametrize("name", ["ieee14_centralized_refined", "ieee118_centralized_refined"])
def test_refined_centralized_fixture_is_the_plain_solve_to_rounding(name):
    # reference solve_centralized(iterative_refinement=True) (solver.py:181-183): one residual correction per
    # solve only polishes the iterate, so the oracle's plain k = 1 solve pins the fixture to 1e-9
    net, ms, part, g = build_case(name)
    assert part.k == 1 and int(g["n_gamma"]) == 0
    res = Oracle(net, ms, part.area_of_bus).solve(trace=True)
    assert res["iterations"] == int(g["iterations"]) and res["converged"] == bool(g["converged"])
    assert np.max(np.abs(res["trace_va"] - g["trace_va"])) < 1e-9
    assert np.max(np.abs(res["trace_vm"] - g["trace_vm"])) < 1e-9
    assert abs(res["objective"] - float(g["objective"])) <= 1e-10 * float(g["objective"])
