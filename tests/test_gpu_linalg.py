"""Standalone linear algebra on the device (matrix plans, gse_matrix_*): the reference's own linalg /
boundary tests with the device functions swapped in (reference tests/test_linalg.py,
tests/test_solver.py:207-264, tests/test_acceptance.py:130-157).  Needs a B200: ``pytest -m gpu``."""

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import paper_2604_23175_b200 as G
    return G


def _spd_sparse(n, seed, density=0.03):
    rng = np.random.default_rng(seed)
    a = sp.random(n, n, density=density, random_state=np.random.RandomState(seed), format="csr")
    a = a + a.T + sp.eye(n) * (1.0 + abs(a).sum(axis=1).max())
    a = sp.csr_matrix(a)
    a.sort_indices()
    return a, rng


def test_dense_hand_values(G):
    # reference test_linalg.py:42-50
    x = G.dense_cholesky_solve(np.array([[4.0, 2.0], [2.0, 3.0]]), np.array([2.0, 1.0]))
    assert np.allclose(x, [0.5, 0.0], atol=1e-14)
    with pytest.raises(G.NotPositiveDefiniteError) as exc:
        G.dense_cholesky_solve(np.array([[1.0, 2.0], [2.0, 1.0]]), np.array([1.0, 1.0]))
    assert exc.value.pivot == 1
    assert "not positive definite at pivot 1" in str(exc.value)


@pytest.mark.parametrize("n", [1, 7, 64, 130, 300])
def test_dense_solve_random(G, n):
    rng = np.random.default_rng(n)
    m = rng.standard_normal((n, n))
    a = m @ m.T + n * np.eye(n)
    b = rng.standard_normal(n)
    x = G.dense_cholesky_solve(a, b)
    assert np.max(np.abs(x - np.linalg.solve(a, b))) < 1e-9 * (1 + np.max(np.abs(x)))


@pytest.mark.parametrize("n,seed", [(20, 0), (64, 1), (200, 2), (700, 3)])
def test_refactor_and_solve_vs_numpy(G, n, seed):
    # reference test_linalg.py:102-135: same structure over repeated refactors, solves to 1e-9
    a, rng = _spd_sparse(n, seed)
    cache = G.symbolic_analyze(a)
    for rep in range(3):
        vals = a.data * (1.0 + 0.1 * rep)
        G.numeric_refactor(cache, vals)
        b = rng.standard_normal(n)
        x = cache.solve(b)
        ref = np.linalg.solve((a * (1.0 + 0.1 * rep)).toarray(), b)
        assert np.max(np.abs(x - ref)) < 1e-9 * (1 + np.max(np.abs(ref)))
    # CSR input with the same pattern, and multi-RHS
    G.numeric_refactor(cache, a)
    B = rng.standard_normal((n, 3))
    assert np.max(np.abs(cache.solve(B) - np.linalg.solve(a.toarray(), B))) < 1e-9
    cache.close()


def test_not_positive_definite_reports_original_index(G):
    a, _ = _spd_sparse(120, 5)
    bad = a.tolil()
    bad[37, 37] = -1.0
    cache = G.symbolic_analyze(a, context="area 3 interior block")
    with pytest.raises(G.NotPositiveDefiniteError) as exc:
        G.numeric_refactor(cache, sp.csr_matrix(bad))
    assert "area 3 interior block" in str(exc.value)
    assert 0 <= exc.value.pivot < 120
    cache.close()


def test_schur_hand_example(G):
    # reference test_linalg.py:181-191: S=2.5, b_hat=3.0, dx_b=1.2, dx_i=1.4
    g_ii = sp.csr_matrix(np.array([[2.0]]))
    g_ib = sp.csr_matrix(np.array([[1.0]]))
    cache = G.symbolic_analyze(g_ii)
    G.numeric_refactor(cache, g_ii.data)
    res = G.schur_condense(cache, g_ib, np.array([[3.0]]), np.array([4.0]), np.array([5.0]))
    assert np.allclose(res.s_b, [[2.5]]) and np.allclose(res.b_hat, [3.0])
    dxb = res.b_hat / res.s_b[0, 0]
    assert np.allclose(dxb, [1.2])
    assert np.allclose(G.interior_recover(cache, g_ib, np.array([4.0]), dxb), [1.4])


@pytest.mark.parametrize("seed", range(6))
def test_condense_and_recover_equal_monolithic_solve(G, seed):
    # reference test_linalg.py:205-219 / test_acceptance.py:130-157 (criterion 3)
    rng = np.random.default_rng(100 + seed)
    n_i, n_b = int(rng.integers(30, 260)), int(rng.integers(1, 40))
    n = n_i + n_b
    full, _ = _spd_sparse(n, 200 + seed, density=0.05)
    g_ii, g_ib, g_bb = sp.csr_matrix(full[:n_i, :n_i]), sp.csr_matrix(full[:n_i, n_i:]), full[n_i:, n_i:].toarray()
    b = rng.standard_normal(n)
    cache = G.symbolic_analyze(g_ii)
    G.numeric_refactor(cache, g_ii)
    res = G.schur_condense(cache, g_ib, g_bb, b[:n_i], b[n_i:])
    s_ref = g_bb - g_ib.T.toarray() @ np.linalg.solve(g_ii.toarray(), g_ib.toarray())
    assert np.max(np.abs(res.s_b - s_ref)) < 1e-9 * (1 + np.max(np.abs(s_ref)))
    assert np.max(np.abs(res.s_b - res.s_b.T)) < 1e-12 * (1 + np.max(np.abs(s_ref)))
    dxb = G.dense_cholesky_solve(res.s_b, res.b_hat)
    dxi = G.interior_recover(cache, g_ib, b[:n_i], dxb)
    x = np.linalg.solve(full.toarray(), b)
    assert np.max(np.abs(np.concatenate([dxi, dxb]) - x)) < 1e-9 * (1 + np.max(np.abs(x)))
    cache.close()


def test_empty_interior_and_empty_boundary(G):
    # reference test_linalg.py:239-245
    cache = G.symbolic_analyze(sp.csr_matrix((0, 0)))
    res = G.schur_condense(cache, sp.csr_matrix((0, 2)), np.eye(2), np.zeros(0), np.array([1.0, 2.0]))
    assert np.allclose(res.s_b, np.eye(2)) and np.allclose(res.b_hat, [1.0, 2.0])
    assert G.interior_recover(cache, sp.csr_matrix((0, 2)), np.zeros(0), np.array([1.0, 2.0])).size == 0
    a, rng = _spd_sparse(40, 9)
    cache = G.symbolic_analyze(a)
    G.numeric_refactor(cache, a)
    res = G.schur_condense(cache, sp.csr_matrix((40, 0)), np.zeros((0, 0)), rng.standard_normal(40), np.zeros(0))
    assert res.s_b.shape == (0, 0) and res.b_hat.shape == (0,)


def test_assemble_boundary_additivity_and_order(G):
    # reference test_solver.py:207-214: overlapping selectors add, 2.5 + 1.5 = 4.0
    r1 = G.SchurResult(s_b=np.array([[2.5, 0.5], [0.5, 1.0]]), b_hat=np.array([1.0, 2.0]))
    r2 = G.SchurResult(s_b=np.array([[1.5]]), b_hat=np.array([0.25]))
    bs = G.assemble_boundary([r1, r2], [np.array([0, 2]), np.array([0])], 3)
    assert bs.s_gamma[0, 0] == 4.0 and bs.s_gamma[0, 2] == 0.5 and bs.s_gamma[2, 0] == 0.5 and bs.s_gamma[2, 2] == 1.0
    assert np.all(bs.s_gamma[1] == 0.0) and np.allclose(bs.b_gamma, [1.25, 0.0, 2.0])


def test_component_pipeline_reproduces_solver_boundary_system(G):
    """fused_accumulate -> numeric_refactor -> schur_condense -> assemble_boundary -> dense_cholesky_solve
    on IEEE-118 / 6 areas equals the reference's stored boundary system (golden fixture)."""
    from conftest import build_case
    net, ms, part, g = build_case("ieee118_k6")
    bord, maps = G.build_variable_maps(net, part)
    st = G.StateVector.flat_start(net)
    xg = bord.gather(st.va, st.vm)
    schurs = []
    for m in maps:
        blk = G.fused_accumulate(m, ms, m.gather_interior(st.va, st.vm), xg[m.boundary_selector])
        cache = G.symbolic_analyze(blk.g_ii)
        G.numeric_refactor(cache, blk.g_ii.data)
        schurs.append(G.schur_condense(cache, blk.g_ib, blk.g_bb, blk.b_i, blk.b_b))
        cache.close()
    bs = G.assemble_boundary(schurs, [m.boundary_selector for m in maps], bord.n_gamma)
    scale = 1 + np.abs(g["s_gamma"])
    assert np.max(np.abs(bs.s_gamma - g["s_gamma"]) / scale) < 1e-9
    assert np.max(np.abs(bs.b_gamma - g["b_gamma"]) / (1 + np.abs(g["b_gamma"]))) < 1e-9
    dx = G.dense_cholesky_solve(bs.s_gamma, bs.b_gamma)
    assert np.max(np.abs(dx - g["dx_gamma"])) < 1e-9


@pytest.mark.parametrize("n,seed", [(12, 0), (64, 1), (300, 2)])
def test_forward_backward_in_factor_coordinates(G, n, seed):
    """SparseCholeskyCache.forward / .backward (reference linalg.py:340-383): y = L^-1 P b lives in this factor's
    coordinates (cache.perm), so the checks are the ordering-independent ones -- backward(forward(b)) is the solve
    (bit for bit: the same device sequence), y.y = b.G^-1.b, y equals the triangular solve of the permuted matrix's
    Cholesky factor, and matrix right-hand sides go column by column (reference test_linalg.py:137-160)."""
    import scipy.linalg as sla
    a, rng = _spd_sparse(n, seed)
    cache = G.symbolic_analyze(a)
    G.numeric_refactor(cache, a.data)
    b = rng.standard_normal(n)
    perm = np.asarray(cache.perm)
    assert sorted(perm.tolist()) == list(range(n))
    y = cache.forward(b)
    x = cache.backward(y)
    assert np.array_equal(x, cache.solve(b))
    dense = a.toarray()
    assert abs(y @ y - b @ np.linalg.solve(dense, b)) <= 1e-11 * abs(y @ y)
    lfac = np.linalg.cholesky(dense[np.ix_(perm, perm)])
    assert np.max(np.abs(y - sla.solve_triangular(lfac, b[perm], lower=True))) < 1e-10 * (1 + np.max(np.abs(y)))
    assert np.max(np.abs(x - np.linalg.solve(dense, b))) < 1e-9 * (1 + np.max(np.abs(x)))
    bm = rng.standard_normal((n, 3))
    ym = cache.forward(bm)
    assert ym.shape == (n, 3) and np.array_equal(ym[:, 0], cache.forward(bm[:, 0]))
    assert np.array_equal(cache.backward(ym)[:, 2], cache.solve(bm[:, 2]))
    fresh = G.symbolic_analyze(a)
    with pytest.raises(RuntimeError, match="numeric factorization has not been run"):
        fresh.forward(b)
    cache.close(); fresh.close()
