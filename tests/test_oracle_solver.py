"""Oracle restatement of the reference's observation operator and CG analysis
(obs.cpp, solver.cpp), pinned to the reference's own tests
(proj/tests/test_solver.cpp:45-284). CPU only."""
import numpy as np
import pytest

import oracle as O


def uniform_op(nx, ny, d, r, mask=None, order=3, k=1):
    one = np.ones((ny, nx))
    m = np.ones((ny, nx), bool) if mask is None else mask
    return O.OracleOp(nx, ny, one * d, one * d, m, one * r, one * r, order=order, k_iterations=k,
                      threads=1)


def obs(op, rows):
    rows = np.asarray(rows, dtype=np.float64).reshape(-1, 4)
    return O.OracleObs(op, rows[:, :2], rows[:, 2], rows[:, 3])


def test_obs_operator_exact_on_affine_fields():  # test_solver.cpp:45-58
    op = uniform_op(8, 8, 1000.0, 2000.0)
    f = np.fromfunction(lambda j, i: 2.0 * i - 3.0 * j + 1.0, (8, 8))
    h = obs(op, [[3.5, 2.0, 0, 1], [5.0, 5.0, 0, 1], [0.25, 6.75, 0, 1]]).h(f)
    assert h[0] == pytest.approx(2.0 * 3.5 - 3.0 * 2.0 + 1.0, rel=1e-14)
    assert h[1] == f[5, 5]  # node hit is exact
    assert h[2] == pytest.approx(2.0 * 0.25 - 3.0 * 6.75 + 1.0, rel=1e-13)


def test_obs_operator_rejects():  # test_solver.cpp:60-74
    m = np.ones((8, 8), bool)
    m[3:5, 3:5] = False
    op = uniform_op(8, 8, 1000.0, 2000.0, mask=m)
    with pytest.raises(O.OracleError, match="land"):
        obs(op, [[3.5, 3.5, 0, 1]])
    with pytest.raises(O.OracleError, match="observation 0"):
        obs(op, [[-0.5, 2.0, 0, 1]])
    m[4, 4] = True
    obs(uniform_op(8, 8, 1000.0, 2000.0, mask=m), [[3.5, 3.5, 0, 1]])


def test_obs_adjoint_dot_identity():  # test_solver.cpp:76-88
    op = uniform_op(10, 9, 1000.0, 2000.0)
    ob = obs(op, [[3.5, 2.0, 0, 1], [7.25, 6.5, 0, 1], [1.0, 1.0, 0, 1]])
    rng = np.random.default_rng(3)
    for _ in range(20):
        u = rng.standard_normal((9, 10))
        w = rng.standard_normal(3)
        assert ob.h(u) @ w == pytest.approx(np.sum(ob.ht(w) * u), rel=1e-12)


def test_cost_origin_and_fd_gradient():  # test_solver.cpp:104-137
    op = uniform_op(8, 8, 6000.0, 12000.0)
    rows = [[3.0, 4.0, 1.0, 0.5], [5.5, 2.5, -0.7, 2.0]]
    ob = obs(op, rows)
    r = ob.cost(np.zeros((8, 8)))
    vals = np.array([1.0, -0.7])
    rv = np.array([0.5, 2.0])
    assert r["j_total"] == pytest.approx(0.5 * np.sum(vals ** 2 / rv), rel=1e-14)
    assert r["j_background"] == 0.0
    assert obs(op, [[3.0, 4.0, 0.0, 0.5], [5.5, 2.5, 0.0, 2.0]]).cost(np.zeros((8, 8)))[
        "j_total"] == 0.0
    chi = np.random.default_rng(19).standard_normal((8, 8))
    g = ob.cost(chi)["gradient"]
    eps = 1e-6
    for i, j in ((2, 3), (0, 0), (7, 5)):
        cp, cm = chi.copy(), chi.copy()
        cp[j, i] += eps
        cm[j, i] -= eps
        fd = (ob.cost(cp)["j_total"] - ob.cost(cm)["j_total"]) / (2 * eps)
        assert g[j, i] == pytest.approx(fd, rel=1e-6)


def test_solve_trivial_cases():  # test_solver.cpp:139-163
    op = uniform_op(12, 12, 6000.0, 12000.0)
    an = obs(op, np.zeros((0, 4))).solve()
    assert an["converged"] and an["cg_iterations"] == 0 and not an["increment"].any()
    an = obs(op, [[6, 6, 0.0, 1.0]]).solve()
    assert an["cg_iterations"] == 0 and not an["increment"].any()
    with pytest.raises(O.OracleError, match="tol"):
        obs(op, [[6, 6, 1.0, 1.0]]).solve(tol=0.0)


def test_solve_single_observation():  # test_solver.cpp:165-192
    op = uniform_op(64, 64, 6000.0, 12000.0)  # sigma = 2
    an = obs(op, [[32, 32, 1.0, 1.0]]).solve(tol=1e-10, max_iter=50)
    assert an["converged"]
    inc = an["increment"]
    jmax, imax = np.unravel_index(np.argmax(inc), inc.shape)
    assert (imax, jmax) == (32, 32)
    peak = inc[32, 32]
    assert 0.0 < peak < 1.0
    sb = np.sqrt(2.0) * 2.0
    sec = inc[32, :] / peak
    gauss = np.exp(-((np.arange(64) - 32.0) ** 2) / (2 * sb * sb))
    assert sec @ gauss / (np.linalg.norm(sec) * np.linalg.norm(gauss)) > 0.99


def test_solve_error_variance_reduces_pull():  # test_solver.cpp:194-206
    op = uniform_op(48, 48, 6000.0, 12000.0)
    tight = obs(op, [[24, 24, 1.0, 1.0], [10, 10, 0.5, 1.0]]).solve(tol=1e-10, max_iter=50)
    loose = obs(op, [[24, 24, 1.0, 2.0], [10, 10, 0.5, 1.0]]).solve(tol=1e-10, max_iter=50)
    assert loose["increment"][24, 24] < tight["increment"][24, 24]


def test_solve_matches_dense_direct_solve():  # test_solver.cpp:208-237
    m = np.ones((12, 12), bool)
    m[4:7, 6] = False
    op = uniform_op(12, 12, 6000.0, 12000.0, mask=m)
    rows = [[3.5, 4.5, 1.0, 0.8], [8.0, 8.0, -0.5, 1.5], [2.0, 9.0, 0.25, 1.0]]
    ob = obs(op, rows)
    n = 144
    B = np.empty((n, n))
    for c in range(n):
        e = np.zeros(n)
        e[c] = 1.0
        B[:, c] = op.apply(6, e.reshape(1, 12, 12)).reshape(-1)
    H = np.stack([ob.ht(np.eye(3)[r]).reshape(-1) for r in range(3)])
    vals = np.array([r[2] for r in rows])
    rinv = np.diag(1.0 / np.array([r[3] for r in rows]))
    A = np.eye(n) + B @ H.T @ rinv @ H
    dense = np.linalg.solve(A, B @ H.T @ rinv @ vals)
    an = ob.solve(tol=1e-13, max_iter=200)
    assert an["converged"]
    cg = an["increment"].reshape(-1)
    assert np.linalg.norm(cg - dense) <= 1e-8 * np.linalg.norm(dense)


def test_solve_max_iter_flag():  # test_solver.cpp:239-250
    op = uniform_op(24, 24, 6000.0, 12000.0)
    an = obs(op, [[5, 5, 1.0, 0.1], [12, 12, -1.0, 0.1], [18, 6, 2.0, 0.1]]).solve(
        tol=1e-15, max_iter=1)
    assert not an["converged"] and an["cg_iterations"] == 1
    assert len(an["gradient_norms"]) == 2
    assert np.linalg.norm(an["increment"]) > 0.0


def test_solve_order_equivalence():  # test_solver.cpp:252-284
    rows = [[24, 24, 1.0, 1.0]]
    d3 = obs(uniform_op(48, 48, 6000.0, 12000.0), rows).solve(tol=1e-10, max_iter=50)
    d1 = obs(uniform_op(48, 48, 6000.0, 12000.0, order=1, k=1), rows).solve(tol=1e-10, max_iter=50)
    d10 = obs(uniform_op(48, 48, 6000.0, 12000.0, order=1, k=10), rows).solve(tol=1e-10,
                                                                              max_iter=50)
    a = d3["increment"]
    diff1 = np.linalg.norm(a - d1["increment"]) / np.linalg.norm(a)
    diff10 = np.linalg.norm(a - d10["increment"]) / np.linalg.norm(a)
    assert diff10 < diff1
