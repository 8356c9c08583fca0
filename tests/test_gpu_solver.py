"""Device observation operator and CG analysis
against the oracle restatement of obs.cpp / solver.cpp: H and H^T
bit-identical, cost and solve within tolerance (only the dot-product
summation order differs), and the reference's own solver tests
(proj/tests/test_solver.cpp) on the device path."""
import numpy as np
import pytest

import oracle as O
from helpers import relmax

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1404_5756_b200 as P
    return P


def pair(P, nx, ny, d, r, mask=None, order=3, k=1, rx=None):
    one = np.ones((ny, nx))
    m = np.ones((ny, nx), bool) if mask is None else mask
    rxa = one * r if rx is None else rx
    grid = P.Grid2D(nx, ny, one * d, one * d, m)
    gpu = P.HorizontalCovarianceOp(grid, P.ScaleField(rxa, rxa),
                                   P.CovarianceOptions(order=P.FilterOrder(order), k_iterations=k))
    cpu = O.OracleOp(nx, ny, one * d, one * d, m, rxa, rxa, order=order, k_iterations=k, threads=4)
    return gpu, cpu


def obs_pair(P, cpu, rows):
    rows = np.asarray(rows, dtype=np.float64).reshape(-1, 4)
    return P.ObsSet(rows[:, :2], rows[:, 2], rows[:, 3]), O.OracleObs(cpu, rows[:, :2], rows[:, 2],
                                                                         rows[:, 3])


def random_rows(rng, n, nx, ny):
    return np.column_stack([rng.uniform(0, nx - 1, n), rng.uniform(0, ny - 1, n),
                            rng.standard_normal(n), rng.uniform(0.3, 2.0, n)])


def test_h_and_ht_bit_identical(P):
    rng = np.random.default_rng(5)
    m = rng.uniform(size=(37, 53)) > 0.2
    gpu, cpu = pair(P, 53, 37, 5000.0, 15000.0, mask=m)
    rows = random_rows(rng, 400, 53, 37)
    rows[:50, :2] = np.floor(rows[:50, :2])  # node hits, repeated cells
    rows[50:60, :2] = rows[60:70, :2]
    keep = [r for r in rows if _has_sea(m, r[0], r[1])]
    go, co = obs_pair(P, cpu, keep)
    f = rng.standard_normal((37, 53))
    v = rng.standard_normal(len(keep))
    assert np.array_equal(P.obs_operator(f, go, gpu), co.h(f))
    assert np.array_equal(P.obs_operator_transpose(v, go, gpu), co.ht(v))


def _has_sea(m, x, y):
    ny, nx = m.shape
    i0 = min(int(np.floor(x)), nx - 2)
    j0 = min(int(np.floor(y)), ny - 2)
    return m[j0, i0] or m[j0, i0 + 1] or m[j0 + 1, i0] or m[j0 + 1, i0 + 1]


def test_obs_errors_match_reference(P):
    m = np.ones((8, 8), bool)
    m[3:5, 3:5] = False
    gpu, _ = pair(P, 8, 8, 1000.0, 2000.0, mask=m)
    f = np.zeros((8, 8))
    with pytest.raises(P.InvalidArgument, match="observation 0: all four stencil corners are land"):
        P.obs_operator(f, P.ObsSet(np.array([[3.5, 3.5]]), [0.0], [1.0]), gpu)
    with pytest.raises(P.InvalidArgument, match="observation 0: position .* is outside the grid"):
        P.obs_operator(f, P.ObsSet(np.array([[-0.5, 2.0]]), [0.0], [1.0]), gpu)
    with pytest.raises(P.InvalidArgument, match="observation 1: error variance must be positive"):
        P.solve(P.ObsSet(np.array([[2.0, 2.0], [5.0, 5.0]]), [1.0, 1.0], [1.0, 0.0]), gpu)
    with pytest.raises(P.InvalidArgument, match="solve: tol must be positive"):
        P.solve(P.ObsSet(np.array([[2.0, 2.0]]), [1.0], [1.0]), gpu, P.SolveOptions(tol=0.0))


@pytest.mark.parametrize("bg", [False, True])
def test_cost_matches_oracle(P, bg):
    rng = np.random.default_rng(7)
    m = rng.uniform(size=(30, 41)) > 0.25
    rx = 6000.0 * rng.uniform(1.5, 4.0, (30, 41))
    gpu, cpu = pair(P, 41, 30, 6000.0, 0.0, mask=m, rx=rx)
    rows = [r for r in random_rows(rng, 60, 41, 30) if _has_sea(m, r[0], r[1])]
    go, co = obs_pair(P, cpu, rows)
    chi = rng.standard_normal((30, 41))
    b = rng.standard_normal((30, 41)) if bg else None
    got = P.cost(chi, go, gpu, background=b)
    want = co.cost(chi, background=b)
    assert got.j_total == pytest.approx(want["j_total"], rel=1e-12)
    assert got.j_background == pytest.approx(want["j_background"], rel=1e-12)
    assert got.j_obs == pytest.approx(want["j_obs"], rel=1e-12)
    assert relmax(got.gradient, want["gradient"]) <= 1e-12


@pytest.mark.parametrize("order,k", [(3, 1), (1, 5)])
def test_solve_matches_oracle(P, order, k):
    rng = np.random.default_rng(11 + order)
    m = rng.uniform(size=(48, 64)) > 0.2
    rx = 6000.0 * rng.uniform(1.5, 4.0, (48, 64))
    gpu, cpu = pair(P, 64, 48, 6000.0, 0.0, mask=m, order=order, k=k, rx=rx)
    rows = [r for r in random_rows(rng, 80, 64, 48) if _has_sea(m, r[0], r[1])]
    go, co = obs_pair(P, cpu, rows)
    bg = rng.standard_normal((48, 64)) * 0.1
    got = P.solve(go, gpu, P.SolveOptions(tol=1e-10, max_iter=60), background=bg)
    want = co.solve(tol=1e-10, max_iter=60, background=bg)
    assert got.converged == want["converged"]
    assert abs(got.cg_iterations - want["cg_iterations"]) <= 1
    assert np.array_equal(got.misfit, want["misfit"])  # H is bit-identical
    assert relmax(got.increment, want["increment"]) <= 1e-8
    assert got.j_obs == pytest.approx(want["j_obs"], rel=1e-8)
    assert got.j_background == pytest.approx(want["j_background"], rel=1e-8)
    n = min(len(got.gradient_norms), len(want["gradient_norms"]))
    assert np.allclose(got.gradient_norms[:n], want["gradient_norms"][:n], rtol=1e-6, atol=0)


def test_reference_solver_cases_on_device(P):
    """test_solver.cpp:139-250 on the device path."""
    gpu, _ = pair(P, 12, 12, 6000.0, 12000.0)
    an = P.solve(P.ObsSet(np.zeros((0, 2)), np.zeros(0), np.zeros(0)), gpu)
    assert an.converged and an.cg_iterations == 0 and not an.increment.any()
    an = P.solve(P.ObsSet(np.array([[6.0, 6.0]]), [0.0], [1.0]), gpu)
    assert an.cg_iterations == 0 and not an.increment.any()

    gpu, _ = pair(P, 64, 64, 6000.0, 12000.0)  # sigma = 2
    an = P.solve(P.ObsSet(np.array([[32.0, 32.0]]), [1.0], [1.0]), gpu,
                 P.SolveOptions(tol=1e-10, max_iter=50))
    assert an.converged
    inc = an.increment
    assert np.unravel_index(np.argmax(inc), inc.shape) == (32, 32)
    peak = inc[32, 32]
    assert 0.0 < peak < 1.0
    sb = np.sqrt(2.0) * 2.0
    sec = inc[32, :] / peak
    gauss = np.exp(-((np.arange(64) - 32.0) ** 2) / (2 * sb * sb))
    assert sec @ gauss / (np.linalg.norm(sec) * np.linalg.norm(gauss)) > 0.99

    gpu, _ = pair(P, 24, 24, 6000.0, 12000.0)
    an = P.solve(P.ObsSet(np.array([[5.0, 5.0], [12.0, 12.0], [18.0, 6.0]]), [1.0, -1.0, 2.0],
                          [0.1, 0.1, 0.1]), gpu, P.SolveOptions(tol=1e-15, max_iter=1))
    assert not an.converged and an.cg_iterations == 1 and len(an.gradient_norms) == 2
    assert np.linalg.norm(an.increment) > 0.0
