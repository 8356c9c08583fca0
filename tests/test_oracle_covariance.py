"""Pin the CPU oracle's masked 2-D operator to proj/tests/test_covariance.cpp
(and acceptance.cpp criteria 6 and 9). The same cases run against the GPU
in test_gpu_covariance.py."""
import math

import numpy as np
import pytest

import oracle as O
from helpers import assemble_dense, checkered_mask, halfwidth, uniform_grid


def make(g, r=12000.0, order=3, k=1, unit_dc=True, ghost=None, variance=None, threads=1,
         rx=None, ry=None, grid_ghost=0):
    rx = np.full((g["ny"], g["nx"]), r) if rx is None else rx
    ry = np.full((g["ny"], g["nx"]), r) if ry is None else ry
    return O.OracleOp(g["nx"], g["ny"], g["dx"], g["dy"], g["mask"], rx, ry, order=order,
                      k_iterations=k, unit_dc=unit_dc, ghost_width=ghost, variance=variance,
                      threads=threads, grid_ghost_width=grid_ghost)


def test_all_sea_row_is_1d():  # test_covariance.cpp:45-63
    g = uniform_grid(300, 4)
    op = make(g, unit_dc=False)
    f = np.zeros((4, 300))
    f[2, 150] = 1.0
    out = op.apply(O.GX, f)
    d = np.zeros(300)
    d[150] = 1.0
    want = O.rf3_apply_1d(d, 2.0)
    assert np.all(np.abs(out[2] - want) <= 1e-14 * (1 + np.abs(want)))
    assert np.linalg.norm(out[0]) == 0.0


def test_land_splits_segments():  # test_covariance.cpp:65-79
    g = uniform_grid(21, 4)
    g["mask"][:, :, 10] = False
    for order in (1, 3):
        op = make(g, order=order, k=5 if order == 1 else 1, unit_dc=False)
        f = np.zeros((4, 21))
        f[1, 4] = 1.0
        out = op.apply(O.GX, f)
        assert out[1, 10] == 0.0
        assert np.all(out[1, 11:] == 0.0)
        assert out[1, 4] > 0.0


def test_short_segments_pass_through():  # test_covariance.cpp:81-96
    g = uniform_grid(5, 4)
    g["mask"][:, :, 2] = False
    op = make(g, unit_dc=False, ghost=0)
    f = np.zeros((4, 5))
    f[1, 0], f[1, 1], f[1, 3] = 2.0, -1.0, 0.5
    out = op.apply(O.GX, f)
    assert (out[1, 0], out[1, 1], out[1, 2], out[1, 3]) == (2.0, -1.0, 0.0, 0.5)


def test_ghost_effect_near_coast():  # test_covariance.cpp:98-118
    g = uniform_grid(40, 4)
    g["mask"][:, :, 30:] = False
    f = np.zeros((4, 40))
    f[1, 27] = 1.0
    r0 = make(g, unit_dc=False, ghost=0).apply(O.GX, f)
    r9 = make(g, unit_dc=False, ghost=18).apply(O.GX, f)
    peak = r9[1].max()
    assert abs(r9[1, 29] - r0[1, 29]) / peak > 1e-4
    for i in range(0, 29 - 12 + 1):
        assert abs(r9[1, i] - r0[1, i]) / peak < 1e-3


def test_land_barrier_blocks_b():  # test_covariance.cpp:120-132
    g = uniform_grid(40, 24)
    g["mask"][:, :, 20] = False
    f = np.zeros((24, 40))
    f[12, 8] = 1.0
    b = make(g).apply(O.B, f)
    assert np.all(b[:, 20:] == 0.0)
    assert b[12, 8] > 0.0


def test_separability():  # test_covariance.cpp:134-154
    g = uniform_grid(64, 64)
    op = make(g, unit_dc=False)
    assert np.linalg.norm(op.apply(O.GY, np.zeros((64, 64)))) == 0.0
    f = np.zeros((64, 64))
    f[32, 32] = 1.0
    out = op.apply(O.GYGX, f)
    d = np.zeros(64)
    d[32] = 1.0
    h = O.rf3_apply_1d(d, 2.0)
    want = np.outer(h, h)
    assert np.all(np.abs(out - want) < 1e-10 * (1 + np.abs(want)))


def test_anisotropy(golden):  # test_covariance.cpp:156-176, acceptance criterion 9
    g = uniform_grid(201, 121, 25000.0, 25000.0)
    op = make(g, unit_dc=False, rx=np.full((121, 201), 350000.0), ry=np.full((121, 201), 100000.0))
    f = np.zeros((121, 201))
    f[60, 100] = 1.0
    out = op.apply(O.GYGX, f)
    ratio = halfwidth(out[60, :], 100) / halfwidth(out[:, 100], 60)
    assert abs(ratio - 3.5) <= 0.05 * 3.5
    # the reference's own measured ratio (test_output.txt:17), 6 digits
    assert abs(ratio - golden["acceptance"]["criterion9_ratio"]) <= 5e-6 * ratio


def test_masked_dot_product():  # test_covariance.cpp:178-197
    g = uniform_grid(20, 20)
    g["mask"] = checkered_mask(20, 20, 99, 0.8)
    rng = np.random.default_rng(31)
    for order in (1, 3):
        op = make(g, order=order, k=5 if order == 1 else 1)
        for _ in range(25):
            u, v = rng.standard_normal((20, 20)), rng.standard_normal((20, 20))
            lhs = np.sum(v * op.apply(O.V, u))
            rhs = np.sum(op.apply(O.VT, v) * u)
            assert abs(lhs - rhs) <= 1e-10 * np.linalg.norm(u) * np.linalg.norm(v)


def test_dense_12x12_transpose_symmetry_psd():  # test_covariance.cpp:199-218
    g = uniform_grid(12, 12)
    g["mask"] = checkered_mask(12, 12, 7, 0.85)
    op = make(g)
    V = assemble_dense(12, 12, lambda e: op.apply(O.V, e))
    Vt = assemble_dense(12, 12, lambda e: op.apply(O.VT, e))
    assert np.abs(Vt - V.T).max() < 1e-12
    B = assemble_dense(12, 12, lambda e: op.apply(O.B, e))
    assert np.abs(B - B.T).max() < 1e-12
    assert np.linalg.eigvalsh(0.5 * (B + B.T)).min() >= -1e-10


def test_b_psd_random():  # test_covariance.cpp:220-231
    g = uniform_grid(16, 16)
    g["mask"] = checkered_mask(16, 16, 3, 0.9)
    op = make(g)
    rng = np.random.default_rng(17)
    for _ in range(100):
        u = rng.standard_normal((16, 16))
        assert np.sum(u * op.apply(O.B, u)) >= -1e-10 * np.sum(u * u)


def test_b_dirac_width_and_locality():  # test_covariance.cpp:233-279
    g = uniform_grid(129, 129)
    op = make(g)
    f = np.zeros((129, 129))
    f[64, 64] = 1.0
    b = op.apply(O.B, f)
    jmax, imax = np.unravel_index(np.argmax(b), b.shape)
    assert (imax, jmax) == (64, 64)
    scale_x = halfwidth(b[64, :], 64) / math.sqrt(2 * math.log(2))
    assert abs(scale_x - math.sqrt(2) * 2) <= 0.05 * math.sqrt(2) * 2
    jj, ii = np.mgrid[0:129, 0:129]
    d2 = (ii - 64) ** 2 + (jj - 64) ** 2
    peak = b[64, 64]
    assert np.abs(b[d2 > (6 * math.sqrt(2) * 2) ** 2]).max() / peak < 3e-4
    assert np.abs(b[d2 > (8 * math.sqrt(2) * 2) ** 2]).max() / peak < 1e-4


def test_zero_variance():  # test_covariance.cpp:281-291
    g = uniform_grid(16, 16)
    op = make(g, variance=np.zeros((16, 16)))
    u = np.random.default_rng(41).standard_normal((16, 16))
    assert np.linalg.norm(op.apply(O.V, u)) == 0.0
    assert np.linalg.norm(op.apply(O.VT, u)) == 0.0


def test_self_adjoint_interior():  # test_covariance.cpp:293-306
    g = uniform_grid(120, 120)
    op = make(g)
    u = np.zeros((120, 120))
    u[40:80, 40:80] = np.random.default_rng(53).standard_normal((40, 40))
    vu, vtu = op.apply(O.V, u), op.apply(O.VT, u)
    assert np.linalg.norm(vu - vtu) / np.linalg.norm(vu) < 1e-6


def test_land_exactly_zero_with_junk_input():  # test_covariance.cpp:308-327
    g = uniform_grid(24, 24)
    g["mask"] = checkered_mask(24, 24, 121, 0.7)
    rng = np.random.default_rng(61)
    land = ~g["mask"][0]
    for order in (1, 3):
        op = make(g, order=order, k=3 if order == 1 else 1)
        u = rng.standard_normal((24, 24))
        for kind in (O.GX, O.GY, O.V, O.VT, O.B):
            assert np.all(op.apply(kind, u)[land] == 0.0)


def test_coefficient_bytes():  # test_covariance.cpp:339-346
    g = uniform_grid(32, 20)
    op1, op3 = make(g, order=1, k=5), make(g)
    assert op3.coefficient_bytes() == 2 * op1.coefficient_bytes()
    assert op1.coefficient_bytes() == 2 * 2 * 8 * 32 * 20


def test_ghost_resolution():  # test_covariance.cpp:348-359
    g = uniform_grid(16, 16)
    assert make(g).ghost_width() == 18
    assert make(g, grid_ghost=7).ghost_width() == 7
    assert make(g, grid_ghost=7, ghost=0).ghost_width() == 0
    assert make(g, ghost=3).ghost_width() == 3


def test_thread_count_invariance():  # test_covariance.cpp:361-374
    g = uniform_grid(48, 40)
    g["mask"] = checkered_mask(48, 40, 5, 0.85)
    u = np.random.default_rng(71).standard_normal((40, 48))
    a = make(g, threads=1).apply(O.B, u)
    b = make(g, threads=4).apply(O.B, u)
    assert np.array_equal(a, b)


def test_third_order_rejects_k():  # test_covariance.cpp:376-381
    g = uniform_grid(8, 8)
    with pytest.raises(O.OracleError, match="single-iteration by construction"):
        make(g, k=2)


def test_acceptance_criterion6_adjoint():  # acceptance.cpp:155-192 (defaults)
    g = uniform_grid(20, 20)
    g["mask"] = checkered_mask(20, 20, 99, 0.8)
    op = make(g)
    rng = np.random.default_rng(31)
    worst = 0.0
    for _ in range(50):
        u, v = rng.standard_normal((20, 20)), rng.standard_normal((20, 20))
        lhs = np.sum(v * op.apply(O.V, u))
        rhs = np.sum(op.apply(O.VT, v) * u)
        worst = max(worst, abs(lhs - rhs) / (np.linalg.norm(u) * np.linalg.norm(v)))
    assert worst <= 1e-10


def test_levels_are_independent_2d_ops():  # loop of 2-D operators
    nx, ny, nlev = 30, 20, 3
    g = uniform_grid(nx, ny, nlev=nlev)
    g["mask"] = checkered_mask(nx, ny, 11, 0.8, nlev=nlev)
    rng = np.random.default_rng(3)
    rx = 12000.0 * rng.uniform(0.8, 2.0, (ny, nx))
    ry = 12000.0 * rng.uniform(0.8, 2.0, (ny, nx))
    op3 = make(g, rx=rx, ry=ry)
    f = rng.standard_normal((2, nlev, ny, nx))
    out = op3.apply(O.V, f)
    for lev in range(nlev):
        g1 = dict(g, mask=g["mask"][lev:lev + 1])
        op1 = make(g1, rx=rx, ry=ry)
        assert op1.ghost_width() == op3.ghost_width(lev)
        for v in range(2):
            assert np.array_equal(op1.apply(O.V, f[v, lev]), out[v, lev])
