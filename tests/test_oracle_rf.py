"""Pin the CPU oracle's 1-D filter core to the reference's own KATs.

Restates proj/tests/test_rf3.cpp and proj/tests/test_rf1.cpp against the
oracle (oracle/librgf_oracle.so), including the kGolden table extracted
verbatim into tests/golden/reference_golden.json, and the captured
acceptance numbers of proj/test_output.txt (criteria 1-4).
"""
import math

import mpmath
import numpy as np
import pytest

import oracle as O

PI = math.pi


def rel(a, b):
    return abs(a - b) / abs(b)


def approx(a, b, eps):
    """doctest::Approx(b).epsilon(eps) == a  (scale 1: |a-b| < eps*(1+max|.|))."""
    return abs(a - b) < eps * (1.0 + max(abs(a), abs(b)))


# ---------------------------------------------------------------- rf3 coefficients
def test_rf3_golden_table(golden):  # test_rf3.cpp:49-61
    for g in golden["kGolden"]["rows"]:
        t = O.rf3_coefficients(g["sigma"])
        for i, k in enumerate(["a0", "a1", "a2", "a3", "alpha1", "alpha2", "alpha3", "beta"]):
            assert rel(t[i], g[k]) <= 1e-12, (g["sigma"], k, t[i], g[k])


def _poly_mp(x):  # oracles.hpp:65-82 restated in 40-digit arithmetic
    mpmath.mp.dps = 40
    x = mpmath.mpf(x)
    a0 = ((x + mpmath.mpf("3.382473")) * x + mpmath.mpf("5.788982")) * x + mpmath.mpf("3.738128")
    a1 = ((3 * x + mpmath.mpf("6.764946")) * x + mpmath.mpf("5.788982")) * x
    a2 = -(3 * x + mpmath.mpf("3.382473")) * x * x
    a3 = x ** 3
    al1, al2, al3 = a1 / a0, a2 / a0, a3 / a0
    beta = (2 * mpmath.pi * x * x) ** mpmath.mpf("0.25") * (1 - (al1 + al2 + al3))
    return [float(v) for v in (a0, a1, a2, a3, al1, al2, al3, beta)]


def test_rf3_high_precision_agreement():  # test_rf3.cpp:63-73
    sigma = 0.3
    while sigma < 24.0:
        t = O.rf3_coefficients(sigma)
        ld = _poly_mp(sigma)
        for i in (0, 1, 2, 4, 7):
            assert approx(t[i], ld[i], 1e-12), (sigma, i)
        sigma *= 1.37


def test_rf3_beta_identity_exact():  # test_rf3.cpp:77-88 (same C expression)
    for s in (0.5, 1.0, 2.0, 5.0, 10.0):
        t = O.rf3_coefficients(s)
        beta = math.pow(2.0 * PI * s * s, 0.25) * (1.0 - (t[4] + t[5] + t[6]))
        assert t[7] == beta
        f = O.rf3_filter_scalars(s)
        fb = math.pow(2.0 * PI * s * s, 0.25) * (1.0 - (f[0] + f[1] + f[2]))
        assert f[3] == fb


def test_rf3_invalid_sigma():  # test_rf3.cpp:90-94
    for s in (0.0, -2.0):
        with pytest.raises(O.OracleError, match="rf3_coefficients: sigma must be positive"):
            O.rf3_coefficients(s)
    with pytest.raises(O.OracleError, match="rf3_filter_scalars: sigma must be positive"):
        O.rf3_filter_scalars(0.0)


def test_rf3_calibration_monotone():  # test_rf3.cpp:96-107
    prev, s = 0.0, 0.3
    while s < 40.0:
        q = O.rf3_length_scale_argument(s, 0)
        assert q > 0 and q >= prev
        prev = q
        assert O.rf3_length_scale_argument(s, 2) == s
        s *= 1.21
    assert O.rf3_length_scale_argument(0.05, 0) == 0.01


def test_rf3_variance_match():  # test_rf3.cpp:109-116
    for s in (0.5, 2.0, 5.0, 14.0):
        q = O.rf3_length_scale_argument(s, 1)
        assert rel(O.rf3_cascade_variance(q), s * s) <= 1e-10


def test_rf3_cascade_variance_matches_kernel():  # test_rf3.cpp:118-135
    sigma, m = 3.0, 512
    q = O.rf3_length_scale_argument(sigma, 1)
    d = np.zeros(m)
    d[m // 2] = 1.0
    h = O.rf3_apply_1d(d, np.full(m, sigma), calibration=1)
    off = np.arange(m) - m // 2
    var = float(np.sum(h * off * off) / np.sum(h))
    assert rel(var, O.rf3_cascade_variance(q)) <= 1e-8
    assert rel(var, sigma * sigma) <= 1e-8


# ---------------------------------------------------------------- rf3 apply
def rf3_straight(s0, a1, a2, a3, b):  # oracles.hpp:54-61
    m = len(s0)
    p = np.zeros(m)
    s = np.zeros(m)
    p[0] = b * s0[0]
    p[1] = b * s0[1] + a1 * p[0]
    p[2] = b * s0[2] + a1 * p[1] + a2 * p[0]
    for i in range(3, m):
        p[i] = b * s0[i] + a1 * p[i - 1] + a2 * p[i - 2] + a3 * p[i - 3]
    s[m - 1] = b * p[m - 1]
    s[m - 2] = b * p[m - 2] + a1 * s[m - 1]
    s[m - 3] = b * p[m - 3] + a1 * s[m - 2] + a2 * s[m - 1]
    for i in range(m - 4, -1, -1):
        s[i] = b * p[i] + a1 * s[i + 1] + a2 * s[i + 2] + a3 * s[i + 3]
    return s


def test_rf3_matches_straight_line():  # test_rf3.cpp:146-155
    rng = np.random.default_rng(5)
    u = rng.standard_normal(64)
    c = O.rf3_filter_scalars(2.0)
    got = O.rf3_apply_1d(u, 2.0)
    want = rf3_straight(u, c[0], c[1], c[2], c[3])
    assert np.linalg.norm(got - want) <= 1e-14 * np.linalg.norm(want)


def test_rf3_zero_in_zero_out():  # test_rf3.cpp:157-160
    assert np.linalg.norm(O.rf3_apply_1d(np.zeros(32), 2.0)) == 0.0


def test_rf3_dc_gain():  # test_rf3.cpp:162-172 and acceptance criterion 3
    for sigma in (2.0, 5.0):
        m = int(16 * sigma) + 64
        out = O.rf3_apply_1d(np.ones(m), sigma)
        want = math.sqrt(2 * PI) * sigma
        assert rel(out[m // 2], want) <= 0.01


def test_rf3_impulse_sum_and_stability():  # test_rf3.cpp:174-193
    m = 300
    d = np.zeros(m)
    d[m // 2] = 1
    h = O.rf3_apply_1d(d, 2.0)
    assert rel(h.sum(), math.sqrt(2 * PI) * 2.0) <= 0.005
    for sigma in (0.5, 2.0, 10.0):
        m = int(4 * sigma) + 64
        d = np.zeros(m)
        d[m // 2] = 1
        h = O.rf3_apply_1d(d, sigma)
        assert np.abs(h).max() < 10 * (2 * PI * sigma * sigma) ** 0.25


def test_rf3_symmetry_shift_linearity():  # test_rf3.cpp:216-249
    m = 301
    d = np.zeros(m)
    d[m // 2] = 1
    h = O.rf3_apply_1d(d, 2.0)
    for dd in range(1, 17):
        assert abs(h[m // 2 + dd] - h[m // 2 - dd]) < 1e-10
    m = 200
    d1 = np.zeros(m)
    d2 = np.zeros(m)
    d1[m // 2] = 1
    d2[m // 2 + 1] = 1
    r1 = O.rf3_apply_1d(d1, 2.0)
    r2 = O.rf3_apply_1d(d2, 2.0)
    assert max(abs(r2[i + 1] - r1[i]) for i in range(16, m - 17)) < 1e-10
    rng = np.random.default_rng(13)
    u, v = rng.standard_normal(90), rng.standard_normal(90)
    lhs = O.rf3_apply_1d(1.9 * u + 0.4 * v, 3.0)
    rhs = 1.9 * O.rf3_apply_1d(u, 3.0) + 0.4 * O.rf3_apply_1d(v, 3.0)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)


def test_rf3_transpose_dot_varying():  # test_rf3.cpp:251-265
    rng = np.random.default_rng(29)
    m = 75
    sigma = rng.uniform(1.0, 5.0, m)
    for _ in range(20):
        u, v = rng.standard_normal(m), rng.standard_normal(m)
        lhs = v @ O.rf3_apply_1d(u, sigma)
        rhs = O.rf3_apply_1d(v, sigma, transpose=True) @ u
        assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(u) * np.linalg.norm(v)


def test_rf3_too_short():  # test_rf3.cpp:267-271
    with pytest.raises(O.OracleError, match="segment length must be >= 4"):
        O.rf3_apply_1d(np.zeros(3), 2.0)


def test_rational_gauss():  # test_rf3.cpp:273-282, acceptance criterion 4
    err0 = abs(O.rational_gauss(0.0) - 1 / math.sqrt(2 * PI))
    assert abs(err0 - 2.52e-3) <= 0.01 * 2.52e-3 and err0 < 2.7e-3
    for t in (0.5, 1.9, 3.05, 6.0):
        assert O.rational_gauss(t) == O.rational_gauss(-t)


# ---------------------------------------------------------------- rf1
def test_rf1_closed_form():  # test_rf1.cpp:18-23
    a, b = O.rf1_coefficients(1.0, 1)
    assert rel(a, 2 - math.sqrt(3)) <= 1e-15
    assert rel(b, math.sqrt(3) - 1) <= 1e-15
    assert a + b == 1.0


def test_rf1_r2_recovery():  # test_rf1.cpp:25-40
    for sigma in (0.5, 1.0, 1.7, 2.0, 4.2, 5.0, 10.0, 25.0):
        for k in (1, 2, 5, 10):
            a, b = O.rf1_coefficients(sigma, k)
            assert 0 < a < 1 and a + b == 1.0
            r2 = 2.0 * k * a / ((1 - a) * (1 - a))
            assert rel(r2, sigma * sigma) <= 1e-12
            q = k / (sigma * sigma)
            assert rel(b, math.sqrt(q * (q + 2)) - q) <= 1e-12


def test_rf1_wide_and_invalid():  # test_rf1.cpp:42-53
    a, b = O.rf1_coefficients(1e8, 1)
    assert 1 - 2e-8 < a < 1 and b < 2e-8
    for s, k in ((0.0, 1), (-1.0, 1), (1.0, 0)):
        with pytest.raises(O.OracleError):
            O.rf1_coefficients(s, k)


def rf1_straight(s0, alpha, beta, k):  # oracles.hpp:32-42
    m = len(s0)
    s = np.array(s0, dtype=float)
    p = np.zeros(m)
    for _ in range(k):
        p[0] = beta * s[0]
        for i in range(1, m):
            p[i] = beta * s[i] + alpha * p[i - 1]
        s[m - 1] = beta * p[m - 1]
        for i in range(m - 2, -1, -1):
            s[i] = beta * p[i] + alpha * s[i + 1]
    return s


def test_rf1_straight_line_and_props():  # test_rf1.cpp:63-114
    rng = np.random.default_rng(7)
    u = rng.standard_normal(64)
    for k in (1, 3):
        a, b = O.rf1_coefficients(2.5, k)
        got = O.rf1_apply_1d(u, 2.5, k)
        want = rf1_straight(u, a, b, k)
        assert np.linalg.norm(got - want) <= 1e-14 * np.linalg.norm(want)
    assert np.linalg.norm(O.rf1_apply_1d(np.zeros(32), 2.0, 5)) == 0.0
    for sigma, k in ((2.0, 1), (2.0, 10), (5.0, 10)):
        m = max(int(8.0 * sigma * math.sqrt(k)) + 1, 16)
        out = O.rf1_apply_1d(np.full(m, 3.25), sigma, k)
        assert rel(out[m // 2], 3.25) <= 0.01
    m = 200
    d1, d2 = np.zeros(m), np.zeros(m)
    d1[m // 2] = 1
    d2[m // 2 + 1] = 1
    r1, r2 = O.rf1_apply_1d(d1, 2.0, 5), O.rf1_apply_1d(d2, 2.0, 5)
    assert max(abs(r2[i + 1] - r1[i]) for i in range(16, m - 17)) < 1e-10


def test_rf1_transpose_dot_varying():  # test_rf1.cpp:134-148
    rng = np.random.default_rng(23)
    m = 70
    sigma = rng.uniform(1.0, 4.0, m)
    for _ in range(20):
        u, v = rng.standard_normal(m), rng.standard_normal(m)
        lhs = v @ O.rf1_apply_1d(u, sigma, 3)
        rhs = O.rf1_apply_1d(v, sigma, 3, transpose=True) @ u
        assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(u) * np.linalg.norm(v)


def test_rf1_too_short():  # test_rf1.cpp:150-155
    with pytest.raises(O.OracleError, match="segment length must be >= 2"):
        O.rf1_apply_1d(np.ones(1), 2.0, 1)


# ---------------------------------------------------- acceptance goldens
def impulse_err(sigma, order, k, length=300):  # diagnostics.cpp:69-95
    c = length // 2
    d = np.zeros(length)
    d[c] = 1.0
    if order == 1:
        h = O.rf1_apply_1d(d, sigma, k)
    else:
        h = O.rf3_apply_1d(d, sigma)
    i = np.arange(length)
    g = np.exp(-((i - c) ** 2) / (2 * sigma * sigma))
    return float(np.linalg.norm(h / h.sum() - g / g.sum()))


def test_acceptance_criterion1_numbers(golden):  # test_output.txt:9
    ref = golden["acceptance"]["criterion1_impulse_l2"]
    got = {"err1": impulse_err(2.0, 1, 1), "err5": impulse_err(2.0, 1, 5),
           "err10": impulse_err(2.0, 1, 10), "err3": impulse_err(2.0, 3, 1)}
    for k, v in got.items():  # the reference printed 6 significant digits
        assert rel(v, ref[k]) <= 5e-6, (k, v, ref[k])


def test_acceptance_criterion3_numbers(golden):  # test_output.txt:11
    for row in golden["acceptance"]["criterion3_dc"]:
        sigma = row["sigma"]
        m = int(16 * sigma * math.sqrt(10.0)) + 64
        g1 = O.rf1_apply_1d(np.ones(m), sigma, 10)[m // 2]
        g3 = O.rf3_apply_1d(np.ones(m), sigma)[m // 2]
        assert rel(g1, row["g1"]) <= 5e-6
        assert rel(g3, row["g3"]) <= 5e-6
