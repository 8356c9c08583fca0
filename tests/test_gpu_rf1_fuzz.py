"""Randomised parity of the 1st-RF against the oracle: line lengths across
the resident shapes (and past them), iid / blob / stripe / all-sea masks,
K in 1..6, ghost widths 0/1/5/40/default, variance, fp64 and fp32, garbage
(NaN, 1e30) on land in the input. tools/dbg/rf1_fuzz.py runs the long form."""
import numpy as np
import pytest

import oracle as O
from helpers import relmax

pytestmark = pytest.mark.gpu
KINDS = ["GX", "GY", "GXT", "GYT", "V", "VT", "B", "GYGX"]


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1404_5756_b200 as P
    return P


def make_mask(rng, style, nlev, ny, nx):
    if style == 0:
        return rng.uniform(size=(nlev, ny, nx)) < rng.uniform(0.3, 0.95)
    if style == 1:
        return np.ones((nlev, ny, nx), bool)
    if style == 2:  # one mask for every level (setup reused from plane to plane)
        base = rng.uniform(size=(ny, nx))
        for _ in range(2):
            base = (base + np.roll(base, 1, 0) + np.roll(base, 1, 1) + np.roll(base, -1, 0) +
                    np.roll(base, -1, 1)) / 5
        return np.repeat((base > np.quantile(base, 0.3))[None], nlev, axis=0)
    mask = np.ones((nlev, ny, nx), bool)  # stripes: single-point land gaps and short segments
    mask[:, :, :: int(rng.integers(2, 6))] = False
    mask[:, :: int(rng.integers(2, 6)), :] = False
    return mask


@pytest.mark.parametrize("seed", range(8))
def test_rf1_random_cases(P, seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(6):
        nx = int(rng.choice([4, 5, 7, 17, 33, 64, 129, 300, 577, 1153, 1200, 2200]))
        ny = int(rng.choice([4, 5, 6, 9, 31, 65, 130, 289, 577, 600, 1100]))
        if nx * ny > 300000:
            ny = max(4, 300000 // nx)
        nlev, nvar, k = int(rng.integers(1, 4)), int(rng.integers(1, 3)), int(rng.integers(1, 7))
        ghost = [None, 0, 1, 5, 40][int(rng.integers(0, 5))]
        mask = make_mask(rng, int(rng.integers(0, 4)), nlev, ny, nx)
        if not mask.any():
            mask[:, 0, 0] = True
        dx = 5000.0 * rng.uniform(0.7, 1.3, (ny, nx))
        dy = np.full((ny, nx), 7000.0)
        smax = float(rng.choice([2.0, 4.5, 10.0]))
        rx = dx * rng.uniform(1.0, smax, (ny, nx))
        ry = dy * rng.uniform(1.0, smax, (ny, nx))
        var = rng.uniform(0.5, 2.0, (nlev, ny, nx)) if rng.uniform() < 0.5 else None
        gpu = P.HorizontalCovarianceOp(P.Grid2D(nx, ny, dx, dy, mask, 0), P.ScaleField(rx, ry),
                                       P.CovarianceOptions(order=P.FilterOrder(1), k_iterations=k,
                                                           ghost_width=ghost, variance=var))
        cpu = O.OracleOp(nx, ny, dx, dy, mask, rx, ry, order=1, k_iterations=k, ghost_width=ghost,
                         variance=var, threads=4)
        f = rng.standard_normal((nvar, nlev, ny, nx))
        f[:, ~mask] = rng.choice([0.0, 1e30, np.nan])  # the reference never reads land inputs
        f32 = rng.uniform() < 0.3
        x = f.astype(np.float32) if f32 else f
        tol = 1e-5 if f32 else 1e-12
        clean = np.where(mask[None], x.astype(np.float64), 0.0)
        for name in rng.choice(KINDS, 3, replace=False):
            got = gpu.apply(getattr(P, name), x)
            want = cpu.apply(getattr(O, name), clean)
            err = relmax(got, want) if np.abs(want).max() > 0 else float(np.abs(got).max())
            info = (seed, nx, ny, nlev, nvar, k, ghost, f32, name, err)
            assert err <= tol, info
            assert np.all(got[:, ~mask] == 0.0) and np.all(np.isfinite(got)), info
