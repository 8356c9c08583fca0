"""Randomised parity sweep of the 1st-RF (line-resident kernel and its fallbacks)
against the oracle: shapes, masks, K, ghost widths, variance, dtypes.
usage: python tools/dbg/rf1_fuzz.py [cases] [seed]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
import paper_1404_5756_b200 as P
from helpers import relmax

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 120
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
KINDS = ["GX", "GY", "GXT", "GYT", "V", "VT", "B", "GYGX"]
bad = 0
worst = 0.0
for t in range(cases):
    nx = int(rng.choice([4, 5, 7, 17, 33, 64, 129, 300, 577, 1153, 1200, 2200]))
    ny = int(rng.choice([4, 5, 6, 9, 31, 65, 130, 289, 577, 600, 1100]))
    if nx * ny > 400000:
        ny = max(4, 400000 // nx)
    nlev = int(rng.integers(1, 4))
    nvar = int(rng.integers(1, 3))
    k = int(rng.integers(1, 7))
    ghost = [None, 0, 1, 5, 40][int(rng.integers(0, 5))]
    style = int(rng.integers(0, 4))
    if style == 0:
        mask = rng.uniform(size=(nlev, ny, nx)) < rng.uniform(0.3, 0.95)
    elif style == 1:
        mask = np.ones((nlev, ny, nx), bool)
    elif style == 2:  # one mask for all levels, blobs
        base = rng.uniform(size=(ny, nx))
        for _ in range(2):
            base = (base + np.roll(base, 1, 0) + np.roll(base, 1, 1) + np.roll(base, -1, 0) + np.roll(base, -1, 1)) / 5
        mask = np.repeat((base > np.quantile(base, 0.3))[None], nlev, axis=0)
    else:  # stripes: land every few points
        mask = np.ones((nlev, ny, nx), bool)
        mask[:, :, :: int(rng.integers(2, 6))] = False
        mask[:, :: int(rng.integers(2, 6)), :] = False
    if not mask.any():
        mask[:, 0, 0] = True
    dx = 5000.0 * rng.uniform(0.7, 1.3, (ny, nx))
    dy = np.full((ny, nx), 7000.0)
    smax = float(rng.choice([2.0, 4.5, 10.0]))
    rx = dx * rng.uniform(1.0, smax, (ny, nx))
    ry = dy * rng.uniform(1.0, smax, (ny, nx))
    var = rng.uniform(0.5, 2.0, (nlev, ny, nx)) if rng.uniform() < 0.5 else None
    try:
        grid = P.Grid2D(nx, ny, dx, dy, mask, 0)
        op = P.HorizontalCovarianceOp(grid, P.ScaleField(rx, ry), P.CovarianceOptions(
            order=P.FilterOrder(1), k_iterations=k, ghost_width=ghost, variance=var))
        cpu = O.OracleOp(nx, ny, dx, dy, mask, rx, ry, order=1, k_iterations=k, ghost_width=ghost,
                         variance=var, threads=8)
    except Exception as e:  # both must reject the same way
        print(t, "ctor", type(e).__name__, str(e)[:80])
        continue
    f = rng.standard_normal((nvar, nlev, ny, nx))
    f[:, ~mask] = rng.choice([0.0, 1e30, np.nan])  # land inputs are ignored
    f32 = rng.uniform() < 0.3
    x = f.astype(np.float32) if f32 else f
    tol = 1e-5 if f32 else 1e-12
    for name in rng.choice(KINDS, 3, replace=False):
        got = op.apply(getattr(P, name), x)
        want = cpu.apply(getattr(O, name), np.where(mask[None], x.astype(np.float64), 0.0))
        e = relmax(got, want) if np.abs(want).max() > 0 else float(np.abs(got).max())
        ok = e <= tol and np.all(got[:, ~mask] == 0.0) and np.all(np.isfinite(got))
        worst = max(worst, e / tol)
        if not ok:
            bad += 1
            print(f"FAIL case {t}: {nx}x{ny}x{nlev}x{nvar} k={k} ghost={ghost} style={style} "
                  f"var={var is not None} f32={f32} {name} err={e:.3e}", flush=True)
    if t % 20 == 0:
        print("case", t, "ok so far; worst err/tol", worst, flush=True)
print("done: failures", bad, "worst err/tol", worst)
