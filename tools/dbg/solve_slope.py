"""Marginal time of a CG iteration: slope of rgf_solve wall time against the iteration count."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1404_5756_b200 as P
from paper_1404_5756_b200 import synth
nobs = 20000
cfg = synth.make_config("C3", nlev=1)
m = cfg.mask[0]
rng = np.random.default_rng(42)
pos = np.column_stack([rng.uniform(0, cfg.nx - 1, 4 * nobs), rng.uniform(0, cfg.ny - 1, 4 * nobs)])
i0 = np.minimum(np.floor(pos[:, 0]).astype(int), cfg.nx - 2)
j0 = np.minimum(np.floor(pos[:, 1]).astype(int), cfg.ny - 2)
ok = m[j0, i0] | m[j0, i0 + 1] | m[j0 + 1, i0] | m[j0 + 1, i0 + 1]
pos = pos[ok][:nobs]
vals = rng.standard_normal(nobs); rv = rng.uniform(0.5, 2.0, nobs)
for order, k in ((3, 1), (1, 5)):
    grid = P.Grid2D(cfg.nx, cfg.ny, cfg.dx, cfg.dy, cfg.mask)
    op = P.HorizontalCovarianceOp(grid, P.ScaleField(cfg.rx, cfg.ry),
                                  P.CovarianceOptions(order=P.FilterOrder(order), k_iterations=k))
    obs = P.ObsSet(pos, vals, rv)
    P.solve(obs, op, P.SolveOptions(tol=1e-30, max_iter=2))
    res = {}
    for it in (2, 6, 12):
        best = 1e9
        for rep in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            an = P.solve(obs, op, P.SolveOptions(tol=1e-30, max_iter=it))
            best = min(best, time.perf_counter() - t0)
        res[it] = (an.cg_iterations, best)
    print(order, k, {i: (n, round(t * 1e3, 3)) for i, (n, t) in res.items()},
          "slope ms/iter", round((res[12][1] - res[2][1]) / (res[12][0] - res[2][0]) * 1e3, 3))

# fixed parts of a solve (last operator): observation handle, a 0-iteration solve
import ctypes
t0 = time.perf_counter(); d = P._DeviceObs(op, obs); torch.cuda.synchronize(); t1 = time.perf_counter()
print("obs handle ms", round((t1 - t0) * 1e3, 3))
for it in (0, 1):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    P.solve(obs, op, P.SolveOptions(tol=1e-30, max_iter=it)); t1 = time.perf_counter()
    print("solve max_iter", it, "ms", round((t1 - t0) * 1e3, 3))
t0 = time.perf_counter(); del d; torch.cuda.synchronize(); print("obs destroy ms", round((time.perf_counter() - t0) * 1e3, 3))
x = np.random.default_rng(0).standard_normal((1, 1, cfg.ny, cfg.nx))
for kind in ("V", "VT"):
    op.apply(getattr(P, kind), x)
    t0 = time.perf_counter(); op.apply(getattr(P, kind), x); print("host apply", kind, "ms", round((time.perf_counter() - t0) * 1e3, 3))
