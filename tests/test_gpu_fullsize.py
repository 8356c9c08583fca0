"""Full-size runs of the BASELINE.json configs (gpu).

* C2 and C3 at their full sizes against the oracle, forward and adjoint,
  3rd-RF and 1st-RF (K=5): relative max-norm 1e-12.
* C4 (2 variables x 75 levels x 1442x1021), fp64 and fp32: the adjoint dot
  test <Vx, y> = <x, V^T y> that BASELINE.json's config 4 asks for, with a
  seeded variance field.
* C5 (4320x2160x100, 7.5 GB per fp64 field): size-independent properties --
  linearity, the adjoint dot test for G_y G_x, exact zeros on land and
  bit-identical reruns.

Dot-test tolerance: |<Vx,y> - <x,V^T y>| <= tol * ||Vx|| ||y|| (the
Cauchy-Schwarz scale of the inner product), tol = 1e-12 fp64, 1e-5 fp32.
"""
import os

import numpy as np
import pytest

import oracle as O
from helpers import relmax

pytestmark = pytest.mark.gpu

TOL64 = 1e-12


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1404_5756_b200 as P
    return P


def _ops(P, cfg, order=3, k=1, variance=None, oracle=True):
    grid = P.Grid2D(cfg.nx, cfg.ny, cfg.dx, cfg.dy, cfg.mask)
    opts = P.CovarianceOptions(order=P.FilterOrder(order), k_iterations=k, variance=variance)
    gpu = P.HorizontalCovarianceOp(grid, P.ScaleField(cfg.rx, cfg.ry), opts)
    cpu = None
    if oracle:
        cpu = O.OracleOp(cfg.nx, cfg.ny, cfg.dx, cfg.dy, cfg.mask, cfg.rx, cfg.ry, order=order,
                         k_iterations=k, variance=variance, threads=os.cpu_count() or 8)
    return gpu, cpu


@pytest.mark.parametrize("name", ["C2", "C3"])
@pytest.mark.parametrize("order,k", [(3, 1), (1, 5)])
def test_full_size_parity_vs_oracle(P, name, order, k):
    from paper_1404_5756_b200 import synth
    cfg = synth.make_config(name)
    var = np.random.default_rng(5).uniform(0.5, 2.0, (cfg.nlev, cfg.ny, cfg.nx))
    gpu, cpu = _ops(P, cfg, order, k, variance=var)
    f = synth.make_field(cfg)
    for kind in ("GYGX", "VT"):
        got = gpu.apply(getattr(P, kind), f)
        want = cpu.apply(getattr(O, kind), f)
        assert relmax(got, want) <= TOL64, (name, order, kind, relmax(got, want))
        assert np.all(got[:, ~cfg.mask] == 0.0)


def _dot_test(P, op, x, y):
    import torch
    vx = op.apply(P.V, x)
    vty = op.apply(P.VT, y)
    torch.cuda.synchronize()
    a = torch.sum(vx.double() * y.double()).item()
    b = torch.sum(x.double() * vty.double()).item()
    scale = torch.linalg.vector_norm(vx.double()).item() * torch.linalg.vector_norm(y.double()).item()
    return abs(a - b) / scale


@pytest.mark.parametrize("dt,tol", [("f64", 1e-12), ("f32", 1e-5)])
def test_c4_adjoint_dot_test(P, dt, tol):
    import torch
    from paper_1404_5756_b200 import synth
    cfg = synth.make_config("C4")
    var = np.random.default_rng(6).uniform(0.5, 2.0, (cfg.nlev, cfg.ny, cfg.nx))
    op, _ = _ops(P, cfg, variance=var, oracle=False)
    tdt = torch.float64 if dt == "f64" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(44)
    shape = (cfg.nvar, cfg.nlev, cfg.ny, cfg.nx)
    x = torch.randn(shape, generator=g, device="cuda", dtype=torch.float64).to(tdt)
    y = torch.randn(shape, generator=g, device="cuda", dtype=torch.float64).to(tdt)
    err = _dot_test(P, op, x, y)
    assert err <= tol, err


def test_c5_full_size_properties(P):
    import torch
    from paper_1404_5756_b200 import synth
    cfg = synth.make_config("C5")
    op, _ = _ops(P, cfg, oracle=False)
    shape = (1, cfg.nlev, cfg.ny, cfg.nx)
    g = torch.Generator(device="cuda").manual_seed(55)
    x = torch.randn(shape, generator=g, device="cuda", dtype=torch.float64)
    y = torch.randn(shape, generator=g, device="cuda", dtype=torch.float64)
    fx = op.apply(P.GYGX, x)
    fy = op.apply(P.GYGX, y)
    # linearity
    fz = op.apply(P.GYGX, 2.0 * x - 3.0 * y)
    lin = (fz - (2.0 * fx - 3.0 * fy)).abs().max() / (2.0 * fx - 3.0 * fy).abs().max()
    assert lin.item() <= TOL64, lin.item()
    # deterministic reruns, bit for bit
    assert torch.equal(op.apply(P.GYGX, x), fx)
    # land is exactly zero
    land = torch.from_numpy(~cfg.mask).cuda()
    assert torch.count_nonzero(fx[0][land]).item() == 0
    # adjoint: <G_y G_x x, y> = <x, G_x^T G_y^T y>
    gty = op.apply(P.GXT, op.apply(P.GYT, y))
    a = torch.sum(fx * y).item()
    b = torch.sum(x * gty).item()
    scale = torch.linalg.vector_norm(fx).item() * torch.linalg.vector_norm(y).item()
    assert abs(a - b) / scale <= TOL64, abs(a - b) / scale


def test_full_size_analysis_vs_oracle(P):
    """3D-VAR analysis at full horizontal size: C3
    level 0 (1442x1021, tripolar-like mask and length scales), 20,000
    observations. H and H^T bit-identical to the oracle; 4 CG iterations of
    the device solve within 1e-10 of the oracle's."""
    from paper_1404_5756_b200 import synth
    cfg = synth.make_config("C3", nlev=1)
    gpu, cpu = _ops(P, cfg)
    m = cfg.mask[0]
    rng = np.random.default_rng(42)
    pos = np.column_stack([rng.uniform(0, cfg.nx - 1, 80000), rng.uniform(0, cfg.ny - 1, 80000)])
    i0 = np.minimum(np.floor(pos[:, 0]).astype(int), cfg.nx - 2)
    j0 = np.minimum(np.floor(pos[:, 1]).astype(int), cfg.ny - 2)
    ok = m[j0, i0] | m[j0, i0 + 1] | m[j0 + 1, i0] | m[j0 + 1, i0 + 1]
    pos = pos[ok][:20000]
    vals = rng.standard_normal(len(pos))
    rv = rng.uniform(0.5, 2.0, len(pos))
    obs = P.ObsSet(pos, vals, rv)
    co = O.OracleObs(cpu, pos, vals, rv)
    f = rng.standard_normal((cfg.ny, cfg.nx))
    assert np.array_equal(P.obs_operator(f, obs, gpu), co.h(f))
    assert np.array_equal(P.obs_operator_transpose(vals, obs, gpu), co.ht(vals))
    got = P.solve(obs, gpu, P.SolveOptions(tol=1e-30, max_iter=4))
    want = co.solve(tol=1e-30, max_iter=4)
    assert got.cg_iterations == want["cg_iterations"] == 4
    assert relmax(got.increment, want["increment"]) <= 1e-10
    assert np.allclose(got.gradient_norms, want["gradient_norms"], rtol=1e-10, atol=0)
