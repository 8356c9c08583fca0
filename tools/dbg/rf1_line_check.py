"""Dev check of the line-resident 1st-RF (rf1_line.cuh): parity against the
oracle and the streaming passes on small grids, then timing on C5-shaped
levels. Run on a GPU box: python tools/dbg/rf1_line_check.py [nlev]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import oracle as O
import paper_1404_5756_b200 as P
from helpers import checkered_mask, relmax, uniform_grid
from paper_1404_5756_b200 import synth

KINDS = ["GX", "GY", "GXT", "GYT", "V", "VT", "B", "GYGX"]


def case(seed, nx, ny, nlev, sea, smin=1.2, smax=4.5):
    rng = np.random.default_rng(seed)
    g = uniform_grid(nx, ny, 5000.0, 7000.0, nlev=nlev)
    g["dx"] = 5000.0 * rng.uniform(0.7, 1.3, (ny, nx))
    g["mask"] = checkered_mask(nx, ny, seed + 1, sea, nlev=nlev) if sea < 1 else np.ones((nlev, ny, nx), bool)
    rx = g["dx"] * rng.uniform(smin, smax, (ny, nx))
    ry = g["dy"] * rng.uniform(smin, smax, (ny, nx))
    return g, rx, ry


def build(g, rx, ry, k, ghost, var, line):
    os.environ["RGF_B200_RF1LINE"] = "1" if line else "0"
    grid = P.Grid2D(g["nx"], g["ny"], g["dx"], g["dy"], g["mask"], 0)
    opts = P.CovarianceOptions(order=P.FilterOrder(1), k_iterations=k, ghost_width=ghost, variance=var)
    return P.HorizontalCovarianceOp(grid, P.ScaleField(rx, ry), opts)


worst = 0.0
bad = 0
for (nx, ny, nlev, sea, k, ghost) in [
        (57, 43, 3, 0.8, 1, None), (57, 43, 3, 0.8, 5, None), (70, 44, 3, 0.65, 2, None),
        (70, 44, 2, 0.65, 5, 0), (70, 44, 2, 0.5, 3, 2), (300, 200, 2, 0.7, 5, None),
        (1000, 517, 1, 0.8, 5, None), (1030, 130, 1, 1.0, 5, None), (64, 2100, 1, 0.9, 2, None),
        (4320, 40, 1, 0.8, 5, None)]:
    g, rx, ry = case(nx + k, nx, ny, nlev, sea)
    var = np.random.default_rng(2).uniform(0.5, 2.0, (nlev, ny, nx))
    cpu = O.OracleOp(nx, ny, g["dx"], g["dy"], g["mask"], rx, ry, order=1, k_iterations=k,
                     ghost_width=ghost, variance=var, threads=8)
    gl = build(g, rx, ry, k, ghost, var, True)
    gs = build(g, rx, ry, k, ghost, var, False)
    f = np.random.default_rng(3).standard_normal((2, nlev, ny, nx))
    for name in KINDS:
        want = cpu.apply(getattr(O, name), f)
        l0 = gl.launch_count()
        got = gl.apply(getattr(P, name), f)
        nl = gl.launch_count() - l0
        old = gs.apply(getattr(P, name), f)
        e1, e2 = relmax(got, want), relmax(old, want)
        land_ok = bool(np.all(got[:, ~g["mask"]] == 0.0))
        worst = max(worst, e1)
        flag = "" if (e1 <= 1e-12 and land_ok) else "  <-- FAIL"
        bad += flag != ""
        print(f"{nx}x{ny}x{nlev} sea={sea} k={k} ghost={ghost} {name:5s} line {e1:.2e} stream {e2:.2e} "
              f"launches {nl} land0 {land_ok}{flag}", flush=True)
    f32 = f.astype(np.float32)
    for name in ("GYGX", "VT"):
        want = cpu.apply(getattr(O, name), f32.astype(np.float64))
        e1 = relmax(gl.apply(getattr(P, name), f32), want)
        flag = "" if e1 <= 1e-5 else "  <-- FAIL"
        bad += flag != ""
        print(f"   f32 {name} line {e1:.2e}{flag}", flush=True)
print("worst fp64", worst, "failures", bad)

# ---- timing on C5-shaped levels
nlev = int(sys.argv[1]) if len(sys.argv) > 1 else 20
c = synth.make_config("C5", nlev=nlev)
f = torch.from_numpy(synth.make_field(c)).cuda()
for dt in (torch.float64, torch.float32):
    x = f.to(dt)
    for line in (True, False):
        os.environ["RGF_B200_RF1LINE"] = "1" if line else "0"
        grid = P.Grid2D(c.nx, c.ny, c.dx, c.dy, c.mask)
        op = P.HorizontalCovarianceOp(grid, P.ScaleField(c.rx, c.ry),
                                      P.CovarianceOptions(order=P.FilterOrder(1), k_iterations=5))
        for kind in ("GX", "GY", "GYGX", "VT"):
            out = op.apply(getattr(P, kind), x)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                out = op.apply(getattr(P, kind), x)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
            print(f"C5 nlev={nlev} {dt} line={line} {kind}: {ms:.3f} ms  {c.nx * c.ny * nlev / ms / 1e6:.2f} Gpt/s",
                  flush=True)
        del op
