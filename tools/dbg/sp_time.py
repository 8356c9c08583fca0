"""Debug: device-path parity of one single-pass case, and x-sweep timing vs row length."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import torch
import paper_1404_5756_b200 as P
import oracle as O
from helpers import relmax
from test_gpu_single_pass import shared_mask, pair

for nx, ny, nlev, host in ((4320, 6, 1, False), (2176, 6, 2, True), (4320, 6, 2, True)):
    mask = shared_mask(nx, ny, nlev, 100 + nx, 0.7, True)
    gpu, cpu = pair(P, nx, ny, mask, 200 + nx)
    f = np.random.default_rng(4).standard_normal((1, nlev, ny, nx))
    t = f if host else torch.from_numpy(f).cuda()
    try:
        got = gpu.apply(P.GX, t)
        torch.cuda.synchronize()
        got = got if host else got.cpu().numpy()
        print("parity", nx, ny, nlev, host, relmax(got, cpu.apply(O.GX, f)), flush=True)
    except Exception as e:
        print("FAIL", nx, ny, nlev, host, e, flush=True)
        break

for nx in (4320, 2176, 1088, 544):
    ny, nlev = 2160, 100 if len(sys.argv) < 2 else int(sys.argv[1])
    m = np.ones((ny, nx), dtype=bool)
    m[:, ::37] = False
    grid = P.Grid2D(nx, ny, np.ones((ny, nx)), np.ones((ny, nx)), np.repeat(m[None], nlev, 0))
    s = np.full((ny, nx), 5.0) + np.random.default_rng(1).uniform(0, 1, (ny, nx))
    op = P.HorizontalCovarianceOp(grid, P.ScaleField(s, s))
    x = torch.randn((1, nlev, ny, nx), device="cuda", dtype=torch.float64)
    y = torch.empty_like(x)
    for _ in range(3):
        op.apply(P.GX, x, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        op.apply(P.GX, x, y)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    n = nx * ny * nlev
    print(f"nx={nx} x-sweep {ms:.3f} ms  {n / ms / 1e6:.1f} Gpt/s  {n * 16 / ms / 1e6:.0f} GB/s", flush=True)
    del op, x, y
