"""Per-section cycle totals of the ring sweeps (dev build with -DRGF_RING_PROF,
loaded through RGF_B200_LIB). usage: ring_prof.py [config] [nlev]"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1404_5756_b200 as P
from paper_1404_5756_b200 import synth
cfgname = sys.argv[1] if len(sys.argv) > 1 else "C5"
nlev = int(sys.argv[2]) if len(sys.argv) > 2 else None
cfg = synth.make_config(cfgname, nlev=nlev)
grid = P.Grid2D(cfg.nx, cfg.ny, cfg.dx, cfg.dy, cfg.mask)
op = P.HorizontalCovarianceOp(grid, P.ScaleField(cfg.rx, cfg.ry), P.CovarianceOptions())
x = torch.randn((1, cfg.nlev, cfg.ny, cfg.nx), device="cuda", dtype=torch.float64)
y = torch.empty_like(x)
buf = (ctypes.c_ulonglong * 8)()
names = ["feed/spill", "bits+prefetch", "mbar wait", "causal", "partA+wb", "partB", "bookkeep", "tail"]
for name, kind in (("x", P.GX), ("y", P.GY), ("xT", P.GXT), ("yT", P.GYT)):
    for _ in range(2):
        op.apply(kind, x, y)
    torch.cuda.synchronize()
    P.lib.rgf_debug_ring_prof(buf, 1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); op.apply(kind, x, y); b.record(); torch.cuda.synchronize()
    P.lib.rgf_debug_ring_prof(buf, 1)
    tot = sum(buf)
    print(f"{name}: {a.elapsed_time(b):.3f} ms  total {tot/1e9:.2f} Gcyc  " +
          "  ".join(f"{n} {100*v/tot:.1f}%" for n, v in zip(names, buf)), flush=True)
