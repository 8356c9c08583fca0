"""Profiling driver: one GX and one GY of the 1st-RF K=5 on C5-shaped levels."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1404_5756_b200 as P
from paper_1404_5756_b200 import synth

nlev = int(sys.argv[1]) if len(sys.argv) > 1 else 20
kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else ["GX", "GY"]
dt = torch.float32 if len(sys.argv) > 3 and sys.argv[3] == "f32" else torch.float64
c = synth.make_config("C5", nlev=nlev)
x = torch.from_numpy(synth.make_field(c)).cuda().to(dt)
grid = P.Grid2D(c.nx, c.ny, c.dx, c.dy, c.mask)
op = P.HorizontalCovarianceOp(grid, P.ScaleField(c.rx, c.ry),
                              P.CovarianceOptions(order=P.FilterOrder(1), k_iterations=5))
for rep in range(2):
    for kind in kinds:
        out = op.apply(getattr(P, kind), x)
torch.cuda.synchronize()
print("ok")
