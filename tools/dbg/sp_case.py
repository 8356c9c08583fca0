"""Debug: one single-pass case (nx, ny, nlev) against the oracle, device path."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import torch
import paper_1404_5756_b200 as P
import oracle as O
from helpers import relmax
from test_gpu_single_pass import shared_mask, pair
nx, ny, nlev = (int(v) for v in sys.argv[1:4])
mask = shared_mask(nx, ny, nlev, 100 + nx, 0.7, True)
gpu, cpu = pair(P, nx, ny, mask, 200 + nx)
f = np.random.default_rng(4).standard_normal((1, nlev, ny, nx))
t = torch.from_numpy(f).cuda()
for name in ("GX", "GXT"):
    got = gpu.apply(getattr(P, name), t)
    torch.cuda.synchronize()
    print(name, relmax(got.cpu().numpy(), cpu.apply(getattr(O, name), f)), flush=True)
