import sys, numpy as np, torch
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import test_gpu_parity as T
import paper_1404_5756_b200 as P, oracle as O
from helpers import relmax
for nx in (57, 64):
    g, rx, ry = T.random_case(700 + 3 + nx, nx=nx, ny=29, nlev=10, sea=0.7, smax=6.0)
    var = np.random.default_rng(21).uniform(0.5, 2.0, (10, 29, nx))
    gpu, cpu = T.build_pair(P, g, rx, ry, order=3, k=1, variance=var)
    f = np.random.default_rng(22).standard_normal((2, 10, 29, nx))
    for name in T.KINDS:
        kind = getattr(P, name)
        host = gpu.apply(kind, f); host2 = gpu.apply(kind, f)
        dev = gpu.apply(kind, torch.from_numpy(f).cuda()).cpu().numpy()
        dev2 = gpu.apply(kind, torch.from_numpy(f).cuda()).cpu().numpy()
        want = cpu.apply(getattr(O, name), f)
        print(nx, name, 'host==dev', np.array_equal(host, dev), 'hostdet', np.array_equal(host,host2), 'devdet', np.array_equal(dev,dev2),
              'err host', relmax(host, want), 'err dev', relmax(dev, want), flush=True)
    g2 = f.astype(np.float32)
    want = gpu.apply(P.VT, g2.copy())
    gpu.apply(P.VT, g2, out=g2)
    print('inplace f32', np.array_equal(g2, want), relmax(g2, want))
    want64 = gpu.apply(P.VT, f.copy()); f2 = f.copy(); gpu.apply(P.VT, f2, out=f2)
    print('inplace f64', np.array_equal(f2, want64), relmax(f2, want64))
