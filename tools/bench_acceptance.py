"""The reference's own timed case (proj/tests/acceptance.cpp:268-300,
proj/test_output.txt:16): 1024x1024, sigma = 2 uniform, all sea, unit_dc,
x+y application, median of 5. BASELINE.md lists its single-thread CPU
figures (3rd-RF 32.1 Mpt/s, 1st-RF K=5 15.1 Mpt/s). Here: the oracle port
with 1 thread and with every host thread, and the B200 path (device-resident,
CUDA events). Prints one JSON line."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1404_5756_b200 as P  # noqa: E402

n = 1024
one = np.ones((n, n))
mask = np.ones((n, n), bool)
rng = np.random.default_rng(1)
f = rng.standard_normal((1, 1, n, n))
out = {"case": "1024x1024, sigma=2 uniform, all sea, unit_dc, x+y (acceptance.cpp:268-300)",
       "reference_published_1thread_Mpts": {"3rd-RF": 32.1, "1st-RF K=5": 15.1}}
quick = "--quick" in sys.argv  # GPU only, 3rd-RF (profiling runs)
for name, order, k in (("3rd-RF", 3, 1),) + ((("1st-RF K=5", 1, 5),) if not quick else ()):
    row = {}
    for threads in (() if quick else (1, os.cpu_count() or 1)):
        op = O.OracleOp(n, n, one, one, mask, one * 2.0, one * 2.0, order=order, k_iterations=k,
                        threads=threads)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            op.apply(O.GYGX, f)
            ts.append(time.perf_counter() - t0)
        row[f"oracle_{threads}t_Mpts"] = n * n / statistics.median(ts) / 1e6
    grid = P.Grid2D(n, n, one, one, mask)
    gop = P.HorizontalCovarianceOp(grid, P.ScaleField(one * 2.0, one * 2.0),
                                   P.CovarianceOptions(order=P.FilterOrder(order), k_iterations=k))
    x = torch.from_numpy(f).cuda()
    y = torch.empty_like(x)
    for _ in range(5):
        gop.apply(P.GYGX, x, y)
    torch.cuda.synchronize()
    ts = []
    for _ in range(21):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gop.apply(P.GYGX, x, y)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    row["b200_Mpts"] = n * n / statistics.median(ts) / 1e6
    row["b200_ms"] = statistics.median(ts) * 1e3
    if not quick:
        want = O.OracleOp(n, n, one, one, mask, one * 2.0, one * 2.0, order=order, k_iterations=k,
                          threads=os.cpu_count() or 1).apply(O.GYGX, f)
        got = y.cpu().numpy()
        row["rel_max_err_vs_oracle"] = float(np.max(np.abs(got - want)) / np.max(np.abs(want)))
    for sname, kind in (("x", P.GX), ("y", P.GY)):
        ts2 = []
        for _ in range(11):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gop.apply(kind, x, y)
            b.record()
            torch.cuda.synchronize()
            ts2.append(a.elapsed_time(b))
        row[f"b200_{sname}_sweep_ms"] = statistics.median(ts2)
    if quick:
        out[name] = row
        continue
    out[name] = row
out["host_threads"] = os.cpu_count()
print(json.dumps(out))
