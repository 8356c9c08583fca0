#!/usr/bin/env python
"""Benchmark of the x+y recursive-filter application (apply_gy . apply_gx,
diagnostics.cpp:182's timed unit) on synthetic BASELINE.json grids.

Default workload: config C5 (4320x2160x100 levels, fp64, 3rd-RF, reference
default options: unit_dc, YvV95, ghost width ceil(9 max sigma)). Levels are
sharded across ranks (one process per GPU, torchrun), no collective on the
data path; weak scaling (every rank owns 100 levels of the same horizontal
grid). Prints ONE JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpoints/s per x+y filter application (3rd-RF)"
METRIC_RF1 = "Gpoints/s per x+y filter application (1st-RF, K={k})"


def metric_name(order, k):
    return METRIC if order == 3 else METRIC_RF1.format(k=k)
HBM_FALLBACK = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--order", type=int, default=3)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--nlev", type=int, default=None, help="levels per rank (default: config)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the 1st-RF / fp32 / adjoint figures (reported by default on 1 GPU)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def measured_traffic(cfg_name, dtype, order, kernel):
    """ncu DRAM bytes (read + write) per launch of the dominant sweep, from
    the committed capture summary (profiles/traffic.json); None if absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        return t[f"{cfg_name}/{dtype}/{order}"][kernel]
    except Exception:
        return None


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class CpuPort:
    """The oracle (C++ restatement of the reference, all host threads) on a
    bounded level sample of the same workload: the operator and the sample
    field are built once; each run() times one x+y application."""

    def __init__(self, cfg, order, k, seconds, levels_cap=None):
        import oracle as O
        self.O = O
        self.cfg = cfg
        self.threads = os.cpu_count() or 1
        self.op = O.OracleOp(cfg.nx, cfg.ny, cfg.dx, cfg.dy, cfg.mask, cfg.rx, cfg.ry,
                             order=order, k_iterations=k, threads=self.threads)
        rng = np.random.default_rng(99)
        f1 = rng.standard_normal((1, 1, cfg.ny, cfg.nx))
        t0 = time.perf_counter()
        self.op.apply(O.GYGX, f1, lev0=0, nlev_sub=1)
        t1 = time.perf_counter() - t0
        nl = max(1, min(cfg.nlev, int(seconds / max(t1, 1e-6))))
        if levels_cap:
            nl = min(nl, levels_cap)
        self.nl = nl
        self.f = rng.standard_normal((1, nl, cfg.ny, cfg.nx))
        pts = cfg.nx * cfg.ny * nl
        self.pts = pts
        self.sample = f"{nl} of {cfg.nlev} levels ({pts} points), 1 application"

    def run(self):
        t0 = time.perf_counter()
        self.op.apply(self.O.GYGX, self.f, lev0=0, nlev_sub=self.nl)
        return self.pts / (time.perf_counter() - t0) / 1e9


def cpu_port_rate(cfg, order, k, seconds, levels_cap=None):
    """One timed oracle application on a level sample; (Gpt/s, sample, cores)."""
    cp = CpuPort(cfg, order, k, seconds, levels_cap)
    return cp.run(), cp.sample, cp.threads


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU algorithm (oracle port; the
    reference itself is unbuildable here) with every host thread."""
    if rank != 0:
        return
    from paper_1404_5756_b200 import synth
    cfg = synth.make_config(args.config, nlev=args.nlev)
    k = args.k or (5 if args.order == 1 else 1)
    # operator and level sample built once; each step is one timed x+y
    # application of ~2 s of CPU work (the whole default run stays ~1 min)
    cp = CpuPort(cfg, args.order, k, 2.0)
    rates = []
    for i in range(args.warmup + args.steps):
        r = cp.run()
        if i >= args.warmup:
            rates.append(r)
    v = statistics.median(rates)
    sample, cores = cp.sample, cp.threads
    line = {"impl": "reference", "metric": metric_name(args.order, args.k or (5 if args.order == 1 else 1)),
            "value": v, "unit": "Gpoints/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": cfg.nx * cfg.ny * cfg.nlev * cfg.nvar / (v * 1e9) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} ({cfg.description}) order={args.order} k={k}",
                       "nx": cfg.nx, "ny": cfg.ny, "nlev": cfg.nlev, "nvar": cfg.nvar},
            "cpu_baseline": {"value": v, "unit": "Gpoints/s", "cores": cores, "kind": "port",
                             "sample": sample + " per step"},
            "e2e": {"value": v, "unit": "Gpoints/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1404_5756_b200 as P
    from paper_1404_5756_b200 import synth

    cfg = synth.make_config(args.config, nlev=args.nlev)
    k = args.k or (5 if args.order == 1 else 1)
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    w = 8 if args.dtype == "f64" else 4
    grid = P.Grid2D(cfg.nx, cfg.ny, cfg.dx, cfg.dy, cfg.mask)
    opts = P.CovarianceOptions(order=P.FilterOrder(args.order), k_iterations=k, device=local)
    t0 = time.perf_counter()
    op = P.HorizontalCovarianceOp(grid, P.ScaleField(cfg.rx, cfg.ry), opts)
    build_s = time.perf_counter() - t0
    shape = (cfg.nvar, cfg.nlev, cfg.ny, cfg.nx)
    gen = torch.Generator(device="cuda").manual_seed(1000 + rank)
    x = torch.randn(shape, generator=gen, device="cuda", dtype=torch.float64).to(tdt)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    def step():
        op.apply(P.GYGX, x, y)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = op.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = op.launch_count() - l0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    n_rank = cfg.nx * cfg.ny * cfg.nlev * cfg.nvar
    value = n_rank * world / (ms * 1e-3) / 1e9

    # final gather of the result into rank 0's field over NCCL (outside the
    # timed region; levels need no other exchange)
    gather = None
    if world > 1:
        from paper_1404_5756_b200.sharding import gather_levels
        torch.cuda.synchronize()
        dist.barrier()
        g0 = time.perf_counter()
        full = gather_levels(y, cfg.nlev * world)
        torch.cuda.synchronize()
        gather = {"ms": (time.perf_counter() - g0) * 1e3, "bytes": n_rank * w * world,
                  "timing": "host wall clock, NCCL gather to rank 0 (not in value)"}
        del full

    # per-kernel timing of the two directional sweeps (dominant kernel)
    sweep_ms = {}
    for name, kind in (("x", P.GX), ("y", P.GY)):
        for _ in range(2):
            op.apply(kind, x, y)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        reps = max(3, args.steps // 2)
        for _ in range(reps):
            op.apply(kind, x, y)
        b.record(stream)
        torch.cuda.synchronize()
        sweep_ms[name] = a.elapsed_time(b) / reps
    dom = max(sweep_ms, key=sweep_ms.get)
    peak, peak_src = peaks()
    nh = cfg.nx * cfg.ny
    coef_words = 4 if args.order == 3 else 2  # per direction (coefficient_bytes()/2)
    bytes_sweep = n_rank * 2 * w + nh * coef_words * 8
    achieved = bytes_sweep / (sweep_ms[dom] * 1e-3) / 1e9
    bytes_xy = synth.bytes_alg(cfg, args.order, w)
    xy_gbs = bytes_xy / (ms * 1e-3) / 1e9

    # e2e through the public API with pinned host buffers
    e2e = None
    if args.e2e_steps > 0:
        hx = torch.empty(shape, dtype=tdt, pin_memory=True)
        hx.copy_(x)
        hy = torch.empty(shape, dtype=tdt, pin_memory=True)
        hxn, hyn = hx.numpy(), hy.numpy()
        op.apply(P.GYGX, hxn)  # warm the host-path buffers
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            res = op.apply(P.GYGX, hxn, out=hyn)
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        del res
        e2e = {"value": n_rank * world / e2e_s / 1e9, "unit": "Gpoints/s",
               "h2d_bytes_per_step": n_rank * w * world, "d2h_bytes_per_step": n_rank * w * world,
               "steps": args.e2e_steps, "timing": "host wall clock around the synchronous "
               "rgf_op_apply(RGF_HOST) call (pinned buffers; H2D + kernels + D2H)"}

    # Other figures BASELINE.json's metric names (1st-RF, fp32, the adjoint):
    # same config and timing method (device-resident, CUDA events, warm-up),
    # reported beside the headline, not in `value`.
    extra = {}
    if world == 1 and args.order == 3 and args.dtype == "f64" and not args.no_extra:
        def timed(op2, kind, x2, y2, reps=3):
            for _ in range(2):
                op2.apply(kind, x2, y2)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(stream)
            for _ in range(reps):
                op2.apply(kind, x2, y2)
            b.record(stream)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps

        def entry(m2, order2, w2):
            ba = synth.bytes_alg(cfg, order2, w2)
            return {"ms": m2, "Gpt/s": n_rank / (m2 * 1e-3) / 1e9,
                    "xy_frac": ba / (m2 * 1e-3) / 1e9 / peaks()[0]}

        m_adj = timed(op, P.VT, x, y)
        extra["3rd-RF adjoint VT f64"] = entry(m_adj, 3, 8)
        for label, o2, k2, dt2, w2 in (("1st-RF K=5 f64", 1, 5, torch.float64, 8),
                                       ("3rd-RF f32", 3, 1, torch.float32, 4)):
            op2 = P.HorizontalCovarianceOp(grid, P.ScaleField(cfg.rx, cfg.ry),
                                           P.CovarianceOptions(order=P.FilterOrder(o2),
                                                               k_iterations=k2, device=local))
            x2 = x.to(dt2)
            y2 = torch.empty_like(x2)
            extra[label] = entry(timed(op2, P.GYGX, x2, y2), o2, w2)
            del op2, x2, y2
        extra["t(1st-RF K=5)/t(3rd-RF)"] = extra["1st-RF K=5 f64"]["ms"] / ms

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, sample, cores = cpu_port_rate(cfg, args.order, k, args.cpu_seconds)
        cpu = {"value": v, "unit": "Gpoints/s", "cores": cores, "kind": "port",
               "sample": sample}

    if rank == 0:
        line = {
            "metric": metric_name(args.order, k), "value": value, "unit": "Gpoints/s",
            "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": f"{args.config} ({cfg.description}) x+y apply_gy.apply_gx, "
                       f"order={args.order} k={k}, levels sharded ({cfg.nlev} per rank)",
                       "nx": cfg.nx, "ny": cfg.ny, "nlev_per_rank": cfg.nlev, "nvar": cfg.nvar,
                       "l2": "inputs larger than L2 (field >> 126 MB)",
                       "options": "unit_dc=1 yvv95 ghost=ceil(9 max sigma) per level"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": measured_traffic(args.config, args.dtype, args.order,
                                                     f"{dom}-sweep"),
                         "kernel": f"{dom}-sweep", "peak_source": peak_src,
                         "bytes_per_launch": bytes_sweep,
                         "xy_bytes_alg_GBs": xy_gbs, "xy_frac": xy_gbs / peak,
                         # BASELINE.json north_star quotes B200's ~8 TB/s nominal
                         "xy_frac_vs_nominal_8000": xy_gbs / 8000.0},
            "sweep_ms": sweep_ms,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "build_seconds": build_s,
        }
        if gather:
            line["gather"] = gather
        if extra:
            line["extra"] = extra
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
