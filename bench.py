#!/usr/bin/env python
"""Benchmark of the x+y recursive-filter application (apply_gy . apply_gx,
diagnostics.cpp:182's timed unit) on synthetic BASELINE.json grids.

Default workload: config C5 (4320x2160x100 levels, fp64, 3rd-RF, reference
default options: unit_dc, YvV95, ghost width ceil(9 max sigma)). Under
torchrun (N>1) the 100 levels are sharded across ranks (strong scaling,
SURVEY §8e / BASELINE configs[4]): each rank filters its contiguous level
block with no collective on the data path; the result is gathered to rank 0
afterwards with grouped NCCL point-to-point (reported as `gather`, not in
`value`). `--scaling weak` gives every rank the full level set instead.
Prints ONE JSON line on rank 0.

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
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N>1: shard the config's levels (strong) or replicate them (weak)")
    ap.add_argument("--ref-budget-s", type=float, default=420.0,
                    help="reference arm: whole-run CPU budget; above it each step times a "
                         "level sample instead of the full level set")
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
            self.rows.append([x.strip() for x in line.split(",")] + [time.perf_counter()])

    def mark(self, start=True):
        """Host time of the timed region's start / end: the summary keeps the
        samples read inside it (the sampler runs from before the warm-up so
        nvidia-smi's start-up does not eat the region)."""
        if start:
            self.t0 = time.perf_counter()
        else:
            self.t1 = time.perf_counter()

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        t0, t1 = getattr(self, "t0", None), getattr(self, "t1", None)
        rows = self.rows
        if t0 is not None and t1 is not None:
            inside = [r for r in rows if t0 <= r[-1] <= t1 + 0.05]
            rows = inside or rows[-1:]
        rows = [r[:-1] for r in rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


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


def load_synth():
    """paper_1404_5756_b200/synth.py as a standalone module: the input
    generators without the package (whose import maps librgf_b200.so), so the
    reference arm's process never loads the product library."""
    import importlib.util
    path = os.path.join(ROOT, "paper_1404_5756_b200", "synth.py")
    spec = importlib.util.spec_from_file_location("rgf_bench_synth", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod
    spec.loader.exec_module(mod)
    return mod


def workload_config(args, cfg, k):
    """The `config` object, identical for both arms and every N."""
    return {"workload": f"{args.config} ({cfg.description}) x+y apply_gy.apply_gx, "
                        f"order={args.order} k={k}",
            "nx": cfg.nx, "ny": cfg.ny, "nlev": cfg.nlev, "nvar": cfg.nvar,
            "l2": "inputs larger than L2 (field >> 126 MB)",
            "options": "unit_dc=1 yvv95 ghost=ceil(9 max sigma) per level"}


class CpuPort:
    """The oracle (C++ restatement of the reference) on `threads` host
    threads over levels [0, nl) of the same workload: the operator and the
    input field are built once; each run() times one x+y application."""

    def __init__(self, cfg, order, k, threads, nl):
        import oracle as O
        self.O = O
        self.threads = threads
        self.op = O.OracleOp(cfg.nx, cfg.ny, cfg.dx, cfg.dy, cfg.mask, cfg.rx, cfg.ry,
                             order=order, k_iterations=k, threads=threads)
        self.nl = max(1, min(cfg.nlev, nl))
        self.f = np.random.default_rng(99).standard_normal((cfg.nvar, self.nl, cfg.ny, cfg.nx))
        self.pts = cfg.nx * cfg.ny * self.nl * cfg.nvar
        self.sample = (f"{self.nl} of {cfg.nlev} levels x {cfg.nvar} var ({self.pts} points), "
                       f"1 x+y application")

    def run(self):
        """(Gpt/s, seconds) of one timed application."""
        t0 = time.perf_counter()
        self.op.apply(self.O.GYGX, self.f, lev0=0, nlev_sub=self.nl)
        dt = time.perf_counter() - t0
        return self.pts / dt / 1e9, dt


def levels_for(cfg, order, k, threads, seconds):
    """Levels of `cfg` one application covers in about `seconds`."""
    probe = CpuPort(cfg, order, k, threads, 1)
    probe.run()
    _, t1 = probe.run()
    return max(1, min(cfg.nlev, int(seconds / max(t1, 1e-6)))), t1


def cpu_baselines(cfg, order, k, seconds):
    """cpu_baseline (all host threads, ~`seconds` of work) and the
    single-thread figure BASELINE.md §3 asks for (test_output.txt:16)."""
    cores = os.cpu_count() or 1
    nl, _ = levels_for(cfg, order, k, cores, seconds)
    cp = CpuPort(cfg, order, k, cores, nl)
    v, _ = cp.run()
    one = CpuPort(cfg, order, k, 1, 1)
    v1, _ = one.run()
    return ({"value": v, "unit": "Gpoints/s", "cores": cores, "kind": "port",
             "sample": cp.sample},
            {"value": v1, "unit": "Gpoints/s", "cores": 1, "kind": "port",
             "sample": one.sample})


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU algorithm on every host thread.
    The reference cannot be built here (Eigen3/CLI11/doctest absent), so this
    is the oracle port (oracle/, a line-by-line restatement pinned to the
    reference's golden vectors). Each step is one timed x+y application over
    the whole config (all levels) unless (warmup+steps) of those would exceed
    --ref-budget-s; then each step covers a level sample and the line says so.
    ms_per_step is the measured time of one step either way."""
    if rank != 0:
        return
    synth = load_synth()
    cfg = synth.make_config(args.config, nlev=args.nlev)
    k = args.k or (5 if args.order == 1 else 1)
    cores = os.cpu_count() or 1
    _, t1 = levels_for(cfg, args.order, k, cores, 1.0)
    runs = args.warmup + args.steps
    nl = cfg.nlev
    if runs * t1 * cfg.nlev > args.ref_budget_s:
        nl = max(1, int(args.ref_budget_s / (runs * t1)))
    cp = CpuPort(cfg, args.order, k, cores, nl)
    rates, secs = [], []
    for i in range(runs):
        r, dt = cp.run()
        if i >= args.warmup:
            rates.append(r)
            secs.append(dt)
    v = cp.pts * len(secs) / sum(secs) / 1e9
    one = CpuPort(cfg, args.order, k, 1, 1)
    v1, _ = one.run()
    line = {"impl": "reference", "metric": metric_name(args.order, k),
            "value": v, "unit": "Gpoints/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.mean(secs) * 1e3,
            "higher_is_better": True, "scaling": "strong" if args.scaling == "strong" else "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": workload_config(args, cfg, k),
            "cpu_baseline": {"value": v, "unit": "Gpoints/s", "cores": cores, "kind": "port",
                             "sample": cp.sample + " per step" +
                             ("" if nl == cfg.nlev else " (level sample: full set over budget)")},
            "cpu_baseline_1thread": {"value": v1, "unit": "Gpoints/s", "cores": 1,
                                     "kind": "port", "sample": one.sample},
            "note": "the oracle computes in fp64 whatever --dtype says (the reference has no "
                    "fp32 operator, types.hpp:14)",
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
    from paper_1404_5756_b200.sharding import (ShardedCovarianceOp, gather_levels,
                                               level_range)

    cfg = synth.make_config(args.config, nlev=args.nlev)
    k = args.k or (5 if args.order == 1 else 1)
    tdt = torch.float64 if args.dtype == "f64" else torch.float32
    w = 8 if args.dtype == "f64" else 4
    strong = args.scaling == "strong"
    # this rank's level block: a contiguous shard (strong) or all levels (weak)
    sw, sr = (world, rank) if strong else (1, 0)
    opts = P.CovarianceOptions(order=P.FilterOrder(args.order), k_iterations=k, device=local)
    t0 = time.perf_counter()
    sop = ShardedCovarianceOp(cfg.nx, cfg.ny, cfg.dx, cfg.dy, cfg.mask, cfg.rx, cfg.ry, opts,
                              nlev=cfg.nlev, world=sw, rank=sr)
    build_s = time.perf_counter() - t0
    nl_local = sop.nlev_local
    shape = (cfg.nvar, nl_local, cfg.ny, cfg.nx)
    gen = torch.Generator(device="cuda").manual_seed(1000 + rank)
    x = torch.randn(shape, generator=gen, device="cuda", dtype=torch.float64).to(tdt)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()

    def step():
        sop.apply(P.GYGX, x, y)

    def launches_now():
        return sop.op.launch_count() if sop.op is not None else 0

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        l0 = launches_now()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clk.mark(True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
        if world > 1:
            dist.barrier()
    launches = launches_now() - l0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        lt = torch.tensor([launches], device="cuda", dtype=torch.float64)
        dist.all_reduce(lt)
        launches = int(lt.item())
    n_local = cfg.nx * cfg.ny * nl_local * cfg.nvar
    n_total = cfg.nx * cfg.ny * cfg.nlev * cfg.nvar * (1 if strong else world)
    value = n_total / (ms * 1e-3) / 1e9

    # final gather of the result into rank 0's field over NCCL (outside the
    # timed region; levels need no other exchange), device-timed, max over ranks
    gather = None
    if world > 1:
        nlev_all = cfg.nlev * (1 if strong else world)
        torch.cuda.synchronize()
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        full = gather_levels(y, nlev_all)
        g1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([g0.elapsed_time(g1)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        gms = float(t.item())
        gather = {"ms": gms, "bytes_into_rank0": (n_total - n_local) * w,
                  "compute_plus_gather_ms": ms + gms,
                  "timing": "CUDA events around grouped NCCL send/recv to rank 0, max over "
                            "ranks (not in value)"}
        del full

    # per-kernel timing of the two directional sweeps (dominant kernel)
    sweep_ms = {}
    if sop.op is not None:
        for name, kind in (("x", P.GX), ("y", P.GY)):
            for _ in range(2):
                sop.apply(kind, x, y)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            reps = max(3, args.steps // 2)
            for _ in range(reps):
                sop.apply(kind, x, y)
            b.record(stream)
            torch.cuda.synchronize()
            sweep_ms[name] = a.elapsed_time(b) / reps
    dom = max(sweep_ms, key=sweep_ms.get) if sweep_ms else "y"
    peak, peak_src = peaks()
    nh = cfg.nx * cfg.ny
    coef_words = 4 if args.order == 3 else 2  # per direction (coefficient_bytes()/2)
    bytes_sweep = n_local * 2 * w + nh * coef_words * 8
    achieved = bytes_sweep / (sweep_ms[dom] * 1e-3) / 1e9 if sweep_ms else 0.0
    bytes_xy = synth.bytes_alg(cfg, args.order, w) * (1 if strong else world)
    xy_gbs = bytes_xy / (ms * 1e-3) / 1e9 / world  # per GPU

    # e2e through the public API with pinned host buffers: every rank moves
    # its own levels host->device->host (direct per-GPU D2H)
    e2e = None
    if args.e2e_steps > 0:
        hx = torch.empty(shape, dtype=tdt, pin_memory=True)
        hx.copy_(x)
        hy = torch.empty(shape, dtype=tdt, pin_memory=True)
        hxn, hyn = hx.numpy(), hy.numpy()
        if sop.op is not None:
            sop.apply(P.GYGX, hxn, out=hyn)  # warm the host-path buffers
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            if sop.op is not None:
                sop.apply(P.GYGX, hxn, out=hyn)
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": n_total / e2e_s / 1e9, "unit": "Gpoints/s",
               "h2d_bytes_per_step": n_total * w, "d2h_bytes_per_step": n_total * w,
               "steps": args.e2e_steps, "timing": "host wall clock around the synchronous "
               "rgf_op_apply(RGF_HOST) call (pinned buffers; H2D + kernels + D2H), max over ranks"}

    # Other figures BASELINE.json's metric names (1st-RF, fp32, the adjoint):
    # same config and timing method (device-resident, CUDA events, warm-up),
    # reported beside the headline, not in `value`.
    extra = {}
    if world == 1 and args.order == 3 and args.dtype == "f64" and not args.no_extra:
        grid = P.Grid2D(cfg.nx, cfg.ny, cfg.dx, cfg.dy, cfg.mask)

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
            return {"ms": m2, "Gpt/s": n_local / (m2 * 1e-3) / 1e9,
                    "xy_frac": ba / (m2 * 1e-3) / 1e9 / peaks()[0]}

        m_adj = timed(sop.op, P.VT, x, y)
        extra["3rd-RF adjoint VT f64"] = entry(m_adj, 3, 8)
        for o2, k2, cases in ((1, 5, (("1st-RF K=5 f64", torch.float64, 8, P.GYGX),
                                       ("1st-RF K=5 adjoint VT f64", torch.float64, 8, P.VT),
                                       ("1st-RF K=5 f32", torch.float32, 4, P.GYGX))),
                              (3, 1, (("3rd-RF f32", torch.float32, 4, P.GYGX),))):
            op2 = P.HorizontalCovarianceOp(grid, P.ScaleField(cfg.rx, cfg.ry),
                                           P.CovarianceOptions(order=P.FilterOrder(o2),
                                                               k_iterations=k2, device=local))
            for label, dt2, w2, kind2 in cases:
                x2 = x.to(dt2)
                y2 = torch.empty_like(x2)
                extra[label] = entry(timed(op2, kind2, x2, y2), o2, w2)
                del x2, y2
            del op2
        extra["t(1st-RF K=5)/t(3rd-RF)"] = extra["1st-RF K=5 f64"]["ms"] / ms

    cpu = cpu1 = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, cpu1 = cpu_baselines(cfg, args.order, k, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": metric_name(args.order, k), "value": value, "unit": "Gpoints/s",
            "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic",
            "config": workload_config(args, cfg, k),
            "sharding": {"mode": args.scaling, "levels_per_rank": [
                level_range(cfg.nlev, sw, r)[1] for r in range(sw)] if strong else cfg.nlev,
                "collective_on_data_path": False},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": measured_traffic(args.config, args.dtype, args.order,
                                                     f"{dom}-sweep"),
                         "kernel": f"{dom}-sweep", "peak_source": peak_src,
                         "bytes_per_launch": bytes_sweep,
                         "xy_bytes_alg_GBs_per_gpu": xy_gbs, "xy_frac": xy_gbs / peak,
                         # BASELINE.json north_star quotes B200's ~8 TB/s nominal
                         "xy_frac_vs_nominal_8000": xy_gbs / 8000.0},
            "sweep_ms": sweep_ms,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "cpu_baseline_1thread": cpu1,
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
