"""Level sharding on CPU: the partition, and a world_size-2
gloo run in which each rank filters its level block (the oracle stands in for
the GPU) and the blocks are gathered to rank 0. The result must equal the
unsharded operator bit for bit, because levels are independent 2-D problems."""
import os
import socket
import tempfile

import numpy as np
import pytest

import oracle as O
from helpers import checkered_mask, uniform_grid
from paper_1404_5756_b200.sharding import (gather_levels, level_costs, level_range,
                                           shard_grid_arrays)

NX, NY, NLEV, NVAR = 40, 30, 5, 2


def case():
    rng = np.random.default_rng(31)
    g = uniform_grid(NX, NY, 5000.0, 6000.0, nlev=NLEV)
    g["mask"] = checkered_mask(NX, NY, 32, 0.75, nlev=NLEV)
    rx = g["dx"] * rng.uniform(1.5, 4.0, (NY, NX))
    ry = g["dy"] * rng.uniform(1.5, 4.0, (NY, NX))
    var = rng.uniform(0.5, 2.0, (NLEV, NY, NX))
    f = rng.standard_normal((NVAR, NLEV, NY, NX))
    return g, rx, ry, var, f


def full_result(kind):
    g, rx, ry, var, f = case()
    op = O.OracleOp(NX, NY, g["dx"], g["dy"], g["mask"], rx, ry, variance=var, threads=1)
    return op.apply(kind, f)


@pytest.mark.parametrize("nlev,world", [(5, 2), (100, 8), (7, 3), (3, 4), (1, 1), (75, 8)])
def test_level_range_partitions(nlev, world):
    seen, sizes = [], []
    for r in range(world):
        l0, n = level_range(nlev, world, r)
        assert n >= 0
        seen.extend(range(l0, l0 + n))
        sizes.append(n)
    assert seen == list(range(nlev))  # contiguous, disjoint, in rank order, complete
    assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, out_path, kind, balanced=False):
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    g, rx, ry, var, f = case()
    costs = level_costs(g["mask"], 36) if balanced else None
    l0, n, m, v = shard_grid_arrays(g["mask"], var, NLEV, world, rank, costs)
    if n == 0:  # more ranks than levels: nothing to filter, still take part
        full = gather_levels(torch.zeros((NVAR, 0, NY, NX), dtype=torch.float64), NLEV,
                             costs=costs)
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.destroy_process_group()
        return
    op = O.OracleOp(NX, NY, g["dx"], g["dy"], m, rx, ry, variance=v, threads=1)
    local = op.apply(kind, np.ascontiguousarray(f[:, l0:l0 + n]))
    full = gather_levels(torch.from_numpy(local), NLEV, costs=costs)
    # max-over-ranks aggregation of a per-rank time, as bench.py does
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        assert float(t.item()) == float(world)
        np.save(out_path, full.numpy())
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("kind,world,balanced", [(O.GYGX, 2, False), (O.V, 2, False),
                                                (O.B, 2, False), (O.GYGX, 6, False),
                                                (O.GYGX, 2, True), (O.VT, 3, True)])
def test_gloo_sharded_equals_unsharded(kind, world, balanced):
    """world 2 (the multi-GPU path's shape) and world 6 > 5 levels (a rank
    with no levels)."""
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "full.npy")
        mp.spawn(_worker, args=(world, _free_port(), out, kind, balanced), nprocs=world,
                 join=True)
        got = np.load(out)
    want = full_result(kind)
    assert got.shape == want.shape
    assert np.array_equal(got, want)


@pytest.mark.parametrize("seed,nlev,world", [(1, 5, 2), (2, 12, 3), (3, 9, 4), (4, 3, 5),
                                             (5, 72, 8), (6, 1, 1)])
def test_cost_balanced_partition_is_optimal(seed, nlev, world):
    """Contiguous, complete, in rank order, and the bottleneck equals the
    brute-force optimum (small cases) / never worse than equal counts."""
    import itertools
    rng = np.random.default_rng(seed)
    costs = rng.uniform(1.0, 3.0, nlev)
    blocks = [level_range(nlev, world, r, costs) for r in range(world)]
    seen = [lv for l0, n in blocks for lv in range(l0, l0 + n)]
    assert seen == list(range(nlev))
    worst = max(costs[l0:l0 + n].sum() for l0, n in blocks)
    even = max(costs[l0:l0 + n].sum() for l0, n in
               (level_range(nlev, world, r) for r in range(world)))
    assert worst <= even + 1e-9
    if nlev <= 12:
        best = np.inf
        for cut in itertools.combinations(range(nlev + 1), world - 1):
            b = (0,) + cut + (nlev,)
            if any(b[i] > b[i + 1] for i in range(world)):
                continue
            best = min(best, max(costs[b[i]:b[i + 1]].sum() for i in range(world)))
        assert worst <= best * (1 + 1e-9)


def test_level_costs_track_land_fraction():
    """C2-like nested masks: deeper levels (more land, shorter segments) get a
    different cost, and a cost-balanced split differs from equal counts."""
    from paper_1404_5756_b200 import synth
    cfg = synth.make_config("C2", nx=200, ny=80)
    c = level_costs(cfg.mask, 72)
    assert c.shape == (cfg.nlev,)
    assert c[0] != c[-1]
    assert [level_range(cfg.nlev, 8, r, c) for r in range(8)] != \
        [level_range(cfg.nlev, 8, r) for r in range(8)]
