"""Level sharding across ranks.

Levels are independent 2-D problems: each has its own mask, segments and
ghost width, and a level's result does not depend on which other levels share
the operator (coefficients at land points are never read, covariance.cpp:303-
310; ghost width and the uniform fast path are per level, covariance.cpp:173-
216). So a field [var][lev][iy][ix] shards over contiguous level ranges with
no collective on the data path; the only exchange is the final gather of the
result into one host field (NCCL over NVLink on GPUs, gloo in the CPU tests).

One process per GPU; ranks come from torch.distributed.
"""
from __future__ import annotations

import dataclasses

import numpy as np


def level_range(nlev: int, world: int, rank: int, costs=None) -> tuple[int, int]:
    """Contiguous level block of `rank`: (first level, count).

    Without `costs`: sizes differ by at most one; ranks beyond nlev get an
    empty block. With per-level `costs` (e.g. `level_costs`): the contiguous
    partition in rank order that minimises the largest block cost (SURVEY
    §8e: C2's land fraction rises 35 -> 70 % with depth, so equal level counts
    are not equal work for the segment-bound kernels)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("level_range: need 0 <= rank < world")
    if costs is None:
        base, extra = divmod(nlev, world)
        count = base + (1 if rank < extra else 0)
        first = rank * base + min(rank, extra)
        return first, count
    c = np.asarray(costs, dtype=np.float64)
    if c.shape != (nlev,) or np.any(c < 0):
        raise ValueError("level_range: costs must be nlev non-negative numbers")
    bounds = _balanced_bounds(c, world)
    return bounds[rank], bounds[rank + 1] - bounds[rank]


def _balanced_bounds(c, world):
    """Block starts (world + 1 entries) of the min-max contiguous partition:
    binary search on the bottleneck over the prefix sums, then a greedy cut
    that leaves enough levels for the remaining ranks."""
    n = len(c)
    pre = np.concatenate([[0.0], np.cumsum(c)])

    def cuts(cap):
        b = [0]
        for r in range(world - 1):
            lo = b[-1]
            # furthest end with block cost <= cap
            hi = int(np.searchsorted(pre, pre[lo] + cap, side="right")) - 1
            b.append(min(max(hi, lo), n))
        b.append(n)
        return b

    lo, hi = float(np.max(c)) if n else 0.0, float(pre[-1])
    for _ in range(100):
        mid = 0.5 * (lo + hi)
        b = cuts(mid)
        if pre[b[-1]] - pre[b[-2]] <= mid * (1 + 1e-12):
            hi = mid
        else:
            lo = mid
    return cuts(hi)


def level_costs(mask, ghost_width) -> np.ndarray:
    """Per-level work estimate for level_range(costs=...): sea points plus
    the ghost-extended steps of every segment end in both sweep directions
    (covariance.cpp:246-273: each segment meeting land is padded by G)."""
    m = np.asarray(mask, dtype=bool)
    if m.ndim == 2:
        m = m[None]
    g = np.broadcast_to(np.asarray(ghost_width, dtype=np.float64), (m.shape[0],))
    sea = m.sum(axis=(1, 2)).astype(np.float64)
    ends_x = (m[:, :, :-1] & ~m[:, :, 1:]).sum(axis=(1, 2))
    ends_y = (m[:, :-1, :] & ~m[:, 1:, :]).sum(axis=(1, 2))
    return sea * 2.0 + g * (ends_x + ends_y)


def shard_grid_arrays(mask, variance, nlev: int, world: int, rank: int, costs=None):
    """Slice the per-level inputs of a global operator for one rank: the mask
    (nlev, ny, nx) or a shared 2-D mask, and the optional variance."""
    l0, n = level_range(nlev, world, rank, costs)
    m = np.asarray(mask)
    if m.ndim == 3:
        m = m[l0:l0 + n]
    v = None
    if variance is not None:
        v = np.asarray(variance)
        v = v[l0:l0 + n] if v.ndim == 3 else v
    return l0, n, m, v


class ShardedCovarianceOp:
    """This rank's part of a global HorizontalCovarianceOp: the operator over
    its level block, with the global grid's horizontal arrays. apply() takes
    and returns the rank-local slice [var][local lev][iy][ix]."""

    def __init__(self, nx, ny, dx, dy, mask, rx, ry, options=None, *, nlev, world, rank,
                 variance=None, costs=None):
        from . import CovarianceOptions, Grid2D, HorizontalCovarianceOp, ScaleField

        self.nlev, self.world, self.rank = nlev, world, rank
        self.costs = costs
        self.lev0, self.nlev_local, m, v = shard_grid_arrays(mask, variance, nlev, world, rank,
                                                             costs)
        opts = options or CovarianceOptions()
        if v is not None:
            opts = dataclasses.replace(opts, variance=v)
        self.op = None
        if self.nlev_local > 0:
            self.op = HorizontalCovarianceOp(Grid2D(nx, ny, dx, dy, m), ScaleField(rx, ry), opts)

    def local_slice(self, field):
        """The rank's levels of a global field [var][lev][iy][ix]."""
        return field[:, self.lev0:self.lev0 + self.nlev_local]

    def apply(self, kind, local_field, out=None, stream=None):
        if self.op is None:
            return local_field if out is None else out
        return self.op.apply(kind, local_field, out=out, stream=stream)


def gather_levels(local, nlev: int, out=None, group=None, dst: int = 0, costs=None):
    """Gather every rank's level block [var][nlev_local][ny][nx] (torch tensor
    on the rank's device for NCCL, or on CPU for gloo) into the full field
    [var][nlev][ny][nx] on rank `dst` (into `out` if given). Other ranks
    return None. One grouped point-to-point exchange (batch_isend_irecv: a
    single ncclGroupStart/End on NCCL), blocks received straight into their
    slice of the output when it is contiguous on the same device. `costs`
    must be the partition the ranks were sharded with."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if rank != dst:
        if local.shape[1] > 0:  # matches the receiver's skip of empty blocks
            reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, local.contiguous(),
                                                      _peer(dst, group), group)])
            for r in reqs:
                r.wait()
        return None
    nvar, _, ny, nx = local.shape
    if out is None:
        out = torch.empty((nvar, nlev, ny, nx), dtype=local.dtype, device=local.device)
    ops, staged = [], []
    for r in range(world):
        l0, n = level_range(nlev, world, r, costs)
        if r == rank:
            out[:, l0:l0 + n].copy_(local)
            continue
        if n == 0:
            continue
        view = out[:, l0:l0 + n]
        if view.is_contiguous() and view.device == local.device:
            buf = view
        else:
            buf = torch.empty((nvar, n, ny, nx), dtype=local.dtype, device=local.device)
            staged.append((view, buf))
        ops.append(dist.P2POp(dist.irecv, buf, _peer(r, group), group))
    if ops:
        for q in dist.batch_isend_irecv(ops):
            q.wait()
    for view, buf in staged:
        view.copy_(buf)
    return out


def _peer(r, group):
    """Global rank of group rank r (P2POp takes global ranks)."""
    import torch.distributed as dist
    return r if group is None else dist.get_global_rank(group, r)
