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


def level_range(nlev: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced level block of `rank`: (first level, count).
    Sizes differ by at most one; ranks beyond nlev get an empty block."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("level_range: need 0 <= rank < world")
    base, extra = divmod(nlev, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, count


def shard_grid_arrays(mask, variance, nlev: int, world: int, rank: int):
    """Slice the per-level inputs of a global operator for one rank: the mask
    (nlev, ny, nx) or a shared 2-D mask, and the optional variance."""
    l0, n = level_range(nlev, world, rank)
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
                 variance=None):
        from . import CovarianceOptions, Grid2D, HorizontalCovarianceOp, ScaleField

        self.nlev, self.world, self.rank = nlev, world, rank
        self.lev0, self.nlev_local, m, v = shard_grid_arrays(mask, variance, nlev, world, rank)
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


def gather_levels(local, nlev: int, out=None, group=None, dst: int = 0):
    """Gather every rank's level block [var][nlev_local][ny][nx] (torch tensor
    on the rank's device for NCCL, or on CPU for gloo) into the full field
    [var][nlev][ny][nx] on rank `dst` (into `out` if given, e.g. a pinned
    host tensor). Other ranks return None. Point-to-point, one block at a
    time, so rank `dst` never holds more than the field plus one block."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if rank != dst:
        if local.shape[1] > 0:  # matches the receiver's skip of empty blocks
            dist.send(local.contiguous(), dst=dst, group=group)
        return None
    nvar, _, ny, nx = local.shape
    if out is None:
        out = torch.empty((nvar, nlev, ny, nx), dtype=local.dtype, device=local.device)
    for r in range(world):
        l0, n = level_range(nlev, world, r)
        if r == rank:
            out[:, l0:l0 + n].copy_(local)
            continue
        if n == 0:
            continue
        view = out[:, l0:l0 + n]
        if view.is_contiguous() and view.device == local.device:
            dist.recv(view, src=r, group=group)
        else:
            tmp = torch.empty((nvar, n, ny, nx), dtype=local.dtype, device=local.device)
            dist.recv(tmp, src=r, group=group)
            view.copy_(tmp)
    return out
