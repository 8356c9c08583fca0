"""Seeded synthetic inputs for the five BASELINE.json configurations.

The paper's real grids (Mediterranean 1742x506x72, global ORCA 1/4) and its
length-scale climatologies are not available; these generators stand in for
them with the shapes, land fractions and length-scale ranges BASELINE.json
names. Everything is a pure function of (config, seed).

Arrays are x fastest: dx, dy, rx, ry are (ny, nx); the mask is
(nlev, ny, nx) bool (True = sea); fields are (nvar, nlev, ny, nx).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class Config:
    name: str
    nx: int
    ny: int
    nlev: int
    nvar: int
    dx: np.ndarray
    dy: np.ndarray
    mask: np.ndarray  # (nlev, ny, nx) bool
    rx: np.ndarray
    ry: np.ndarray
    description: str

    @property
    def n_points(self) -> int:
        return self.nx * self.ny * self.nlev * self.nvar


def _smoothed_noise(rng, ny, nx, sigma):
    from scipy.ndimage import gaussian_filter
    return gaussian_filter(rng.standard_normal((ny, nx)), sigma=sigma, mode="reflect")


def _scaled(field, lo, hi):
    f = (field - field.min()) / (field.max() - field.min())
    return lo + (hi - lo) * f


def _nested_masks(noise, land_fracs):
    """sea = noise > quantile(land fraction), one mask per level (nested)."""
    qs = np.quantile(noise, land_fracs)
    return noise[None, :, :] > qs[:, None, None]


PRESETS = {
    # name: (nx, ny, nlev, nvar)
    "C1": (256, 128, 1, 1),
    "C2": (871, 253, 72, 1),
    "C3": (1442, 1021, 75, 1),
    "C4": (1442, 1021, 75, 2),
    "C5": (4320, 2160, 100, 1),
}


def make_config(name: str, seed: int = 1404, nlev: int | None = None, nx: int | None = None,
                ny: int | None = None) -> Config:
    """Build config `name` (C1..C5). nlev/nx/ny override the preset for
    reduced-size parity runs with the same generators."""
    pnx, pny, pnlev, nvar = PRESETS[name]
    nx = nx or pnx
    ny = ny or pny
    nlev = nlev or pnlev
    rng = np.random.default_rng(seed)
    if name == "C1":
        # 2-D all sea, dx=dy=1, L=4 grid spacings (BASELINE.json configs[0])
        dx = np.ones((ny, nx))
        dy = np.ones((ny, nx))
        mask = np.ones((nlev, ny, nx), dtype=bool)
        rx = np.full((ny, nx), 4.0)
        ry = np.full((ny, nx), 4.0)
        desc = "all sea, dx=dy=1, L=4 uniform"
    elif name == "C2":
        # Mediterranean-like: smoothed noise, land 35% at the surface rising
        # linearly to 70% at the bottom; L smooth in [3, 8] grid spacings.
        dx = np.full((ny, nx), 1.0)
        dy = np.full((ny, nx), 1.0)
        noise = _smoothed_noise(rng, ny, nx, 4.0)
        fr = 0.35 + 0.35 * np.arange(nlev) / max(pnlev - 1, 1)
        mask = _nested_masks(noise, fr)
        L = _scaled(_smoothed_noise(rng, ny, nx, 20.0), 3.0, 8.0)
        rx, ry = L * dx, L * dy
        desc = "smoothed-noise basin, land 35%->70% with depth, L in [3,8]"
    elif name in ("C3", "C4"):
        # global-like: lat in [-78, 90], dx = dx0 cos(lat), dy = dy0,
        # L = max(2, 6 cos lat) grid spacings, ~30% land in short segments.
        dx0, dy0 = 27750.0, 27750.0
        lat = -78.0 + (np.arange(ny) + 0.5) * (168.0 / ny)
        coslat = np.cos(np.deg2rad(lat))[:, None] * np.ones((1, nx))
        dx = dx0 * coslat
        dy = np.full((ny, nx), dy0)
        noise = _smoothed_noise(rng, ny, nx, 2.0)
        mask = np.repeat((noise > np.quantile(noise, 0.30))[None], nlev, axis=0)
        L = np.maximum(2.0, 6.0 * coslat)
        rx, ry = L * dx, L * dy
        desc = "tripolar-like lat grid, dx=dx0 cos(lat), 30% land, L=max(2,6cos(lat))"
    elif name == "C5":
        # 1/12 degree-like: 30% land, L smooth in [2, 10] grid spacings
        dx = np.full((ny, nx), 9250.0)
        dy = np.full((ny, nx), 9250.0)
        noise = _smoothed_noise(rng, ny, nx, 6.0)
        mask = np.repeat((noise > np.quantile(noise, 0.30))[None], nlev, axis=0)
        L = _scaled(_smoothed_noise(rng, ny, nx, 20.0), 2.0, 10.0)
        rx, ry = L * dx, L * dy
        desc = "1/12-deg-like, 30% land, L in [2,10]"
    else:
        raise ValueError(name)
    return Config(name, nx, ny, nlev, nvar, np.ascontiguousarray(dx), np.ascontiguousarray(dy),
                  np.ascontiguousarray(mask), np.ascontiguousarray(rx), np.ascontiguousarray(ry),
                  desc)


def make_field(cfg: Config, seed: int = 7, nvar: int | None = None, dtype=np.float64):
    """N(0,1) input per point per level per variable; C1 adds a unit impulse
    at the centre (BASELINE.json configs[0])."""
    nvar = nvar or cfg.nvar
    rng = np.random.default_rng(seed)
    f = rng.standard_normal((nvar, cfg.nlev, cfg.ny, cfg.nx))
    if cfg.name == "C1":
        f[:, :, cfg.ny // 2, cfg.nx // 2] += 1.0
    return f.astype(dtype)


def bytes_alg(cfg: Config, order: int, word: int, sigma_is_field: bool = True) -> int:
    """N*4*w + N_sigma*c*8, c = 8 (3rd-RF) | 4 (1st-RF)."""
    n = cfg.n_points
    n_sigma = cfg.nx * cfg.ny if sigma_is_field else 0
    c = 8 if order == 3 else 4
    return n * 4 * word + n_sigma * c * 8


def analytic_gaussian(n, c, sigma):
    i = np.arange(n)
    g = np.exp(-((i - c) ** 2) / (2 * sigma * sigma))
    return g / g.sum()


__all__ = ["Config", "PRESETS", "make_config", "make_field", "bytes_alg", "analytic_gaussian"]
del math
