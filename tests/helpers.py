"""Shared test helpers: grid builders, independent segment enumeration, dense
assembly, error norms. Arrays are (nlev, ny, nx) / (ny, nx), x fastest."""
import numpy as np


def uniform_grid(nx, ny, dx=6000.0, dy=6000.0, nlev=1):
    return dict(nx=nx, ny=ny, dx=np.full((ny, nx), dx), dy=np.full((ny, nx), dy),
                mask=np.ones((nlev, ny, nx), dtype=bool))


def checkered_mask(nx, ny, seed, sea_frac, nlev=1):
    """test_covariance.cpp:34-41 analogue (numpy RNG; not mt19937-identical)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(size=(nlev, ny, nx)) < sea_frac


def segments_reference(line_mask):
    """covariance.cpp:246-258 maximal sea runs -> list of (start, len)."""
    out = []
    n = len(line_mask)
    i = 0
    while i < n:
        if not line_mask[i]:
            i += 1
            continue
        j = i
        while j + 1 < n and line_mask[j + 1]:
            j += 1
        out.append((i, j - i + 1))
        i = j + 1
    return out


def segments_numpy(mask3, direction):
    """Vectorised run detection: offsets[nlines+1], segs[nsegs,2] in the
    C ABI's line order (dir 0: lev*ny+iy rows; dir 1: lev*nx+ix columns)."""
    m = np.asarray(mask3, dtype=bool)
    if direction == 0:
        lines = m.reshape(-1, m.shape[2])
    else:
        lines = np.transpose(m, (0, 2, 1)).reshape(-1, m.shape[1])
    nl, n = lines.shape
    pad = np.zeros((nl, n + 2), dtype=np.int8)
    pad[:, 1:-1] = lines
    d = np.diff(pad, axis=1)
    sl, sc = np.nonzero(d == 1)
    el, ec = np.nonzero(d == -1)
    assert np.array_equal(sl, el)
    counts = np.bincount(sl, minlength=nl)
    off = np.zeros(nl + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    segs = np.stack([sc, ec - sc], axis=1).astype(np.int32)
    return off, segs


def relmax(got, want):
    """Relative max-norm error ||got-want||_inf / ||want||_inf (north_star)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = np.max(np.abs(want))
    num = np.max(np.abs(got - want))
    return float(num / den) if den > 0 else float(num)


def assemble_dense(nx, ny, apply):
    """oracles.hpp:105-117: column c = apply(e_c), x-fastest indexing."""
    n = nx * ny
    m = np.zeros((n, n))
    for col in range(n):
        e = np.zeros((ny, nx))
        e.flat[col] = 1.0
        m[:, col] = np.asarray(apply(e)).reshape(-1)
    return m


def halfwidth(line, c):
    hm = line[c] / 2.0
    i = c
    while line[i] > hm:
        i += 1
    return (i - 1 - c) + (line[i - 1] - hm) / (line[i - 1] - line[i])
