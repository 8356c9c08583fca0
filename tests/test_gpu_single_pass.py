"""Single-pass sweeps (csrc/sweep_sp.cuh) against the oracle (gpu).

The single-pass x sweep runs when every level shares one mask (one mask
class, one ghost width): a row is cut into up to 16 chunks, one per CTA of a
thread-block cluster, and the chunks exchange 3-value entry states through
distributed shared memory. These cases stress what the chunking can break:
segments that cross one or many chunk boundaries (all-sea rows cross all of
them), segment ends and starts on the first / last points of a chunk, partial
last chunks and sub-tiles, rows whose byte length is not a 16 B multiple
(pitched device copies), planes that do not fill the 32 lanes, the plane
groups of 100 levels, every operator kind with and without unit-DC and
variance. Tolerance 1e-12 relative max-norm (fp64), land exactly 0.
Reference arithmetic: covariance.cpp:228-352 through oracle/rgf_oracle.cpp.
"""
import numpy as np
import pytest

import oracle as O
from helpers import relmax, uniform_grid

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
KINDS = ["GX", "GY", "GXT", "GYT", "V", "VT", "B", "GYGX"]


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1404_5756_b200 as P
    return P


def shared_mask(nx, ny, nlev, seed, sea=0.8, runs=False):
    rng = np.random.default_rng(seed)
    if runs:  # long sea runs (smoothed noise) -> segments spanning chunks
        from scipy.ndimage import gaussian_filter
        z = gaussian_filter(rng.standard_normal((ny, nx)), 6.0)
        m = z > np.quantile(z, 1 - sea)
    else:
        m = rng.uniform(size=(ny, nx)) < sea
    return np.repeat(m[None], nlev, axis=0)


def pair(P, nx, ny, mask, seed, smin=1.2, smax=10.0, variance=None, unit_dc=True, order=3):
    rng = np.random.default_rng(seed)
    nlev = mask.shape[0]
    g = uniform_grid(nx, ny, 5000.0, 6000.0, nlev=nlev)
    g["dx"] = 5000.0 * rng.uniform(0.8, 1.2, (ny, nx))
    g["mask"] = mask
    rx = g["dx"] * rng.uniform(smin, smax, (ny, nx))
    ry = g["dy"] * rng.uniform(smin, smax, (ny, nx))
    grid = P.Grid2D(nx, ny, g["dx"], g["dy"], mask)
    opts = P.CovarianceOptions(order=P.FilterOrder(order), unit_dc=unit_dc, variance=variance)
    gpu = P.HorizontalCovarianceOp(grid, P.ScaleField(rx, ry), opts)
    cpu = O.OracleOp(nx, ny, g["dx"], g["dy"], mask, rx, ry, order=order, unit_dc=unit_dc,
                     variance=variance, threads=8)
    return gpu, cpu


def check_all(P, gpu, cpu, f, mask, kinds=KINDS):
    for name in kinds:
        got = gpu.apply(getattr(P, name), f)
        want = cpu.apply(getattr(O, name), f)
        assert relmax(got, want) <= TOL64, (name, relmax(got, want))
        assert np.all(got[:, ~mask] == 0.0), name


@pytest.mark.parametrize("nx,ny,nlev,nvar,sea,runs", [
    (40, 30, 3, 2, 0.8, False),     # one chunk
    (300, 20, 2, 1, 0.9, True),     # two chunks, partial second
    (600, 16, 3, 2, 0.7, True),     # three chunks
    (1442, 12, 2, 1, 0.7, False),   # C3/C4 row length: 6 chunks
    (4320, 6, 2, 1, 0.7, True),     # C5 row length: 16 chunks (cluster of 16)
    (601, 10, 2, 2, 0.8, True),     # odd row length (pitched device copy)
])
def test_single_pass_x_random_shared_masks(P, nx, ny, nlev, nvar, sea, runs):
    mask = shared_mask(nx, ny, nlev, 100 + nx, sea, runs)
    var = np.random.default_rng(3).uniform(0.5, 2.0, (nlev, ny, nx))
    gpu, cpu = pair(P, nx, ny, mask, 200 + nx, variance=var)
    f = np.random.default_rng(4).standard_normal((nvar, nlev, ny, nx))
    check_all(P, gpu, cpu, f, mask)


@pytest.mark.parametrize("nx", [544, 4320, 1000])
def test_single_pass_all_sea_rows_cross_every_chunk(P, nx):
    """All sea: one segment per row across all chunks, no closures (grid
    edges have no ghosts): the carries S and T cross every boundary."""
    mask = np.ones((2, 8, nx), dtype=bool)
    gpu, cpu = pair(P, nx, 8, mask, 300 + nx, smin=6.0, smax=10.0)
    f = np.random.default_rng(5).standard_normal((1, 2, 8, nx))
    check_all(P, gpu, cpu, f, mask, ["GX", "GXT", "GYGX", "VT"])


def test_single_pass_segment_edges_at_chunk_boundaries(P):
    """Land placed so segments start / end on the first, second, last and
    second-to-last points of chunks (chunk length 272 at nx = 600 -> 3
    chunks of 208 after balancing; the test derives the boundaries)."""
    nx, ny, nlev = 600, 24, 2
    rc = ((nx + 2) // 3 + 15) // 16 * 16
    mask = np.ones((nlev, ny, nx), dtype=bool)
    for r in range(ny):
        for b in (rc, 2 * rc):
            off = r % 6
            # land at boundary-relative offsets -3..+2 varying by row
            pos = b + [-3, -2, -1, 0, 1, 2][off]
            mask[:, r, pos] = False
            if r % 2:
                mask[:, r, pos + 1] = False
    var = np.random.default_rng(6).uniform(0.5, 2.0, (nlev, ny, nx))
    gpu, cpu = pair(P, nx, ny, mask, 400, smin=3.0, smax=9.0, variance=var)
    f = np.random.default_rng(7).standard_normal((1, nlev, ny, nx))
    check_all(P, gpu, cpu, f, mask)


def test_single_pass_many_planes_and_options(P):
    """100 levels (4 plane groups of 25) and unit_dc off."""
    nx, ny, nlev = 560, 6, 100
    mask = shared_mask(nx, ny, nlev, 8, 0.75, True)
    gpu, cpu = pair(P, nx, ny, mask, 9, unit_dc=False)
    f = np.random.default_rng(10).standard_normal((1, nlev, ny, nx))
    check_all(P, gpu, cpu, f, mask, ["GX", "GXT", "GYGX"])


def test_single_pass_is_the_x_path(P, monkeypatch):
    """One launch per x sweep (the checkpointed form takes two), and
    RGF_B200_SP=0 (read at creation) selects the checkpointed kernels; both
    agree within the fp64 tolerance."""
    import torch
    nx, ny, nlev = 800, 16, 4
    mask = shared_mask(nx, ny, nlev, 11, 0.8, True)
    gpu, cpu = pair(P, nx, ny, mask, 12)
    monkeypatch.setenv("RGF_B200_SP", "0")
    ck, _ = pair(P, nx, ny, mask, 12)
    monkeypatch.delenv("RGF_B200_SP")
    f = torch.from_numpy(np.random.default_rng(13).standard_normal((1, nlev, ny, nx))).cuda()
    for op, launches in ((gpu, 1), (ck, 2)):
        op.apply(P.GX, f)  # tables built on first use
        torch.cuda.synchronize()
        l0 = op.launch_count()
        op.apply(P.GX, f)
        torch.cuda.synchronize()
        assert op.launch_count() - l0 == launches
    a = gpu.apply(P.GXT, f).cpu().numpy()
    b = ck.apply(P.GXT, f).cpu().numpy()
    assert relmax(a, b) <= TOL64
    assert relmax(a, cpu.apply(O.GXT, f.cpu().numpy())) <= TOL64
