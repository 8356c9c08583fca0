"""GPU parity: the CUDA path through the C ABI against the CPU oracle on the
same seeded inputs. Tolerances (north_star): relative max-norm 1e-12 for
fp64, 1e-5 for fp32 (oracle = fp64 applied to the fp32-rounded input);
segment/mask indexing bit-exact."""
import numpy as np
import pytest

import oracle as O
from helpers import checkered_mask, relmax, segments_numpy, uniform_grid

pytestmark = pytest.mark.gpu

TOL64 = 1e-12
TOL32 = 1e-5


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1404_5756_b200 as P
    return P


def build_pair(P, g, rx, ry, order=3, k=1, unit_dc=True, ghost=None, variance=None,
               calibration=0, grid_ghost=0):
    grid = P.Grid2D(g["nx"], g["ny"], g["dx"], g["dy"], g["mask"], grid_ghost)
    opts = P.CovarianceOptions(order=P.FilterOrder(order), k_iterations=k, unit_dc=unit_dc,
                               ghost_width=ghost, variance=variance,
                               calibration=P.Rf3Calibration(calibration))
    gpu = P.HorizontalCovarianceOp(grid, P.ScaleField(rx, ry), opts)
    cpu = O.OracleOp(g["nx"], g["ny"], g["dx"], g["dy"], g["mask"], rx, ry, order=order,
                     k_iterations=k, unit_dc=unit_dc, ghost_width=ghost, variance=variance,
                     threads=4, calibration=calibration, grid_ghost_width=grid_ghost)
    return gpu, cpu


def random_case(seed, nx=57, ny=43, nlev=3, sea=0.8, smin=1.2, smax=4.5):
    rng = np.random.default_rng(seed)
    g = uniform_grid(nx, ny, 5000.0, 7000.0, nlev=nlev)
    g["dx"] = 5000.0 * rng.uniform(0.7, 1.3, (ny, nx))
    g["mask"] = checkered_mask(nx, ny, seed + 1, sea, nlev=nlev)
    rx = g["dx"] * rng.uniform(smin, smax, (ny, nx))
    ry = g["dy"] * rng.uniform(smin, smax, (ny, nx))
    return g, rx, ry


KINDS = ["GX", "GY", "GXT", "GYT", "V", "VT", "B", "GYGX"]


@pytest.mark.parametrize("order,k,nx", [(3, 1, 57), (3, 1, 58), (3, 1, 96), (1, 1, 57),
                                        (1, 5, 57)])
def test_all_kinds_fp64_random_masks(P, order, k, nx):
    """nx=57: unaligned rows (register-batched kernels); nx=58/96: bulk-copy
    y-sweep with a partial and a full last column tile."""
    g, rx, ry = random_case(10 + order + k, nx=nx)
    var = np.random.default_rng(2).uniform(0.5, 2.0, (3, 43, nx))
    gpu, cpu = build_pair(P, g, rx, ry, order=order, k=k, variance=var)
    f = np.random.default_rng(3).standard_normal((2, 3, 43, nx))
    for name in KINDS:
        kind = getattr(P, name)
        got = gpu.apply(kind, f)
        want = cpu.apply(getattr(O, name), f)
        assert relmax(got, want) <= TOL64, (name, relmax(got, want))
        land = ~g["mask"]
        assert np.all(got[:, land] == 0.0), name


@pytest.mark.parametrize("order,k,nx", [(3, 1, 57), (3, 1, 60), (1, 5, 57), (3, 1, 96), (3, 1, 160)])
def test_fp32_storage(P, order, k, nx):
    g, rx, ry = random_case(40 + order, nx=nx)
    gpu, cpu = build_pair(P, g, rx, ry, order=order, k=k)
    f32 = np.random.default_rng(4).standard_normal((1, 3, 43, nx)).astype(np.float32)
    for name in ("GYGX", "VT", "B"):
        got = gpu.apply(getattr(P, name), f32)
        assert got.dtype == np.float32
        want = cpu.apply(getattr(O, name), f32.astype(np.float64))
        assert relmax(got, want) <= TOL32, (name, relmax(got, want))


def test_segments_bit_exact(P):
    g, rx, ry = random_case(5, nx=64, ny=50, nlev=4, sea=0.6)
    gpu, _ = build_pair(P, g, rx, ry)
    for d in (0, 1):
        off, segs = gpu.segments(d)
        roff, rsegs = segments_numpy(g["mask"], d)
        assert np.array_equal(off, roff)
        assert np.array_equal(segs, rsegs)


def test_coefficient_tables(P):
    g, rx, ry = random_case(6, sea=0.7)
    for order, k in ((3, 1), (1, 5)):
        gpu, _ = build_pair(P, g, rx, ry, order=order, k=k)
        any_sea = g["mask"].any(axis=0)
        for d, (r, s) in enumerate(((rx, g["dx"]), (ry, g["dy"]))):
            c = gpu.coefficients(d)
            sig = np.where(any_sea, r / s, 1.0)
            for idx in zip(*np.nonzero(any_sea)):
                if order == 3:
                    want = O.rf3_filter_scalars(sig[idx])
                    assert c["alpha1"][idx] == want[0]
                    assert c["alpha2"][idx] == want[1]
                    assert c["alpha3"][idx] == want[2]
                    assert abs(c["beta"][idx] - want[3]) <= 4 * np.spacing(abs(want[3]))
                    assert c["inv_dc"][idx] == 1.0 / (np.sqrt(2 * np.pi) * sig[idx])
                else:
                    want = O.rf1_coefficients(sig[idx], k)
                    assert c["alpha1"][idx] == want[0]
                    assert c["beta"][idx] == want[1]


def test_scalar_builders(P, golden):
    for row in golden["kGolden"]["rows"]:
        t = P.rf3_coefficients(row["sigma"])
        o = O.rf3_coefficients(row["sigma"])
        assert (t.a0, t.a1, t.a2, t.a3, t.alpha1, t.alpha2, t.alpha3) == tuple(o[:7])
        assert abs(t.beta - o[7]) <= 4 * np.spacing(abs(o[7]))
        assert abs(t.beta - row["beta"]) <= 1e-12 * abs(row["beta"])
    for cal in (0, 1, 2):
        for s in (0.05, 0.7, 2.5, 7.3, 14.0):
            f = P.rf3_filter_scalars(s, P.Rf3Calibration(cal))
            o = O.rf3_filter_scalars(s, cal)
            assert (f.alpha1, f.alpha2, f.alpha3, f.q) == (o[0], o[1], o[2], o[4])
            assert abs(f.beta - o[3]) <= 4 * np.spacing(abs(o[3]))
    for s in (0.5, 2.0, 25.0):
        for k in (1, 5, 10):
            a = P.rf1_coefficients(s, k)
            o = O.rf1_coefficients(s, k)
            assert (a.alpha, a.beta) == (o[0], o[1])
    with pytest.raises(P.InvalidArgument, match="sigma must be positive"):
        P.rf3_coefficients(0.0)


def test_1d_entry_points(P):
    rng = np.random.default_rng(9)
    m = 75
    sig = rng.uniform(1.0, 5.0, m)
    x = rng.standard_normal((6, m))
    for tr in (False, True):
        got = (P.rf3_apply_transpose_1d if tr else P.rf3_apply_1d)(x, sig)
        for i in range(6):
            want = O.rf3_apply_1d(x[i], sig, transpose=tr)
            assert relmax(got[i], want) <= 1e-13
        got = (P.rf1_apply_transpose_1d if tr else P.rf1_apply_1d)(x, sig, 3)
        for i in range(6):
            want = O.rf1_apply_1d(x[i], sig, 3, transpose=tr)
            assert relmax(got[i], want) <= 1e-13
    with pytest.raises(P.InvalidArgument, match="segment length must be >= 4"):
        P.rf3_apply_1d(np.zeros(3), 2.0)


def test_c1_config_parity_and_gaussian(P):
    from paper_1404_5756_b200 import synth
    c = synth.make_config("C1")
    f = synth.make_field(c)
    g = dict(nx=c.nx, ny=c.ny, dx=c.dx, dy=c.dy, mask=c.mask)
    for order, k in ((3, 1), (1, 5)):
        gpu, cpu = build_pair(P, g, c.rx, c.ry, order=order, k=k)
        got = gpu.apply(P.GYGX, f)
        want = cpu.apply(O.GYGX, f)
        assert relmax(got, want) <= TOL64
    # impulse-only run against the analytic Gaussian (unit_dc=false,
    # unit-sum error as diagnostics.cpp:86-93)
    gpu, _ = build_pair(P, g, c.rx, c.ry, unit_dc=False)
    d = np.zeros((c.ny, c.nx))
    d[c.ny // 2, c.nx // 2] = 1.0
    h = gpu.apply(P.GYGX, d)
    gx = synth.analytic_gaussian(c.nx, c.nx // 2, 4.0)
    gy = synth.analytic_gaussian(c.ny, c.ny // 2, 4.0)
    err = np.linalg.norm(h / h.sum() - np.outer(gy, gx))
    assert err < 0.02


def test_edge_cases(P):
    rng = np.random.default_rng(21)
    # tiny grid, ghost_width=0 with short segments passing through
    g = uniform_grid(5, 4)
    g["mask"][:, :, 2] = False
    rx = ry = np.full((4, 5), 12000.0)
    gpu, cpu = build_pair(P, g, rx, ry, unit_dc=False, ghost=0)
    f = rng.standard_normal((4, 5))
    for kind in ("GX", "GY", "B"):
        assert np.array_equal(gpu.apply(getattr(P, kind), f), cpu.apply(getattr(O, kind), f))
    # all-land level, single-point segments, per-level ghost widths
    nx, ny = 31, 17
    g = uniform_grid(nx, ny, nlev=4)
    g["mask"][0] = False
    g["mask"][1] = checkered_mask(nx, ny, 2, 0.3)[0]
    g["mask"][2] = checkered_mask(nx, ny, 3, 0.9)[0]
    rx = 6000.0 * rng.uniform(1.0, 6.0, (ny, nx))
    ry = 6000.0 * rng.uniform(1.0, 6.0, (ny, nx))
    gpu, cpu = build_pair(P, g, rx, ry)
    for lev in range(4):
        assert gpu.effective_ghost_width(lev) == cpu.ghost_width(lev)
    f = rng.standard_normal((4, ny, nx))
    for kind in ("V", "VT", "B"):
        got, want = gpu.apply(getattr(P, kind), f), cpu.apply(getattr(O, kind), f)
        assert relmax(got, want) <= TOL64
        assert np.all(got[0] == 0.0)
    # ghost resolution (test_covariance.cpp:348-359)
    g = uniform_grid(16, 16)
    r = np.full((16, 16), 12000.0)
    assert build_pair(P, g, r, r)[0].effective_ghost_width() == 18
    assert build_pair(P, g, r, r, grid_ghost=7)[0].effective_ghost_width() == 7
    assert build_pair(P, g, r, r, grid_ghost=7, ghost=0)[0].effective_ghost_width() == 0


def test_reference_error_messages(P):
    g = uniform_grid(8, 8)
    r = np.full((8, 8), 12000.0)
    with pytest.raises(P.InvalidArgument, match="single-iteration by construction"):
        build_pair(P, g, r, r, order=3, k=2)
    with pytest.raises(P.InvalidArgument, match="k_iterations must be >= 1"):
        build_pair(P, g, r, r, order=1, k=0)
    bad = r.copy()
    bad[3, 5] = -1.0
    with pytest.raises(P.InvalidArgument, match=r"non-positive or non-finite radius at sea point \(5,3\)"):
        build_pair(P, g, bad, r)
    g2 = uniform_grid(8, 8)
    g2["dx"][1, 1] = 0.0
    with pytest.raises(P.InvalidArgument, match="grid spacing must be strictly positive"):
        build_pair(P, g2, r, r)


def test_deterministic_reruns(P):
    g, rx, ry = random_case(77)
    gpu, _ = build_pair(P, g, rx, ry)
    f = np.random.default_rng(1).standard_normal((3, 43, 57))
    a = gpu.apply(P.B, f)
    b = gpu.apply(P.B, f)
    assert np.array_equal(a, b)


def test_c2_subset_forward_adjoint(P):
    from paper_1404_5756_b200 import synth
    c = synth.make_config("C2", nlev=6)
    g = dict(nx=c.nx, ny=c.ny, dx=c.dx, dy=c.dy, mask=c.mask)
    f = synth.make_field(c)
    for order, k in ((3, 1), (1, 5)):
        gpu, cpu = build_pair(P, g, c.rx, c.ry, order=order, k=k)
        for kind in ("GYGX", "VT"):
            got = gpu.apply(getattr(P, kind), f)
            want = cpu.apply(getattr(O, kind), f)
            assert relmax(got, want) <= TOL64, (order, kind, relmax(got, want))


def test_torch_device_path(P):
    import torch
    g, rx, ry = random_case(88)
    gpu, cpu = build_pair(P, g, rx, ry)
    f = np.random.default_rng(5).standard_normal((2, 3, 43, 57))
    t = torch.from_numpy(f).cuda()
    out = gpu.apply(P.GYGX, t)
    torch.cuda.synchronize()
    assert relmax(out.cpu().numpy(), cpu.apply(O.GYGX, f)) <= TOL64
    assert gpu.launch_count() > 0


def test_exact_mode_matches_oracle_to_rounding(P, monkeypatch):
    """RGF_B200_EXACT=1 selects the segment-serial kernel with the reference's
    unfused arithmetic; only beta's pow() may differ by an ulp."""
    g, rx, ry = random_case(123)
    monkeypatch.setenv("RGF_B200_EXACT", "1")
    gpu, cpu = build_pair(P, g, rx, ry)
    monkeypatch.delenv("RGF_B200_EXACT")
    f = np.random.default_rng(8).standard_normal((3, 43, 57))
    for name in ("GYGX", "VT"):
        got = gpu.apply(getattr(P, name), f)
        want = cpu.apply(getattr(O, name), f)
        assert relmax(got, want) <= 1e-14, (name, relmax(got, want))


def test_many_planes_partial_blocks(P):
    """40 planes (2 vars x 20 levels): y-sweep CTAs with 16 and 8 planes."""
    g, rx, ry = random_case(321, nx=64, ny=37, nlev=20, sea=0.75)
    gpu, cpu = build_pair(P, g, rx, ry)
    f = np.random.default_rng(6).standard_normal((2, 20, 37, 64))
    for name in ("GYGX", "VT", "GY", "GYT"):
        got = gpu.apply(getattr(P, name), f)
        want = cpu.apply(getattr(O, name), f)
        assert relmax(got, want) <= TOL64, (name, relmax(got, want))


def test_streaming_vs_exact_path(P, monkeypatch):
    """The streaming path (FMA + right-ghost closure) against the exact
    segment-serial path on a C5-like mask with sigma up to 10 (G = 90)."""
    from paper_1404_5756_b200 import synth
    c = synth.make_config("C5", nlev=2, nx=600, ny=300)
    g = dict(nx=c.nx, ny=c.ny, dx=c.dx, dy=c.dy, mask=c.mask)
    f = synth.make_field(c)
    fast, cpu = build_pair(P, g, c.rx, c.ry)
    assert fast.effective_ghost_width() == cpu.ghost_width()
    for name in ("GYGX", "VT", "B"):
        got = fast.apply(getattr(P, name), f)
        want = cpu.apply(getattr(O, name), f)
        assert relmax(got, want) <= TOL64, (name, relmax(got, want))


@pytest.mark.parametrize("sea", [0.45, 0.7])
def test_short_segments_tma_paths(P, sea):
    """Many length-1/2 segments (corrections at j-1, j-2 skipped), segment ends
    on stage boundaries, aligned rows (TMA paths, fused closure)."""
    g, rx, ry = random_case(900 + int(sea * 100), nx=96, ny=40, nlev=2, sea=sea)
    gpu, cpu = build_pair(P, g, rx, ry)
    f = np.random.default_rng(12).standard_normal((2, 40, 96))
    for name in ("GX", "GY", "GXT", "GYT", "B"):
        got = gpu.apply(getattr(P, name), f)
        want = cpu.apply(getattr(O, name), f)
        assert relmax(got, want) <= TOL64, (name, relmax(got, want))
        assert np.all(got[~g["mask"]] == 0.0)


@pytest.mark.parametrize("order,k,nx", [(3, 1, 64), (3, 1, 57), (1, 5, 64)])
def test_host_pipeline_matches_device_path(P, order, k, nx):
    """Host-memory applies run as a level-chunked H2D/compute/D2H pipeline
    (10 levels -> chunks of 3, 2 vars -> 8 chunks over 3 device slots). The
    result must be bit-identical to the one-shot device apply, for every kind,
    with per-level ghost widths (several closure classes) and in place."""
    import torch
    g, rx, ry = random_case(700 + order + nx, nx=nx, ny=29, nlev=10, sea=0.7, smax=6.0)
    var = np.random.default_rng(21).uniform(0.5, 2.0, (10, 29, nx))
    gpu, cpu = build_pair(P, g, rx, ry, order=order, k=k, variance=var)
    f = np.random.default_rng(22).standard_normal((2, 10, 29, nx))
    for name in KINDS:
        kind = getattr(P, name)
        host = gpu.apply(kind, f)
        dev = gpu.apply(kind, torch.from_numpy(f).cuda())
        torch.cuda.synchronize()
        assert np.array_equal(host, dev.cpu().numpy()), name
        if name in ("GYGX", "B"):
            assert relmax(host, cpu.apply(getattr(O, name), f)) <= TOL64, name
    g2 = f.astype(np.float32)
    want = gpu.apply(P.VT, g2.copy())
    gpu.apply(P.VT, g2, out=g2)  # in place through the pipeline
    assert np.array_equal(g2, want)


def test_segment_ends_at_checkpoint_block_edges(P):
    """Checkpointed sweeps cut lines into blocks (64 points in x, 32 rows in
    y). Land cells are placed so segments end on a block's first, second and
    last points and start on its first two, so the folded ghost entries owe
    corrections to the block on the left."""
    nx, ny, nlev = 200, 100, 5
    g = uniform_grid(nx, ny, 5000.0, 6000.0, nlev=nlev)
    mask = np.ones((nlev, ny, nx), dtype=bool)
    xland = [[65], [66], [64], [62, 63], [1, 127, 130, 191]]
    yland = [[33], [34], [32], [30, 31], [1, 63, 66, 95]]
    for lev in range(nlev):
        mask[lev][:, xland[lev]] = False
        mask[lev][yland[lev], :] = False
    g["mask"] = mask
    rng = np.random.default_rng(77)
    rx = g["dx"] * rng.uniform(1.5, 4.0, (ny, nx))
    ry = g["dy"] * rng.uniform(1.5, 4.0, (ny, nx))
    var = rng.uniform(0.5, 2.0, (nlev, ny, nx))
    gpu, cpu = build_pair(P, g, rx, ry, variance=var)
    f = rng.standard_normal((2, nlev, ny, nx))
    for name in KINDS:
        got = gpu.apply(getattr(P, name), f)
        want = cpu.apply(getattr(O, name), f)
        assert relmax(got, want) <= TOL64, (name, relmax(got, want))
        assert np.all(got[:, ~mask] == 0.0)
    got32 = gpu.apply(P.B, f.astype(np.float32))
    want32 = cpu.apply(O.B, f.astype(np.float32).astype(np.float64))
    assert relmax(got32, want32) <= TOL32


def test_level_sharded_ops_match_full_op(P):
    """Per-rank operators over level blocks (paper_1404_5756_b200.sharding),
    run here one after the other on one GPU, reproduce the full operator bit
    for bit: a level's result does not depend on the other levels."""
    from paper_1404_5756_b200.sharding import ShardedCovarianceOp
    g, rx, ry = random_case(404, nx=64, ny=40, nlev=7, sea=0.7)
    var = np.random.default_rng(9).uniform(0.5, 2.0, (7, 40, 64))
    f = np.random.default_rng(10).standard_normal((2, 7, 40, 64))
    full, _ = build_pair(P, g, rx, ry, variance=var)
    for name in ("GYGX", "B"):
        want = full.apply(getattr(P, name), f)
        parts = []
        for r in range(3):
            sop = ShardedCovarianceOp(64, 40, g["dx"], g["dy"], g["mask"], rx, ry,
                                      P.CovarianceOptions(), nlev=7, world=3, rank=r,
                                      variance=var)
            parts.append(sop.apply(getattr(P, name), np.ascontiguousarray(sop.local_slice(f))))
        assert np.array_equal(np.concatenate(parts, axis=1), want), name


@pytest.mark.parametrize("nx,dt", [(57, "f64"), (61, "f32"), (58, "f32")])
def test_unaligned_rows_device_path_pitched(P, nx, dt):
    """Rows whose byte length is not a 16 B multiple run the checkpointed
    kernels on an internal pitched copy (device applies) or pitched slots
    (host applies); both must agree with the oracle and with each other."""
    import torch
    g, rx, ry = random_case(600 + nx, nx=nx, ny=45, nlev=4, sea=0.7)
    gpu, cpu = build_pair(P, g, rx, ry)
    f = np.random.default_rng(15).standard_normal((2, 4, 45, nx))
    if dt == "f32":
        f = f.astype(np.float32)
    tol = TOL64 if dt == "f64" else TOL32
    for name in ("GYGX", "VT", "B"):
        host = gpu.apply(getattr(P, name), f)
        dev = gpu.apply(getattr(P, name), torch.from_numpy(f).cuda())
        torch.cuda.synchronize()
        assert np.array_equal(host, dev.cpu().numpy()), name
        want = cpu.apply(getattr(O, name), f.astype(np.float64))
        assert relmax(host, want) <= tol, (name, relmax(host, want))


@pytest.mark.parametrize("k", [1, 2, 5])
def test_rf1_streaming_path(P, monkeypatch, k):
    """RGF_B200_RF1LINE=0: the 1st-RF as 2K streaming passes per sweep (ghost
    zones folded into per-segment convolutions), against the oracle and
    against the segment-serial exact kernel (RGF_B200_EXACT=1, reference
    arithmetic). It is the fallback of the line-resident kernel."""
    g, rx, ry = random_case(800 + k, nx=70, ny=44, nlev=3, sea=0.65)
    var = np.random.default_rng(17).uniform(0.5, 2.0, (3, 44, 70))
    monkeypatch.setenv("RGF_B200_RF1LINE", "0")
    gpu, cpu = build_pair(P, g, rx, ry, order=1, k=k, variance=var)
    monkeypatch.delenv("RGF_B200_RF1LINE")
    monkeypatch.setenv("RGF_B200_EXACT", "1")
    exact, _ = build_pair(P, g, rx, ry, order=1, k=k, variance=var)
    monkeypatch.delenv("RGF_B200_EXACT")
    import torch
    f = np.random.default_rng(18).standard_normal((2, 3, 44, 70))
    ft = torch.from_numpy(f).cuda()
    for name in KINDS:
        l0 = gpu.launch_count()
        gpu.apply(getattr(P, name), ft)  # device path: one launch set per sweep
        torch.cuda.synchronize()
        sweeps = {"GX": 1, "GY": 1, "GXT": 1, "GYT": 1, "V": 2, "VT": 2, "B": 4, "GYGX": 2}[name]
        # 2K passes + (2K-1) entry-state kernels per sweep
        assert gpu.launch_count() - l0 == (4 * k - 1) * sweeps, (name, gpu.launch_count() - l0)
        got = gpu.apply(getattr(P, name), f)
        want = cpu.apply(getattr(O, name), f)
        assert relmax(got, want) <= TOL64, (name, relmax(got, want))
        assert relmax(got, exact.apply(getattr(P, name), f)) <= TOL64, name


@pytest.mark.parametrize("k,nx,ny,ghost", [(1, 70, 44, None), (2, 57, 43, None), (5, 70, 44, None),
                                           (5, 96, 40, 0), (3, 64, 50, 2), (5, 300, 200, None)])
def test_rf1_line_resident_path(P, monkeypatch, k, nx, ny, ghost):
    """The default 1st-RF path (rf1_line.cuh): one launch per sweep runs all K
    iterations with the line resident on chip, each pass a parallel scan.
    Every kind in fp64 and fp32 against the oracle and the exact kernel;
    ghost_width = 0 covers the pass-through of isolated points
    (covariance.cpp:260-269); nx = 57 rows are not 16 B aligned (cp.async
    pieces instead of bulk copies)."""
    g, rx, ry = random_case(900 + k + nx, nx=nx, ny=ny, nlev=3, sea=0.65)
    var = np.random.default_rng(17).uniform(0.5, 2.0, (3, ny, nx))
    gpu, cpu = build_pair(P, g, rx, ry, order=1, k=k, variance=var, ghost=ghost)
    monkeypatch.setenv("RGF_B200_EXACT", "1")
    exact, _ = build_pair(P, g, rx, ry, order=1, k=k, variance=var, ghost=ghost)
    monkeypatch.delenv("RGF_B200_EXACT")
    import torch
    f = np.random.default_rng(18).standard_normal((2, 3, ny, nx))
    ft = torch.from_numpy(f).cuda()
    land = ~g["mask"]
    for name in KINDS:
        l0 = gpu.launch_count()
        dev = gpu.apply(getattr(P, name), ft)
        torch.cuda.synchronize()
        sweeps = {"GX": 1, "GY": 1, "GXT": 1, "GYT": 1, "V": 2, "VT": 2, "B": 4, "GYGX": 2}[name]
        assert gpu.launch_count() - l0 == sweeps, (name, gpu.launch_count() - l0)
        want = cpu.apply(getattr(O, name), f)
        got = dev.cpu().numpy()
        assert relmax(got, want) <= TOL64, (name, relmax(got, want))
        assert np.all(got[:, land] == 0.0), name
        assert relmax(got, exact.apply(getattr(P, name), f)) <= TOL64, name
        assert np.array_equal(gpu.apply(getattr(P, name), f), got), name  # host pipeline
    f32 = f.astype(np.float32)
    for name in ("GYGX", "VT", "B"):
        got = gpu.apply(getattr(P, name), f32)
        want = cpu.apply(getattr(O, name), f32.astype(np.float64))
        assert got.dtype == np.float32 and relmax(got, want) <= TOL32, (name, relmax(got, want))


def test_rf1_line_resident_shared_masks_and_long_lines(P):
    """Levels with one mask reuse a CTA's links, masks and zone tables from
    plane to plane (several planes per CTA, the next plane's row prefetched);
    a 4400-point row takes the 512-thread shape and a 2300-row column does
    not fit the resident shapes (streaming fallback for that direction)."""
    rng = np.random.default_rng(31)
    nx, ny, nlev = 64, 1300, 6
    g = uniform_grid(nx, ny, 5000.0, 7000.0, nlev=nlev)
    g["mask"] = np.repeat(checkered_mask(nx, ny, 5, 0.7, nlev=1), nlev, axis=0)
    rx = g["dx"] * rng.uniform(1.2, 4.5, (ny, nx))
    ry = g["dy"] * rng.uniform(1.2, 4.5, (ny, nx))
    gpu, cpu = build_pair(P, g, rx, ry, order=1, k=5)
    f = rng.standard_normal((1, nlev, ny, nx))
    for name in ("GYGX", "VT"):
        assert relmax(gpu.apply(getattr(P, name), f), cpu.apply(getattr(O, name), f)) <= TOL64, name
    for nx, ny in ((4400, 24), (40, 2300)):
        g = uniform_grid(nx, ny, 5000.0, 7000.0, nlev=2)
        g["mask"] = checkered_mask(nx, ny, 9, 0.8, nlev=2)
        rx = g["dx"] * rng.uniform(1.2, 6.0, (ny, nx))
        ry = g["dy"] * rng.uniform(1.2, 6.0, (ny, nx))
        gpu, cpu = build_pair(P, g, rx, ry, order=1, k=3)
        f = rng.standard_normal((1, 2, ny, nx))
        for name in ("GYGX", "VT"):
            assert relmax(gpu.apply(getattr(P, name), f), cpu.apply(getattr(O, name), f)) <= TOL64, \
                (nx, ny, name)


@pytest.mark.parametrize("nx,dt", [(96, "f64"), (160, "f32"), (64, "f64")])
def test_paired_x_tiles_match_single(P, monkeypatch, nx, dt):
    """Rows a whole number of blocks long take the paired x tiles (256 B
    runs, k_xck1p/k_xck2p); RGF_B200_XPAIR=0 (read at first launch) is not
    switchable inside one process, so compare against the oracle and check
    every kind, with variance and per-level masks; nx = 96 gives an odd
    block count (6 blocks of 16 -> 3 tiles; 160 fp32 -> 5 blocks of 32)."""
    g, rx, ry = random_case(950 + nx, nx=nx, ny=41, nlev=4, sea=0.7)
    var = np.random.default_rng(23).uniform(0.5, 2.0, (4, 41, nx))
    gpu, cpu = build_pair(P, g, rx, ry, variance=var)
    f = np.random.default_rng(24).standard_normal((2, 4, 41, nx))
    tol = TOL64
    if dt == "f32":
        f = f.astype(np.float32)
        tol = TOL32
    for name in KINDS:
        got = gpu.apply(getattr(P, name), f)
        want = cpu.apply(getattr(O, name), f.astype(np.float64))
        assert relmax(got, want) <= tol, (name, relmax(got, want))
        assert np.all(got[:, ~g["mask"]] == 0.0), name



@pytest.mark.parametrize("nx,dt", [(80, "f64"), (96, "f64"), (96, "f32")])
def test_rf1_block_multiple_rows(P, nx, dt):
    """1st-RF streaming passes on rows a whole number of 128 B blocks long,
    odd and even block counts, fp64 and fp32, every kind with variance."""
    g, rx, ry = random_case(970 + nx, nx=nx, ny=33, nlev=3, sea=0.65)
    var = np.random.default_rng(25).uniform(0.5, 2.0, (3, 33, nx))
    gpu, cpu = build_pair(P, g, rx, ry, order=1, k=5, variance=var)
    f = np.random.default_rng(26).standard_normal((2, 3, 33, nx))
    tol = TOL64
    if dt == "f32":
        f = f.astype(np.float32)
        tol = TOL32
    for name in KINDS:
        got = gpu.apply(getattr(P, name), f)
        want = cpu.apply(getattr(O, name), f.astype(np.float64))
        assert relmax(got, want) <= tol, (name, relmax(got, want))
        assert np.all(got[:, ~g["mask"]] == 0.0), name


@pytest.mark.parametrize("nlev,nvar,nx,ny,dt", [(1, 1, 96, 64, "f64"), (3, 2, 128, 40, "f64"),
                                                (1, 1, 160, 48, "f32"), (2, 1, 57, 44, "f64"),
                                                (1, 1, 64, 43, "f64"), (1, 1, 96, 45, "f32")])
def test_few_plane_x_sweep_transposed(P, monkeypatch, nlev, nvar, nx, ny, dt):
    """RGF_B200_XT=1: with <= 8 planes the x sweep runs as a y sweep on the transposed field
    (lanes = rows; x tables built in the transposed frame, closures
    included; odd ny pads the transposed rows to a 16 B pitch): every kind
    against the oracle, in place too, with variance and per-level masks."""
    monkeypatch.setenv("RGF_B200_XT", "1")  # opt-in, read at operator creation
    g, rx, ry = random_case(990 + nx + nlev, nx=nx, ny=ny, nlev=nlev, sea=0.7)
    var = np.random.default_rng(27).uniform(0.5, 2.0, (nlev, ny, nx))
    gpu, cpu = build_pair(P, g, rx, ry, variance=var)
    f = np.random.default_rng(28).standard_normal((nvar, nlev, ny, nx))
    tol = TOL64
    if dt == "f32":
        f = f.astype(np.float32)
        tol = TOL32
    for name in KINDS:
        got = gpu.apply(getattr(P, name), f)
        want = cpu.apply(getattr(O, name), f.astype(np.float64))
        assert relmax(got, want) <= tol, (name, relmax(got, want))
        assert np.all(got[:, ~g["mask"]] == 0.0), name
    h = f.copy()
    gpu.apply(P.GX, h, out=h)
    assert relmax(h, cpu.apply(O.GX, f.astype(np.float64))) <= tol


def test_concurrent_applies_on_two_streams(P):
    """The reference's apply_* are const and safe to call concurrently
    (covariance.cpp:21-34, thread_local scratch). Two host threads apply the
    same operator on two CUDA streams (device fields) and a third thread
    uses host arrays; the op's shared scratch is event-guarded, so every
    result equals the oracle's."""
    import threading
    import torch
    g, rx, ry = random_case(77, nx=96, ny=64, nlev=3, sea=0.8)
    gpu, cpu = build_pair(P, g, rx, ry)
    rng = np.random.default_rng(78)
    fields = [rng.standard_normal((2, 3, 64, 96)) for _ in range(3)]
    kinds = ["GYGX", "VT", "B"]
    wants = [cpu.apply(getattr(O, k), f) for k, f in zip(kinds, fields)]
    got = [None] * 3
    errors = []

    def dev(i):
        try:
            s = torch.cuda.Stream()
            x = torch.from_numpy(fields[i]).cuda()
            torch.cuda.synchronize()
            with torch.cuda.stream(s):
                outs = [gpu.apply(getattr(P, kinds[i]), x) for _ in range(20)]
            s.synchronize()
            got[i] = [o.cpu().numpy() for o in outs]
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    def host(i):
        try:
            got[i] = [gpu.apply(getattr(P, kinds[i]), fields[i]) for _ in range(5)]
        except Exception as e:  # pragma: no cover
            errors.append(e)

    ts = [threading.Thread(target=dev, args=(0,)), threading.Thread(target=dev, args=(1,)),
          threading.Thread(target=host, args=(2,))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for i in range(3):
        for r in got[i]:
            assert relmax(r, wants[i]) <= TOL64, (kinds[i], relmax(r, wants[i]))


def test_apply_out_argument_is_checked(P):
    """A caller-supplied `out` must match the field's dtype, shape and layout
    (and device for tensors): the C ABI writes field-sized data through it."""
    import torch
    g, rx, ry = random_case(79, nx=64, ny=40, nlev=1)
    gpu, _ = build_pair(P, g, rx, ry)
    f = np.random.default_rng(80).standard_normal((1, 1, 40, 64))
    with pytest.raises(P.InvalidArgument):
        gpu.apply(P.GYGX, f, out=np.empty(f.shape, np.float32))
    with pytest.raises(P.InvalidArgument):
        gpu.apply(P.GYGX, f, out=np.empty((1, 1, 40, 32)))
    with pytest.raises(P.InvalidArgument):
        gpu.apply(P.GYGX, f, out=np.empty((1, 1, 64, 40)).transpose(0, 1, 3, 2))
    t = torch.from_numpy(f).cuda()
    with pytest.raises(P.InvalidArgument):
        gpu.apply(P.GYGX, t, out=torch.empty_like(t, dtype=torch.float32))
    with pytest.raises(P.InvalidArgument):
        gpu.apply(P.GYGX, t, out=torch.empty((1, 1, 64, 40), dtype=t.dtype,
                                             device="cuda").transpose(2, 3))
    ok = np.empty_like(f)
    assert gpu.apply(P.GYGX, f, out=ok) is ok


def test_1d_entry_points_with_coefficient_tables(P):
    """rf3_filter_coefficients / the rf1 table overload (rf3.hpp:191-210,
    rf1.hpp:96-110) and the filters taking those tables (rf3.hpp:292-334,
    rf1.hpp:113-155): tables match the oracle's per-point builders, filtering
    with them equals the sigma entry points bit for bit and the oracle within
    1e-14 of the output scale; the scalar helpers rf3_cascade_variance and
    rf3_length_scale_argument (rf3.hpp:101-154) match the oracle."""
    rng = np.random.default_rng(31)
    m = 97
    sig = rng.uniform(0.8, 9.5, m)
    x = rng.standard_normal((5, m))
    for cal in (0, 1, 2):
        c = P.rf3_filter_coefficients(sig, P.Rf3Calibration(cal))
        for i in (0, 17, 96):
            s = O.rf3_filter_scalars(sig[i], cal)  # alpha1 alpha2 alpha3 beta q
            got_a = np.array([c.alpha1[i], c.alpha2[i], c.alpha3[i], c.beta[i]])
            assert np.all(np.abs(got_a - s[:4]) <= 4 * np.spacing(np.abs(s[:4]))), (cal, i)
        for tr in (False, True):
            got = P.rf3_filter(x, c, transpose=tr)
            if cal == 0:
                same = (P.rf3_apply_transpose_1d if tr else P.rf3_apply_1d)(x, sig)
                assert np.array_equal(got, same)
            for r in range(5):
                want = O.rf3_apply_1d_coeffs(x[r], c.alpha1, c.alpha2, c.alpha3, c.beta,
                                             transpose=tr)
                assert relmax(got[r], want) <= 1e-14
    for k in (1, 4):
        c1 = P.rf1_coefficients_table(sig, k)
        for i in (0, 50):
            s1 = O.rf1_coefficients(sig[i], k)
            assert c1.alpha[i] == s1[0] and c1.beta[i] == s1[1]
        for tr in (False, True):
            got = P.rf1_filter(x, c1, transpose=tr)
            same = (P.rf1_apply_transpose_1d if tr else P.rf1_apply_1d)(x, sig, k)
            assert np.array_equal(got, same)
    for q in (0.5, 2.0, 7.5):
        assert P.rf3_cascade_variance(q) == pytest.approx(O.rf3_cascade_variance(q), rel=1e-14)
    for s0 in (0.3, 2.0, 8.0):
        for cal in (0, 1, 2):
            assert P.rf3_length_scale_argument(s0, P.Rf3Calibration(cal)) == pytest.approx(
                O.rf3_length_scale_argument(s0, cal), rel=1e-13)
    with pytest.raises(P.InvalidArgument, match="segment length must be >= 4"):
        P.rf3_filter(np.zeros(3), P.rf3_filter_coefficients(np.ones(3)))
    with pytest.raises(P.InvalidArgument, match="sigma must be positive"):
        P.rf3_filter_coefficients(np.array([1.0, -1.0]))


def test_batched_diagnostics_match_oracle(P):
    """Many impulse studies and Remark-1 checks at once (diagnostics.cpp:69-135,
    SURVEY §8f row 4), one device thread per study, against the oracle's
    per-study restatement: responses within 1e-13 of their peak, the error
    norms within 1e-10 relative (device exp vs glibc exp), same verdicts."""
    sig = np.array([0.7, 1.5, 2.0, 4.0, 6.5, 10.0])
    for order, k in ((3, 1), (1, 1), (1, 5)):
        rep = P.impulse_responses(sig, P.FilterOrder.third if order == 3 else P.FilterOrder.first,
                                  k, 257)
        for i, s0 in enumerate(sig):
            h, sh, e2, emax = O.impulse_response(s0, order, k, 257)
            assert np.max(np.abs(rep.h[i] - h)) <= 1e-13 * np.max(np.abs(h))
            assert rep.sum_h[i] == pytest.approx(sh, rel=1e-13)
            assert rep.err_h_l2[i] == pytest.approx(e2, rel=1e-10)
            assert rep.err_h_max[i] == pytest.approx(emax, rel=1e-10)
    x = np.random.default_rng(32).standard_normal((6, 301))
    for order, k in ((3, 1), (1, 5)):
        r = P.remark1_bound_checks(x, sig, P.FilterOrder.third if order == 3 else P.FilterOrder.first, k)
        for i in range(6):
            lhs, rhs, err, holds = O.remark1(x[i], sig[i], order, k)
            assert r["lhs"][i] == pytest.approx(lhs, rel=1e-10)
            assert r["rhs"][i] == pytest.approx(rhs, rel=1e-10)
            assert r["err_h_l2"][i] == pytest.approx(err, rel=1e-10)
            assert bool(r["holds"][i]) == holds
    with pytest.raises(P.InvalidArgument, match="length must be >= 4"):
        P.impulse_responses([2.0], P.FilterOrder.third, 1, 3)


@pytest.mark.parametrize("nx,ny,sea,dt,nvar", [(96, 64, 0.8, "f64", 1), (57, 43, 0.7, "f64", 2),
                                               (300, 5, 0.9, "f64", 1), (7, 300, 0.9, "f32", 1),
                                               (128, 1000, 1.0, "f64", 1), (600, 217, 0.85, "f32", 3)])
def test_single_level_chunked_sweeps(P, nx, ny, sea, dt, nvar):
    """Single-level operators (the reference's 2-D API) run the chunked sweep
    (sweep_few.cuh: 16 row chunks per 32-column tile, carries folded in
    shared memory; x lines through the transposed field): every kind with
    variance against the oracle, including lines shorter than the chunk
    count, all-sea lines crossing every chunk, odd sizes and fp32."""
    g, rx, ry = random_case(1200 + nx + ny, nx=nx, ny=ny, nlev=1, sea=sea, smax=9.5)
    var = np.random.default_rng(29).uniform(0.5, 2.0, (1, ny, nx))
    gpu, cpu = build_pair(P, g, rx, ry, variance=var)
    f = np.random.default_rng(30).standard_normal((nvar, 1, ny, nx))
    tol = TOL64
    if dt == "f32":
        f = f.astype(np.float32)
        tol = TOL32
    for name in KINDS:
        got = gpu.apply(getattr(P, name), f)
        want = cpu.apply(getattr(O, name), f.astype(np.float64))
        assert relmax(got, want) <= tol, (name, relmax(got, want))
        assert np.all(got[:, ~g["mask"]] == 0.0), name
