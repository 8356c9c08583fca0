"""Container I/O (io.cpp:133-281) against the oracle's
restatement of io.cpp (nlohmann::json, oracle/rgf_oracle_io.cpp).

CPU: host-path round trips are byte-identical between the product writer
(its own header writer/parser, csrc/container_io.cuh) and the oracle's
nlohmann-based writer/reader in both directions; the error messages are
io.cpp's. GPU: fields stream into and out of device memory through pinned
chunks (fields larger than one 32 MB chunk, fp64 and fp32, level stacks)."""
import filecmp

import numpy as np
import pytest

import oracle as O
import paper_1404_5756_b200 as P


def grid_case(nx=37, ny=23, seed=3):
    rng = np.random.default_rng(seed)
    dx = rng.uniform(1000, 5000, (ny, nx))
    dy = rng.uniform(1000, 5000, (ny, nx))
    mask = rng.uniform(size=(ny, nx)) < 0.8
    return P.Grid2D(nx, ny, dx, dy, mask, 7)


def test_grid_round_trip_matches_oracle(tmp_path):
    g = grid_case()
    a, b = tmp_path / "ours.grid", tmp_path / "oracle.grid"
    P.save_grid(g, a)
    O.save_grid(b, g.dx, g.dy, g.mask, g.ghost_width)
    assert filecmp.cmp(a, b, shallow=False)  # identical bytes, header included
    assert open(a, "rb").readline() == (b'{"endianness":"little","format":"rgf-grid",'
                                        b'"ghost_width":7,"nx":37,"ny":23,'
                                        b'"sections":["dx","dy","mask"]}\n')
    back = P.load_grid(b)
    dx, dy, mask, gw = O.load_grid(a, g.nx, g.ny)
    for got in (back,):
        assert (got.nx, got.ny, got.ghost_width) == (37, 23, 7)
        assert np.array_equal(got.dx, g.dx) and np.array_equal(got.dy, g.dy)
        assert np.array_equal(got.mask, g.mask)
    assert np.array_equal(dx, g.dx) and np.array_equal(mask, g.mask) and gw == 7
    P.save_grid(back, tmp_path / "again.grid")
    assert filecmp.cmp(a, tmp_path / "again.grid", shallow=False)


def test_scale_and_field_round_trips_match_oracle(tmp_path):
    g = grid_case()
    rng = np.random.default_rng(4)
    s = P.ScaleField(g.dx * rng.uniform(1, 9, g.dx.shape), g.dy * rng.uniform(1, 9, g.dy.shape))
    P.save_scale_field(s, tmp_path / "a.scale")
    O.save_scale(tmp_path / "b.scale", s.rx, s.ry)
    assert filecmp.cmp(tmp_path / "a.scale", tmp_path / "b.scale", shallow=False)
    back = P.load_scale_field(tmp_path / "b.scale", g)
    assert np.array_equal(back.rx, s.rx) and np.array_equal(back.ry, s.ry)
    f = rng.standard_normal((g.ny, g.nx))
    P.save_state_field(f, tmp_path / "a.field")
    O.save_field(tmp_path / "b.field", f)
    assert filecmp.cmp(tmp_path / "a.field", tmp_path / "b.field", shallow=False)
    assert np.array_equal(P.load_state_field(tmp_path / "b.field", g), f)
    assert np.array_equal(O.load_field(tmp_path / "a.field", g.nx, g.ny), f)
    f32 = P.load_state_field(tmp_path / "a.field", g, dtype=np.float32)
    assert f32.dtype == np.float32 and np.array_equal(f32, f.astype(np.float32))


def test_level_stack_extension(tmp_path):
    """nlev > 1 fields carry an "nlev" key; the reference's reader (the oracle)
    still reads the first level."""
    g = grid_case(20, 9)
    f = np.random.default_rng(5).standard_normal((3, g.ny, g.nx))
    P.save_state_field(f, tmp_path / "s.field")
    assert P.container_info(tmp_path / "s.field")["nlev"] == 3
    assert np.array_equal(P.load_state_field(tmp_path / "s.field", g, nlev=3), f)
    assert np.array_equal(O.load_field(tmp_path / "s.field", g.nx, g.ny), f[0])
    with pytest.raises(P.IOError_, match="level count does not match"):
        P.load_state_field(tmp_path / "s.field", g, nlev=2)


def test_io_errors_match_reference_messages(tmp_path):
    g = grid_case()
    with pytest.raises(P.IOError_, match="cannot open"):
        P.load_state_field(tmp_path / "missing.field", g)
    P.save_state_field(np.zeros((g.ny, g.nx)), tmp_path / "f.field")
    with pytest.raises(P.IOError_, match='expected a "rgf-grid" container'):
        P.load_grid(tmp_path / "f.field")
    small = grid_case(20, 9)
    with pytest.raises(P.IOError_, match="field file dimensions do not match the grid"):
        P.load_state_field(tmp_path / "f.field", small)
    raw = open(tmp_path / "f.field", "rb").read()
    open(tmp_path / "t.field", "wb").write(raw[:-8])
    with pytest.raises(P.IOError_, match=r'payload section "values" is truncated'):
        P.load_state_field(tmp_path / "t.field", g)
    with pytest.raises(O.OracleError, match=r'payload section "values" is truncated'):
        O.load_field(tmp_path / "t.field", g.nx, g.ny)
    P.save_grid(g, tmp_path / "g.grid")
    open(tmp_path / "x.grid", "wb").write(open(tmp_path / "g.grid", "rb").read() + b"\0")
    with pytest.raises(P.IOError_, match="trailing bytes after grid payload"):
        P.load_grid(tmp_path / "x.grid")
    with pytest.raises(O.OracleError, match="trailing bytes after grid payload"):
        O.load_grid(tmp_path / "x.grid", g.nx, g.ny)
    hdr = b'{"endianness":"big","format":"rgf-field","nx":37,"ny":23,"sections":["values"]}\n'
    open(tmp_path / "b.field", "wb").write(hdr + raw.split(b"\n", 1)[1])
    with pytest.raises(P.IOError_, match="only little-endian payloads are supported"):
        P.load_state_field(tmp_path / "b.field", g)
    open(tmp_path / "m.field", "wb").write(b'{"format":"rgf-field",\n')
    with pytest.raises(P.IOError_, match="malformed container header"):
        P.load_state_field(tmp_path / "m.field", g)
    bad = P.Grid2D(g.nx, g.ny, -g.dx, g.dy, g.mask)
    P.save_grid(bad, tmp_path / "bad.grid")
    with pytest.raises(P.InvalidArgument, match="grid spacing must be strictly positive"):
        P.load_grid(tmp_path / "bad.grid")
    s = P.ScaleField(np.full((g.ny, g.nx), 5000.0), np.full((g.ny, g.nx), 5000.0))
    s.rx[4, 6] = -1.0
    g.mask[4, 6] = True
    P.save_scale_field(s, tmp_path / "bad.scale")
    with pytest.raises(P.InvalidArgument, match=r"radius at sea point \(6,4\)"):
        P.load_scale_field(tmp_path / "bad.scale", g)


@pytest.mark.gpu
@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_field_streams_into_and_out_of_device_memory(tmp_path, dt):
    """A C5-sized level (4320 x 2160, 74.6 MB: three 32 MB pinned chunks) and a
    3-level stack stream straight into device memory and back; the files are
    byte-identical to the host writer's and to the oracle's."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    g = P.Grid2D.uniform(4320, 2160, 9250.0, 9250.0)
    rng = np.random.default_rng(6)
    for nlev in (1, 3):
        shape = (nlev, g.ny, g.nx) if nlev > 1 else (g.ny, g.nx)
        f = rng.standard_normal(shape).astype(dt)
        P.save_state_field(f, tmp_path / "h.field")
        d = P.load_state_field(tmp_path / "h.field", g, nlev=nlev, dtype=dt, device="cuda")
        torch.cuda.synchronize()
        assert d.is_cuda and torch.equal(d.cpu(), torch.from_numpy(f))
        P.save_state_field(d, tmp_path / "d.field")
        assert filecmp.cmp(tmp_path / "h.field", tmp_path / "d.field", shallow=False)
        if nlev == 1:
            O.save_field(tmp_path / "o.field", f.astype(np.float64))
            assert filecmp.cmp(tmp_path / "h.field", tmp_path / "o.field", shallow=False)
