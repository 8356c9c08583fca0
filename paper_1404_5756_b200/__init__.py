"""B200-native recursive-filter horizontal covariance operator (arXiv 1404.5756).

Python mirror of the reference C++ interface (``rgf`` namespace of
/root/reference/proj/include/rgf): ``Grid2D``, ``ScaleField``,
``uniform_scale``, ``CovarianceOptions``, ``HorizontalCovarianceOp`` with the
seven ``apply_*`` methods, ``effective_ghost_width`` and
``coefficient_bytes``, plus the scalar coefficient builders and 1-D entry
points. Every call goes through the C ABI in ``include/rgf_b200.h``
(``librgf_b200.so``, sm_100a kernels). There is no CPU fallback: without the
built library the import fails, without a GPU the calls raise.

Array convention: numpy/torch arrays are C-ordered ``(ny, nx)`` per level, so
element ``[iy, ix]`` sits at ``iy*nx + ix`` — the reference's x-fastest
layout (types.hpp:25-28). Batched fields are ``(nvar, nlev, ny, nx)``.
"""
from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass, field as dc_field
from typing import Optional

import numpy as np

__all__ = [
    "FilterOrder", "Rf3Calibration", "Grid2D", "ScaleField", "uniform_scale",
    "CovarianceOptions", "HorizontalCovarianceOp", "InvalidArgument", "DeviceError",
    "rf3_coefficients", "rf3_filter_scalars", "rf1_coefficients",
    "rf3_apply_1d", "rf3_apply_transpose_1d", "rf1_apply_1d", "rf1_apply_transpose_1d",
    "rf3_cascade_variance", "rf3_length_scale_argument", "Rf3Coefficients", "Rf1Coefficients",
    "rf3_filter_coefficients", "rf1_coefficients_table", "rf3_filter", "rf1_filter",
    "container_info", "load_grid", "save_grid", "load_scale_field", "save_scale_field",
    "load_state_field", "save_state_field", "IOError_",
    "impulse_responses", "remark1_bound_checks", "ImpulseReports",
    "lib", "LIB_PATH",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RGF_B200_LIB") or os.path.join(_HERE, "librgf_b200.so")  # dev override

if not os.path.exists(LIB_PATH):  # fail loudly: the product has no fallback
    raise ImportError(
        f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`")

lib = ctypes.CDLL(LIB_PATH)

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


class _GridDesc(ctypes.Structure):
    _fields_ = [("nx", _i64), ("ny", _i64), ("nlev", _i64), ("dx", _vp), ("dy", _vp),
                ("mask", _vp), ("ghost_width", _i64)]


class _Options(ctypes.Structure):
    _fields_ = [("order", _i32), ("k_iterations", _i32), ("unit_dc", _i32),
                ("calibration", _i32), ("ghost_width", _i64), ("variance", _vp),
                ("threads", _i32), ("device", _i32)]


lib.rgf_last_error.restype = ctypes.c_char_p
lib.rgf_options_default.argtypes = [ctypes.POINTER(_Options)]
lib.rgf_options_default.restype = None
lib.rgf_op_create.argtypes = [ctypes.POINTER(_GridDesc), _vp, _vp, ctypes.POINTER(_Options),
                              ctypes.POINTER(_vp)]
lib.rgf_op_destroy.argtypes = [_vp]
lib.rgf_op_apply.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _i64, ctypes.c_int, _vp]
lib.rgf_op_ghost_width.argtypes = [_vp, _i64, ctypes.POINTER(_i64)]
lib.rgf_op_coefficient_bytes.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint64)]
lib.rgf_op_device_bytes.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint64)]
lib.rgf_op_launch_count.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint64)]
lib.rgf_op_segments.argtypes = [_vp, ctypes.c_int, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                _vp, _vp]
lib.rgf_op_coefficients.argtypes = [_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp]
lib.rgf_rf3_coefficients.argtypes = [ctypes.c_double, _dp]
lib.rgf_rf3_filter_scalars.argtypes = [ctypes.c_double, ctypes.c_int, _dp]
lib.rgf_rf1_coefficients.argtypes = [ctypes.c_double, ctypes.c_int, _dp]
lib.rgf_rf3_apply_1d.argtypes = [_vp, _vp, _i64, _i64, ctypes.c_int, ctypes.c_int, _vp]
lib.rgf_rf1_apply_1d.argtypes = [_vp, _vp, _i64, _i64, ctypes.c_int, ctypes.c_int, _vp]
lib.rgf_rf3_cascade_variance.argtypes = [ctypes.c_double, _dp]
lib.rgf_impulse_responses.argtypes = [_vp, _i64, ctypes.c_int, ctypes.c_int, _i64, ctypes.c_int,
                                      _vp, _vp, _vp, _vp]
lib.rgf_remark1_checks.argtypes = [_vp, _vp, _i64, _i64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   _vp]
lib.rgf_container_info.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(_i64),
                                   ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                   ctypes.POINTER(_i64)]
lib.rgf_grid_load.argtypes = [ctypes.c_char_p, _i64, _i64, _vp, _vp, _vp, ctypes.POINTER(_i64)]
lib.rgf_grid_save.argtypes = [ctypes.c_char_p, ctypes.POINTER(_GridDesc)]
lib.rgf_scale_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(_GridDesc), _vp, _vp]
lib.rgf_scale_save.argtypes = [ctypes.c_char_p, _i64, _i64, _vp, _vp]
lib.rgf_field_load.argtypes = [ctypes.c_char_p, _i64, _i64, _i64, ctypes.c_int, _vp,
                               ctypes.c_int, _vp]
lib.rgf_field_save.argtypes = [ctypes.c_char_p, _i64, _i64, _i64, ctypes.c_int, _vp,
                               ctypes.c_int, _vp]
lib.rgf_rf3_length_scale_argument.argtypes = [ctypes.c_double, ctypes.c_int, _dp]
lib.rgf_rf3_filter_coefficients.argtypes = [_vp, _i64, ctypes.c_int, _vp, _vp, _vp, _vp]
lib.rgf_rf1_coefficients_table.argtypes = [_vp, _i64, ctypes.c_int, _vp, _vp]
lib.rgf_rf3_filter.argtypes = [_vp, _vp, _vp, _vp, _vp, _i64, _i64, ctypes.c_int, _vp]
lib.rgf_rf1_filter.argtypes = [_vp, _vp, _vp, _i64, _i64, ctypes.c_int, ctypes.c_int, _vp]

# C ABI constants (include/rgf_b200.h)
GX, GY, GXT, GYT, V, VT, B, GYGX = range(8)
F64, F32 = 0, 1
HOST, DEVICE = 0, 1


class InvalidArgument(ValueError):
    """The reference's std::invalid_argument (same message text)."""


class DeviceError(RuntimeError):
    """CUDA failure (no device, launch error, out of memory)."""


def _check(status: int) -> None:
    if status == 0:
        return
    msg = lib.rgf_last_error().decode()
    if status == 1:
        raise InvalidArgument(msg)
    if status == 3:
        raise DeviceError(msg)
    raise RuntimeError(msg)


class FilterOrder(enum.IntEnum):  # types.hpp:30
    first = 1
    third = 3


class Rf3Calibration(enum.IntEnum):  # types.hpp:39
    yvv95 = 0
    variance_match = 1
    none = 2


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


@dataclass
class Grid2D:
    """grid.hpp:20-37, with an optional level axis on the mask.

    dx, dy: (ny, nx) metres. mask: (ny, nx) or (nlev, ny, nx), True = sea.
    """
    nx: int
    ny: int
    dx: np.ndarray
    dy: np.ndarray
    mask: np.ndarray
    ghost_width: int = 0

    @staticmethod
    def uniform(nx: int, ny: int, dx: float, dy: float, ghost_width: int = 0,
                nlev: int = 1) -> "Grid2D":
        shape = (ny, nx) if nlev == 1 else (nlev, ny, nx)
        return Grid2D(nx, ny, np.full((ny, nx), float(dx)), np.full((ny, nx), float(dy)),
                      np.ones(shape, dtype=bool), ghost_width)

    @property
    def nlev(self) -> int:
        return 1 if np.ndim(self.mask) == 2 else int(np.shape(self.mask)[0])

    def size(self) -> int:
        return self.nx * self.ny

    def all_sea(self) -> bool:
        return bool(np.all(self.mask))


@dataclass
class ScaleField:
    """grid.hpp:40-52: per-point correlation radii (metres), (ny, nx)."""
    rx: np.ndarray
    ry: np.ndarray

    def sigma_x(self, grid: Grid2D) -> np.ndarray:  # grid.cpp:57-59 (2-D grids)
        return np.where(grid.mask, self.rx / grid.dx, 1.0)

    def sigma_y(self, grid: Grid2D) -> np.ndarray:
        return np.where(grid.mask, self.ry / grid.dy, 1.0)


def uniform_scale(grid: Grid2D, r: float) -> ScaleField:
    """grid.cpp:69-76."""
    if not r > 0:
        raise InvalidArgument("uniform_scale: radius must be positive")
    return ScaleField(np.full((grid.ny, grid.nx), float(r)), np.full((grid.ny, grid.nx), float(r)))


@dataclass
class CovarianceOptions:
    """covariance.hpp:17-25 (plus the CUDA device ordinal)."""
    order: FilterOrder = FilterOrder.third
    k_iterations: int = 1
    unit_dc: bool = True
    ghost_width: Optional[int] = None
    variance: Optional[np.ndarray] = None
    threads: int = 0
    calibration: Rf3Calibration = Rf3Calibration.yvv95
    device: int = 0


class HorizontalCovarianceOp:
    """covariance.hpp:35-79: V_H = G_y G_x on a masked grid and its relatives.

    apply_* accept numpy arrays (host: copied to the device and back, like
    the reference's out-of-place StateField returns) or CUDA torch tensors
    (device-resident, asynchronous on the current stream).
    """

    def __init__(self, grid: Grid2D, scales: ScaleField,
                 options: Optional[CovarianceOptions] = None):
        options = options or CovarianceOptions()
        self.grid_ = grid
        self.options_ = options
        nx, ny, nlev = int(grid.nx), int(grid.ny), grid.nlev
        shape_ok = (np.shape(grid.dx) == (ny, nx) and np.shape(grid.dy) == (ny, nx))
        if not shape_ok:
            raise InvalidArgument("Grid2D: spacing field shape mismatch")
        if np.shape(grid.mask)[-2:] != (ny, nx):
            raise InvalidArgument("Grid2D: mask shape mismatch")
        if np.shape(scales.rx) != (ny, nx) or np.shape(scales.ry) != (ny, nx):
            raise InvalidArgument("ScaleField: shape does not match grid")
        self._dx = np.ascontiguousarray(grid.dx, dtype=np.float64)
        self._dy = np.ascontiguousarray(grid.dy, dtype=np.float64)
        self._mask = np.ascontiguousarray(np.reshape(grid.mask, (nlev, ny, nx)), dtype=np.uint8)
        self._rx = np.ascontiguousarray(scales.rx, dtype=np.float64)
        self._ry = np.ascontiguousarray(scales.ry, dtype=np.float64)
        desc = _GridDesc(nx, ny, nlev, _ptr(self._dx), _ptr(self._dy), _ptr(self._mask),
                         int(grid.ghost_width))
        opt = _Options()
        lib.rgf_options_default(ctypes.byref(opt))
        opt.order = int(options.order)
        opt.k_iterations = int(options.k_iterations)
        opt.unit_dc = 1 if options.unit_dc else 0
        opt.calibration = int(options.calibration)
        opt.ghost_width = -1 if options.ghost_width is None else int(options.ghost_width)
        if options.ghost_width is not None and options.ghost_width < 0:
            raise InvalidArgument("covariance: ghost_width < 0")
        self._var = None
        if options.variance is not None:
            var = np.asarray(options.variance, dtype=np.float64)
            if var.shape[-2:] != (ny, nx) or (var.ndim == 3 and var.shape[0] != nlev):
                raise InvalidArgument("covariance: variance field shape mismatch")
            self._var = np.ascontiguousarray(np.broadcast_to(var.reshape((-1, ny, nx)),
                                                             (nlev, ny, nx)))
            opt.variance = _ptr(self._var)
        opt.threads = int(options.threads)
        opt.device = int(options.device)
        handle = _vp()
        _check(lib.rgf_op_create(ctypes.byref(desc), _ptr(self._rx), _ptr(self._ry),
                                 ctypes.byref(opt), ctypes.byref(handle)))
        self._h = handle

    def __del__(self):
        if lib is None:  # interpreter teardown
            return
        h = getattr(self, "_h", None)
        if h:
            lib.rgf_op_destroy(h)
            self._h = None

    # -- reference accessors (covariance.hpp:49-56)
    def grid(self) -> Grid2D:
        return self.grid_

    def options(self) -> CovarianceOptions:
        return self.options_

    def effective_ghost_width(self, level: int = 0) -> int:
        out = _i64()
        _check(lib.rgf_op_ghost_width(self._h, level, ctypes.byref(out)))
        return out.value

    def coefficient_bytes(self) -> int:
        out = ctypes.c_uint64()
        _check(lib.rgf_op_coefficient_bytes(self._h, ctypes.byref(out)))
        return out.value

    def device_bytes(self) -> int:
        out = ctypes.c_uint64()
        _check(lib.rgf_op_device_bytes(self._h, ctypes.byref(out)))
        return out.value

    def launch_count(self) -> int:
        out = ctypes.c_uint64()
        _check(lib.rgf_op_launch_count(self._h, ctypes.byref(out)))
        return out.value

    def segments(self, direction: int):
        """(offsets[nlines+1], segs[nsegs, 2]) built by the segmentation kernel."""
        nl, ns = _i64(), _i64()
        _check(lib.rgf_op_segments(self._h, direction, ctypes.byref(nl), ctypes.byref(ns),
                                   None, None))
        off = np.empty(nl.value + 1, dtype=np.int64)
        segs = np.empty((max(ns.value, 1), 2), dtype=np.int32)
        _check(lib.rgf_op_segments(self._h, direction, None, None, _ptr(off), _ptr(segs)))
        return off, segs[: ns.value]

    def coefficients(self, direction: int) -> dict:
        nh = self.grid_.nx * self.grid_.ny
        shp = (self.grid_.ny, self.grid_.nx)
        out = {k: np.zeros(shp) for k in ("alpha1", "alpha2", "alpha3", "beta", "inv_dc")}
        _check(lib.rgf_op_coefficients(self._h, direction, *(_ptr(out[k]) for k in
                                       ("alpha1", "alpha2", "alpha3", "beta", "inv_dc"))))
        del nh
        return out

    # -- applies (covariance.cpp:362-398)
    def apply(self, kind: int, field, out=None, stream=None):
        """Generic entry: kind in {GX, GY, GXT, GYT, V, VT, B, GYGX}."""
        try:
            import torch  # plumbing only
            is_torch = isinstance(field, torch.Tensor)
        except ImportError:  # pragma: no cover
            is_torch = False
        nx, ny, nlev = self.grid_.nx, self.grid_.ny, self.grid_.nlev
        if is_torch:
            return self._apply_torch(kind, field, out, stream)
        f = np.asarray(field)
        if f.dtype not in (np.float64, np.float32):
            f = f.astype(np.float64)
        if f.shape[-2:] != (ny, nx) or f.size % (nx * ny * nlev) != 0:
            raise InvalidArgument("apply: field is not on the expected grid")
        f = np.ascontiguousarray(f)
        nvar = f.size // (nx * ny * nlev)
        if out is None:
            res = np.empty_like(f)
        else:  # the C ABI writes f.nbytes through this pointer: check it first
            res = out
            if (not isinstance(res, np.ndarray) or res.dtype != f.dtype or res.shape != f.shape
                    or not res.flags.c_contiguous or not res.flags.writeable):
                raise InvalidArgument("apply: out must be a writeable C-contiguous array with "
                                      "the field's dtype and shape")
        dtype = F64 if f.dtype == np.float64 else F32
        _check(lib.rgf_op_apply(self._h, kind, dtype, _ptr(f), _ptr(res), nvar, HOST, None))
        return res

    def _apply_torch(self, kind, field, out, stream):
        import torch
        nx, ny, nlev = self.grid_.nx, self.grid_.ny, self.grid_.nlev
        if not field.is_cuda:
            raise InvalidArgument("apply: torch tensors must be on the CUDA device")
        if field.dtype not in (torch.float64, torch.float32) or not field.is_contiguous():
            raise InvalidArgument("apply: expected a contiguous float64/float32 tensor")
        if tuple(field.shape[-2:]) != (ny, nx) or field.numel() % (nx * ny * nlev):
            raise InvalidArgument("apply: field is not on the expected grid")
        if field.device != torch.device("cuda", int(self.options_.device)):
            raise InvalidArgument("apply: field is not on the operator's device")
        nvar = field.numel() // (nx * ny * nlev)
        if out is None:
            res = torch.empty_like(field)
        else:
            res = out
            if (not isinstance(res, torch.Tensor) or res.dtype != field.dtype
                    or res.shape != field.shape or res.device != field.device
                    or not res.is_contiguous()):
                raise InvalidArgument("apply: out must be a contiguous tensor with the field's "
                                      "dtype, shape and device")
        dtype = F64 if field.dtype == torch.float64 else F32
        st = stream if stream is not None else torch.cuda.current_stream(field.device)
        _check(lib.rgf_op_apply(self._h, kind, dtype, field.data_ptr(), res.data_ptr(), nvar,
                                DEVICE, st.cuda_stream))
        return res

    def apply_gx(self, f):
        return self.apply(GX, f)

    def apply_gy(self, f):
        return self.apply(GY, f)

    def apply_gx_transpose(self, f):
        return self.apply(GXT, f)

    def apply_gy_transpose(self, f):
        return self.apply(GYT, f)

    def apply_v(self, f):
        return self.apply(V, f)

    def apply_v_transpose(self, f):
        return self.apply(VT, f)

    def apply_b(self, f):
        return self.apply(B, f)


# ---------------------------------------------------------------- scalars
@dataclass
class Rf3PolynomialSet:  # rf3.hpp:71-76
    a0: float
    a1: float
    a2: float
    a3: float
    alpha1: float
    alpha2: float
    alpha3: float
    beta: float


@dataclass
class Rf3Scalars:  # rf3.hpp:159-164
    alpha1: float
    alpha2: float
    alpha3: float
    beta: float
    q: float


@dataclass
class Rf1Scalars:  # rf1.hpp:66-70
    alpha: float
    beta: float


def rf3_coefficients(sigma: float) -> Rf3PolynomialSet:
    out = (ctypes.c_double * 8)()
    _check(lib.rgf_rf3_coefficients(float(sigma), out))
    return Rf3PolynomialSet(*out)


def rf3_filter_scalars(sigma: float, calibration: Rf3Calibration = Rf3Calibration.yvv95
                       ) -> Rf3Scalars:
    out = (ctypes.c_double * 5)()
    _check(lib.rgf_rf3_filter_scalars(float(sigma), int(calibration), out))
    return Rf3Scalars(*out)


def rf1_coefficients(sigma: float, k: int) -> Rf1Scalars:
    out = (ctypes.c_double * 2)()
    _check(lib.rgf_rf1_coefficients(float(sigma), int(k), out))
    return Rf1Scalars(*out)


def _apply_1d(fn, x, sigma, *args):
    x = np.ascontiguousarray(x, dtype=np.float64)
    m = x.shape[-1]
    sig = np.ascontiguousarray(np.broadcast_to(np.asarray(sigma, dtype=np.float64), (m,)))
    out = np.empty_like(x)
    nlines = x.size // m if m else 0
    _check(fn(_ptr(x), _ptr(sig), m, max(nlines, 1), *args, _ptr(out)))
    return out


def rf3_apply_1d(x, sigma, calibration=Rf3Calibration.yvv95):
    """rf3.hpp:318-325 with rf3_filter_coefficients(sigma) (rf3.hpp:191-210)."""
    return _apply_1d(lib.rgf_rf3_apply_1d, x, sigma, int(calibration), 0)


def rf3_apply_transpose_1d(x, sigma, calibration=Rf3Calibration.yvv95):
    return _apply_1d(lib.rgf_rf3_apply_1d, x, sigma, int(calibration), 1)


def rf1_apply_1d(x, sigma, k):
    """rf1.hpp:139-146 with rf1_coefficients(sigma, k) (rf1.hpp:96-110)."""
    return _apply_1d(lib.rgf_rf1_apply_1d, x, sigma, int(k), 0)


def rf1_apply_transpose_1d(x, sigma, k):
    return _apply_1d(lib.rgf_rf1_apply_1d, x, sigma, int(k), 1)


def rf3_cascade_variance(q: float) -> float:
    """rf3.hpp:101-108."""
    out = ctypes.c_double()
    _check(lib.rgf_rf3_cascade_variance(float(q), ctypes.byref(out)))
    return out.value


def rf3_length_scale_argument(sigma: float, calibration: Rf3Calibration) -> float:
    """rf3.hpp:143-154."""
    out = ctypes.c_double()
    _check(lib.rgf_rf3_length_scale_argument(float(sigma), int(calibration), ctypes.byref(out)))
    return out.value


@dataclass
class Rf3Coefficients:  # rf3.hpp:183-189 (Rf3CoefficientsT)
    alpha1: np.ndarray
    alpha2: np.ndarray
    alpha3: np.ndarray
    beta: np.ndarray


@dataclass
class Rf1Coefficients:  # rf1.hpp:87-92 (Rf1CoefficientsT)
    alpha: np.ndarray
    beta: np.ndarray
    k_iterations: int = 1


def rf3_filter_coefficients(sigma, calibration=Rf3Calibration.yvv95) -> Rf3Coefficients:
    """rf3.hpp:191-210: per-point tables from a sigma array (device)."""
    sig = np.ascontiguousarray(sigma, dtype=np.float64).ravel()
    t = [np.empty_like(sig) for _ in range(4)]
    _check(lib.rgf_rf3_filter_coefficients(_ptr(sig), sig.size, int(calibration),
                                           *(_ptr(a) for a in t)))
    return Rf3Coefficients(*t)


def rf1_coefficients_table(sigma, k) -> Rf1Coefficients:
    """rf1.hpp:96-110: the table overload of rf1_coefficients (device)."""
    sig = np.ascontiguousarray(sigma, dtype=np.float64).ravel()
    a, b = np.empty_like(sig), np.empty_like(sig)
    _check(lib.rgf_rf1_coefficients_table(_ptr(sig), sig.size, int(k), _ptr(a), _ptr(b)))
    return Rf1Coefficients(a, b, int(k))


def _filter_tables(x, m, fn, tabs, *args):
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape[-1] != m or any(np.size(t) != m for t in tabs):
        raise InvalidArgument("rf filter: coefficient length mismatch")
    tabs = [np.ascontiguousarray(t, dtype=np.float64) for t in tabs]
    out = np.empty_like(x)
    nlines = x.size // m if m else 0
    _check(fn(_ptr(x), *(_ptr(t) for t in tabs), m, max(nlines, 1), *args, _ptr(out)))
    return out


def rf3_filter(x, c: Rf3Coefficients, transpose=False):
    """rf3_filter_in_place / _transpose_in_place / rf3_apply_1d(segment, c)
    (rf3.hpp:292-334) over the last axis of x, with caller tables."""
    x = np.asarray(x, dtype=np.float64)
    return _filter_tables(x, x.shape[-1], lib.rgf_rf3_filter,
                          (c.alpha1, c.alpha2, c.alpha3, c.beta), int(bool(transpose)))


def rf1_filter(x, c: Rf1Coefficients, transpose=False):
    """rf1_filter_in_place / _transpose_in_place / rf1_apply_1d(segment, c)
    (rf1.hpp:113-155) over the last axis of x, with caller tables."""
    x = np.asarray(x, dtype=np.float64)
    return _filter_tables(x, x.shape[-1], lib.rgf_rf1_filter, (c.alpha, c.beta),
                          int(c.k_iterations), int(bool(transpose)))


# --------------------------------------------------------------------------
# Batched diagnostics (diagnostics.cpp:69-135)
@dataclass
class ImpulseReports:  # diagnostics.hpp ImpulseReport, one row per study
    sigma: np.ndarray
    order: FilterOrder
    k: int
    h: np.ndarray        # (n, length) raw responses to a Dirac at length/2
    g: np.ndarray        # (n, length) sampled Gaussians at the same offsets
    sum_h: np.ndarray
    err_h_l2: np.ndarray
    err_h_max: np.ndarray


def impulse_responses(sigmas, order: FilterOrder, k: int, length: int,
                      calibration: Rf3Calibration = Rf3Calibration.yvv95) -> ImpulseReports:
    """impulse_response (diagnostics.cpp:69-96) for many sigmas at once, one
    device thread per study."""
    sig = np.ascontiguousarray(np.atleast_1d(sigmas), dtype=np.float64)
    n = sig.size
    h = np.empty((n, length))
    o = np.empty((3, n))
    ordv = RGF_ORDER[FilterOrder(order)]
    _check(lib.rgf_impulse_responses(_ptr(sig), n, ordv, int(k), int(length), int(calibration),
                                     _ptr(h), _ptr(o[0]), _ptr(o[1]), _ptr(o[2])))
    c = length // 2
    off = np.arange(length) - c
    g = np.exp(-(off[None, :] ** 2) / (2 * sig[:, None] ** 2))
    return ImpulseReports(sig, FilterOrder(order), int(k), h, g, o[0].copy(), o[1].copy(),
                          o[2].copy())


def remark1_bound_checks(s0, sigmas, order: FilterOrder, k: int,
                         calibration: Rf3Calibration = Rf3Calibration.yvv95) -> dict:
    """remark1_bound_check (diagnostics.cpp:102-135) for n inputs (n, m) with
    one sigma each -> arrays lhs, rhs, err_h_l2, holds."""
    x = np.ascontiguousarray(np.atleast_2d(s0), dtype=np.float64)
    n, m = x.shape
    sig = np.ascontiguousarray(np.broadcast_to(np.asarray(sigmas, dtype=np.float64), (n,)))
    o = np.empty((n, 4))
    _check(lib.rgf_remark1_checks(_ptr(x), _ptr(sig), n, m, RGF_ORDER[FilterOrder(order)], int(k),
                                  int(calibration), _ptr(o)))
    return {"lhs": o[:, 0], "rhs": o[:, 1], "err_h_l2": o[:, 2], "holds": o[:, 3] != 0}


RGF_ORDER = {FilterOrder.first: 1, FilterOrder.third: 3}


# --------------------------------------------------------------------------
# Container I/O (io.cpp:133-281). Binary rgf-grid /
# rgf-scale / rgf-field containers; fields stream straight into device memory
# when a torch device is requested.
class IOError_(RuntimeError):
    """The reference's std::runtime_error from io.cpp (same message text)."""


def _io(status):
    if status == 2:
        raise IOError_(lib.rgf_last_error().decode())
    _check(status)


def container_info(path) -> dict:
    fmt = ctypes.create_string_buffer(32)
    nx, ny, g, nl = _i64(), _i64(), _i64(), _i64()
    _io(lib.rgf_container_info(str(path).encode(), fmt, ctypes.byref(nx), ctypes.byref(ny),
                               ctypes.byref(g), ctypes.byref(nl)))
    return {"format": fmt.value.decode(), "nx": nx.value, "ny": ny.value,
            "ghost_width": g.value, "nlev": nl.value}


def load_grid(path) -> Grid2D:
    """io.cpp:133-181 load_grid (binary) with Grid2D::validate (grid.cpp:27-39)."""
    info = container_info(path)
    nx, ny = info["nx"], info["ny"]
    if nx < 1 or ny < 1:
        raise IOError_("container header is missing nx/ny")
    dx, dy = np.empty((ny, nx)), np.empty((ny, nx))
    mask = np.empty((ny, nx), dtype=np.uint8)
    g = _i64()
    _io(lib.rgf_grid_load(str(path).encode(), nx, ny, _ptr(dx), _ptr(dy), _ptr(mask),
                          ctypes.byref(g)))
    return Grid2D(nx, ny, dx, dy, mask.astype(bool), g.value)


def _desc(grid: Grid2D):
    dx = np.ascontiguousarray(grid.dx, dtype=np.float64)
    dy = np.ascontiguousarray(grid.dy, dtype=np.float64)
    m = np.ascontiguousarray(np.reshape(grid.mask, (-1, grid.ny, grid.nx))[0], dtype=np.uint8)
    return _GridDesc(grid.nx, grid.ny, 1, _ptr(dx), _ptr(dy), _ptr(m), int(grid.ghost_width)), \
        (dx, dy, m)


def save_grid(grid: Grid2D, path) -> None:
    """io.cpp:183-202 save_grid (level 0 of the mask)."""
    d, keep = _desc(grid)
    _io(lib.rgf_grid_save(str(path).encode(), ctypes.byref(d)))
    del keep


def load_scale_field(path, grid: Grid2D) -> ScaleField:
    """io.cpp:204-235 load_scale_field (binary) with ScaleField::validate."""
    rx, ry = np.empty((grid.ny, grid.nx)), np.empty((grid.ny, grid.nx))
    d, keep = _desc(grid)
    _io(lib.rgf_scale_load(str(path).encode(), ctypes.byref(d), _ptr(rx), _ptr(ry)))
    del keep
    return ScaleField(rx, ry)


def save_scale_field(scales: ScaleField, path) -> None:
    """io.cpp:237-249."""
    rx = np.ascontiguousarray(scales.rx, dtype=np.float64)
    ry = np.ascontiguousarray(scales.ry, dtype=np.float64)
    ny, nx = rx.shape
    _io(lib.rgf_scale_save(str(path).encode(), nx, ny, _ptr(rx), _ptr(ry)))


def load_state_field(path, grid: Grid2D, nlev: int = 1, dtype=np.float64, device=None):
    """io.cpp:251-269 load_state_field (binary): (nlev, ny, nx) levels. With
    `device` (a torch CUDA device) the payload streams into device memory
    through pinned chunks (no full host copy) and a torch tensor is returned."""
    dt = F64 if np.dtype(dtype) == np.float64 else F32
    shape = (nlev, grid.ny, grid.nx) if nlev > 1 else (grid.ny, grid.nx)
    if device is None:
        out = np.empty(shape, dtype=np.float64 if dt == F64 else np.float32)
        _io(lib.rgf_field_load(str(path).encode(), grid.nx, grid.ny, nlev, dt, _ptr(out), HOST,
                               None))
        return out
    import torch
    out = torch.empty(shape, dtype=torch.float64 if dt == F64 else torch.float32, device=device)
    st = torch.cuda.current_stream(out.device)
    _io(lib.rgf_field_load(str(path).encode(), grid.nx, grid.ny, nlev, dt, out.data_ptr(), DEVICE,
                           st.cuda_stream))
    return out


def save_state_field(values, path) -> None:
    """io.cpp:271-281 save_state_field; `values` (…, ny, nx) numpy or CUDA
    torch tensor (streamed out of device memory through pinned chunks)."""
    try:
        import torch
        is_torch = isinstance(values, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_torch = False
    if is_torch:
        if not values.is_cuda or not values.is_contiguous():
            raise InvalidArgument("save_state_field: expected a contiguous CUDA tensor")
        ny, nx = values.shape[-2:]
        nlev = values.numel() // (nx * ny)
        dt = F64 if values.dtype == torch.float64 else F32
        st = torch.cuda.current_stream(values.device)
        _io(lib.rgf_field_save(str(path).encode(), nx, ny, nlev, dt, values.data_ptr(), DEVICE,
                               st.cuda_stream))
        return
    v = np.ascontiguousarray(values)
    if v.dtype not in (np.float64, np.float32):
        v = v.astype(np.float64)
    ny, nx = v.shape[-2:]
    nlev = v.size // (nx * ny)
    _io(lib.rgf_field_save(str(path).encode(), nx, ny, nlev, F64 if v.dtype == np.float64 else F32,
                           _ptr(v), HOST, None))


# --------------------------------------------------------------------------
# Observation operator and 3D-VAR analysis, mirroring
# obs.hpp:15-46 and solver.hpp:19-55 on a one-level operator. H and H^T run on
# the device bit-identically to the reference (deterministic gather for H^T);
# the CG loop keeps chi, r, p, Ap on the device, one scalar per dot product
# comes back per step.
class _Analysis(ctypes.Structure):
    _fields_ = [("cg_iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("n_gradient_norms", _i64), ("final_relative_residual", ctypes.c_double),
                ("j_background", ctypes.c_double), ("j_obs", ctypes.c_double)]


lib.rgf_obs_create.argtypes = [_vp, ctypes.c_int32, _i64, _vp, _vp, _vp, _vp,
                               ctypes.POINTER(_vp)]
lib.rgf_obs_destroy.argtypes = [_vp]
lib.rgf_obs_apply.argtypes = [_vp, ctypes.c_int, _vp, _vp, ctypes.c_int, _vp]
lib.rgf_cost.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
lib.rgf_solve.argtypes = [_vp, _vp, ctypes.c_double, ctypes.c_int32, _vp, _vp, _vp, _vp,
                          ctypes.POINTER(_Analysis)]


@dataclass
class ObsSet:
    """obs.hpp:15-25: positions (n, 2) fractional grid indices (x, y), values,
    per-observation error variances."""
    positions: np.ndarray
    values: np.ndarray
    r_var: np.ndarray

    def size(self) -> int:
        return int(np.asarray(self.values).size)


@dataclass
class SolveOptions:
    """solver.hpp:19-22."""
    tol: float = 1e-6
    max_iter: int = 30


@dataclass
class Analysis:
    """solver.hpp:24-33."""
    increment: np.ndarray
    misfit: np.ndarray
    cg_iterations: int
    gradient_norms: list
    converged: bool
    final_relative_residual: float
    j_background: float
    j_obs: float


@dataclass
class CostReport:
    """solver.hpp:35-40."""
    j_total: float
    j_background: float
    j_obs: float
    gradient: np.ndarray


class _DeviceObs:
    """rgf_obs handle: stencils validated on creation (obs.cpp:18-44).
    `where` is a Grid2D or an operator (its grid and device)."""

    def __init__(self, where, obs: ObsSet):
        op = where if hasattr(where, "grid") else None
        g = op.grid() if op is not None else where
        device = int(op.options().device) if op is not None else 0
        pos = np.asarray(obs.positions, dtype=np.float64).reshape(-1, 2)
        vals = np.ascontiguousarray(obs.values, dtype=np.float64).reshape(-1)
        rv = np.ascontiguousarray(obs.r_var, dtype=np.float64).reshape(-1)
        if not (pos.shape[0] == vals.size == rv.size):
            raise InvalidArgument("ObsSet: inconsistent column lengths")
        self.n = vals.size
        self._keep = [np.ascontiguousarray(pos[:, 0]), np.ascontiguousarray(pos[:, 1]), vals, rv]
        m0 = np.ascontiguousarray(np.asarray(g.mask).reshape(-1, g.ny, g.nx)[0], dtype=np.uint8)
        self._keep.append(m0)
        desc = _GridDesc(g.nx, g.ny, 1, None, None, _ptr(m0), 0)
        h = _vp()
        _check(lib.rgf_obs_create(ctypes.byref(desc), device, self.n,
                                  *(_ptr(a) for a in self._keep[:4]), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if lib is None:  # interpreter teardown
            return
        h = getattr(self, "_h", None)
        if h and lib is not None:
            lib.rgf_obs_destroy(h)
            self._h = None


def _grid_of(where):
    return where.grid() if hasattr(where, "grid") else where


def _field2d(where, f):
    g = _grid_of(where)
    f = np.ascontiguousarray(f, dtype=np.float64)
    if f.size != g.nx * g.ny:
        raise InvalidArgument("field does not match the grid")
    return f.reshape(g.ny, g.nx)


def obs_operator(field, obs: ObsSet, grid) -> np.ndarray:
    """H: bilinear interpolation at each observation (obs.cpp:59-71).
    `grid`: the field's Grid2D (or an operator on it)."""
    f = _field2d(grid, field)
    d = _DeviceObs(grid, obs)
    out = np.empty(d.n)
    if d.n:
        _check(lib.rgf_obs_apply(d._h, 0, _ptr(f), _ptr(out), 0, None))
    return out


def obs_operator_transpose(vec, obs: ObsSet, grid) -> np.ndarray:
    """H^T: scatter with the same bilinear weights (obs.cpp:73-87)."""
    v = np.ascontiguousarray(vec, dtype=np.float64).reshape(-1)
    d = _DeviceObs(grid, obs)
    if v.size != d.n:
        raise InvalidArgument("obs_operator_transpose: vector length mismatch")
    g = _grid_of(grid)
    out = np.empty((g.ny, g.nx))
    _check(lib.rgf_obs_apply(d._h, 1, _ptr(v) if v.size else _ptr(out), _ptr(out), 0, None))
    return out


def misfit(background_at_obs, obs: ObsSet) -> np.ndarray:
    """d = y - H(x_b) (obs.cpp:89-93)."""
    b = np.asarray(background_at_obs, dtype=np.float64).reshape(-1)
    y = np.asarray(obs.values, dtype=np.float64).reshape(-1)
    if b.size != y.size:
        raise InvalidArgument("misfit: vector length mismatch")
    return y - b


def cost(chi, obs: ObsSet, op: "HorizontalCovarianceOp", background=None) -> CostReport:
    """J(chi) and its gradient (solver.cpp:35-50)."""
    c = _field2d(op, chi)
    bg = None if background is None else _field2d(op, background)
    d = _DeviceObs(op, obs)
    j3 = np.empty(3)
    grad = np.empty_like(c)
    _check(lib.rgf_cost(op._h, d._h, _ptr(c), None if bg is None else _ptr(bg), _ptr(j3),
                        _ptr(grad)))
    return CostReport(float(j3[0]), float(j3[1]), float(j3[2]), grad)


def solve(obs: ObsSet, op: "HorizontalCovarianceOp", options: SolveOptions = SolveOptions(),
          background=None) -> Analysis:
    """CG on (I + V^T H^T R^-1 H V) chi = V^T H^T R^-1 d, increment V chi
    (solver.cpp:52-114), on the device."""
    if not (options.tol > 0):
        raise InvalidArgument("solve: tol must be positive")
    if options.max_iter < 0:
        raise InvalidArgument("solve: max_iter must be >= 0")
    bg = None if background is None else _field2d(op, background)
    d = _DeviceObs(op, obs)
    g = op.grid()
    inc = np.empty((g.ny, g.nx))
    mis = np.empty(max(d.n, 1))
    gn = np.empty(options.max_iter + 1)
    an = _Analysis()
    _check(lib.rgf_solve(op._h, d._h, float(options.tol), int(options.max_iter),
                         None if bg is None else _ptr(bg), _ptr(inc), _ptr(mis), _ptr(gn),
                         ctypes.byref(an)))
    return Analysis(inc, mis[:d.n].copy(), int(an.cg_iterations),
                    list(gn[:an.n_gradient_norms]), bool(an.converged),
                    float(an.final_relative_residual), float(an.j_background), float(an.j_obs))


__all__ += ["ObsSet", "SolveOptions", "Analysis", "CostReport", "obs_operator",
            "obs_operator_transpose", "misfit", "cost", "solve"]
