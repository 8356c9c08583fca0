"""CPU ORACLE binding — TEST INFRASTRUCTURE ONLY.

ctypes wrapper over ``oracle/librgf_oracle.so``, the Eigen-free C++
restatement of the reference hot path (see rgf_oracle.h). Imported only by
tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs, as the
checker or the timed CPU baseline; the product package never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librgf_oracle.so")


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return LIB_PATH


build()
lib = ctypes.CDLL(LIB_PATH)

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_d = ctypes.c_double
lib.rgfo_last_error.restype = ctypes.c_char_p
lib.rgfo_rf3_coefficients.argtypes = [_d, _vp]
lib.rgfo_rf3_filter_scalars.argtypes = [_d, ctypes.c_int, _vp]
lib.rgfo_rf3_cascade_variance.argtypes = [_d]
lib.rgfo_rf3_cascade_variance.restype = _d
lib.rgfo_rf3_length_scale_argument.argtypes = [_d, ctypes.c_int]
lib.rgfo_rf3_length_scale_argument.restype = _d
lib.rgfo_rf1_coefficients.argtypes = [_d, ctypes.c_int, _vp]
lib.rgfo_rational_gauss.argtypes = [_d]
lib.rgfo_rational_gauss.restype = _d
lib.rgfo_rf3_apply_1d.argtypes = [_vp, _vp, _i64, ctypes.c_int, ctypes.c_int, _vp]
lib.rgfo_rf1_apply_1d.argtypes = [_vp, _vp, _i64, ctypes.c_int, ctypes.c_int, _vp]
lib.rgfo_rf3_apply_1d_coeffs.argtypes = [_vp, _vp, _vp, _vp, _vp, _i64, ctypes.c_int, _vp]
lib.rgfo_op_create.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp, _i64, _vp, _vp, ctypes.c_int,
                               ctypes.c_int, ctypes.c_int, _i64, _vp, ctypes.c_int,
                               ctypes.c_int, ctypes.POINTER(_vp)]
lib.rgfo_op_destroy.argtypes = [_vp]
lib.rgfo_op_apply.argtypes = [_vp, ctypes.c_int, _vp, _vp, _i64, _i64, _i64]
lib.rgfo_op_ghost_width.argtypes = [_vp, _i64]
lib.rgfo_op_ghost_width.restype = _i64
lib.rgfo_op_coefficient_bytes.argtypes = [_vp]
lib.rgfo_op_coefficient_bytes.restype = ctypes.c_uint64
lib.rgfo_obs_create.argtypes = [_vp, _i64, _vp, _vp, _vp, _vp, _vp]
lib.rgfo_obs_destroy.argtypes = [_vp]
lib.rgfo_obs_apply.argtypes = [_vp, _vp, ctypes.c_int, _vp, _vp]
lib.rgfo_cost.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
lib.rgfo_solve.argtypes = [_vp, _vp, _d, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp]
lib.rgfo_op_uniform.argtypes = [_vp, _i64, ctypes.c_int]
lib.rgfo_resolve_thread_count.argtypes = [ctypes.c_int]
lib.rgfo_io_last_error.restype = ctypes.c_char_p
lib.rgfo_diag_last_error.restype = ctypes.c_char_p
lib.rgfo_impulse_response.argtypes = [_d, ctypes.c_int, ctypes.c_int, _i64, ctypes.c_int, _vp,
                                      _vp, _vp, _vp]
lib.rgfo_remark1.argtypes = [_vp, _i64, _d, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp]
lib.rgfo_load_grid.argtypes = [ctypes.c_char_p, _i64, _i64, _vp, _vp, _vp, ctypes.POINTER(_i64)]
lib.rgfo_save_grid.argtypes = [ctypes.c_char_p, _i64, _i64, _i64, _vp, _vp, _vp]
lib.rgfo_load_scale.argtypes = [ctypes.c_char_p, _i64, _i64, _vp, _vp]
lib.rgfo_save_scale.argtypes = [ctypes.c_char_p, _i64, _i64, _vp, _vp]
lib.rgfo_load_field.argtypes = [ctypes.c_char_p, _i64, _i64, _vp]
lib.rgfo_save_field.argtypes = [ctypes.c_char_p, _i64, _i64, _vp]

GX, GY, GXT, GYT, V, VT, B, GYGX = range(8)


class OracleError(ValueError):
    pass


def _check(status):
    if status != 0:
        raise OracleError(lib.rgfo_last_error().decode())


def _p(a):
    return a.ctypes.data


def rf3_coefficients(sigma):
    out = np.zeros(8)
    _check(lib.rgfo_rf3_coefficients(float(sigma), _p(out)))
    return out  # a0 a1 a2 a3 alpha1 alpha2 alpha3 beta


def rf3_filter_scalars(sigma, calibration=0):
    out = np.zeros(5)
    _check(lib.rgfo_rf3_filter_scalars(float(sigma), int(calibration), _p(out)))
    return out  # alpha1 alpha2 alpha3 beta q


def rf1_coefficients(sigma, k):
    out = np.zeros(2)
    _check(lib.rgfo_rf1_coefficients(float(sigma), int(k), _p(out)))
    return out


def rf3_cascade_variance(q):
    return lib.rgfo_rf3_cascade_variance(float(q))


def rf3_length_scale_argument(sigma, calibration):
    return lib.rgfo_rf3_length_scale_argument(float(sigma), int(calibration))


def rational_gauss(t):
    return lib.rgfo_rational_gauss(float(t))


def rf3_apply_1d(x, sigma, calibration=0, transpose=False):
    x = np.ascontiguousarray(x, dtype=np.float64)
    sig = np.ascontiguousarray(np.broadcast_to(np.asarray(sigma, dtype=np.float64), x.shape))
    out = np.empty_like(x)
    _check(lib.rgfo_rf3_apply_1d(_p(x), _p(sig), x.size, int(calibration), int(transpose),
                                 _p(out)))
    return out


def rf1_apply_1d(x, sigma, k, transpose=False):
    x = np.ascontiguousarray(x, dtype=np.float64)
    sig = np.ascontiguousarray(np.broadcast_to(np.asarray(sigma, dtype=np.float64), x.shape))
    out = np.empty_like(x)
    _check(lib.rgfo_rf1_apply_1d(_p(x), _p(sig), x.size, int(k), int(transpose), _p(out)))
    return out


def rf3_apply_1d_coeffs(x, a1, a2, a3, b, transpose=False):
    arrs = [np.ascontiguousarray(v, dtype=np.float64) for v in (x, a1, a2, a3, b)]
    out = np.empty_like(arrs[0])
    _check(lib.rgfo_rf3_apply_1d_coeffs(*(_p(v) for v in arrs), arrs[0].size, int(transpose),
                                        _p(out)))
    return out


class OracleOp:
    """Loop of per-level 2-D HorizontalCovarianceOp instances (CPU)."""

    def __init__(self, nx, ny, dx, dy, mask, rx, ry, order=3, k_iterations=1, unit_dc=True,
                 ghost_width=None, grid_ghost_width=0, variance=None, threads=1,
                 calibration=0):
        self.nx, self.ny = int(nx), int(ny)
        mask = np.asarray(mask)
        self.nlev = 1 if mask.ndim == 2 else mask.shape[0]
        self._keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (dx, dy, rx, ry)]
        self._mask = np.ascontiguousarray(mask.reshape(self.nlev, ny, nx), dtype=np.uint8)
        var = None
        if variance is not None:
            var = np.ascontiguousarray(np.broadcast_to(
                np.asarray(variance, dtype=np.float64).reshape(-1, ny, nx), (self.nlev, ny, nx)))
            self._keep.append(var)
        h = _vp()
        dxa, dya, rxa, rya = self._keep[:4]
        _check(lib.rgfo_op_create(self.nx, self.ny, self.nlev, _p(dxa), _p(dya), _p(self._mask),
                                  int(grid_ghost_width), _p(rxa), _p(rya), int(order),
                                  int(k_iterations), 1 if unit_dc else 0,
                                  -1 if ghost_width is None else int(ghost_width),
                                  None if var is None else _p(var), int(threads),
                                  int(calibration), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if lib is None:  # interpreter teardown
            return
        if getattr(self, "_h", None):
            lib.rgfo_op_destroy(self._h)
            self._h = None

    def ghost_width(self, level=0):
        return lib.rgfo_op_ghost_width(self._h, level)

    def coefficient_bytes(self):
        return lib.rgfo_op_coefficient_bytes(self._h)

    def uniform(self, level, direction):
        return bool(lib.rgfo_op_uniform(self._h, level, direction))

    def apply(self, kind, field, lev0=0, nlev_sub=0):
        f = np.ascontiguousarray(field, dtype=np.float64)
        planes = nlev_sub if nlev_sub > 0 else self.nlev
        nvar = f.size // (self.nx * self.ny * planes)
        out = np.empty_like(f)
        _check(lib.rgfo_op_apply(self._h, kind, _p(f), _p(out), nvar, lev0, nlev_sub))
        return out


# ------------------------------------------------------------- obs + CG
class OracleObs:
    """ObsSet on a one-level OracleOp (obs.cpp:18-93): positions (n, 2) in
    fractional grid indices (x, y), values, r_var."""

    def __init__(self, op, positions, values, r_var):
        pos = np.asarray(positions, dtype=np.float64).reshape(-1, 2)
        self.op = op
        self.n = pos.shape[0]
        self._keep = [np.ascontiguousarray(pos[:, 0]), np.ascontiguousarray(pos[:, 1]),
                      np.ascontiguousarray(values, dtype=np.float64),
                      np.ascontiguousarray(r_var, dtype=np.float64)]
        h = _vp()
        _check(lib.rgfo_obs_create(op._h, self.n, *(_p(a) for a in self._keep), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if lib is None:  # interpreter teardown
            return
        if getattr(self, "_h", None):
            lib.rgfo_obs_destroy(self._h)
            self._h = None

    def h(self, field):
        f = np.ascontiguousarray(field, dtype=np.float64)
        out = np.empty(self.n)
        _check(lib.rgfo_obs_apply(self.op._h, self._h, 0, _p(f), _p(out)))
        return out

    def ht(self, vec):
        v = np.ascontiguousarray(vec, dtype=np.float64)
        out = np.empty((self.op.ny, self.op.nx))
        _check(lib.rgfo_obs_apply(self.op._h, self._h, 1, _p(v), _p(out)))
        return out

    def cost(self, chi, background=None):
        c = np.ascontiguousarray(chi, dtype=np.float64)
        bg = None if background is None else np.ascontiguousarray(background, dtype=np.float64)
        j3 = np.empty(3)
        g = np.empty_like(c)
        _check(lib.rgfo_cost(self.op._h, self._h, _p(c), None if bg is None else _p(bg), _p(j3),
                             _p(g)))
        return {"j_total": j3[0], "j_background": j3[1], "j_obs": j3[2], "gradient": g}

    def solve(self, tol=1e-6, max_iter=30, background=None):
        bg = None if background is None else np.ascontiguousarray(background, dtype=np.float64)
        inc = np.empty((self.op.ny, self.op.nx))
        mis = np.empty(max(self.n, 1))
        gn = np.empty(max_iter + 1)
        info = np.zeros(3, dtype=np.int64)
        out3 = np.empty(3)
        _check(lib.rgfo_solve(self.op._h, self._h, float(tol), int(max_iter),
                              None if bg is None else _p(bg), _p(inc), _p(mis), _p(gn),
                              info.ctypes.data_as(ctypes.c_void_p), _p(out3)))
        return {"increment": inc, "misfit": mis[:self.n], "cg_iterations": int(info[0]),
                "converged": bool(info[1]), "gradient_norms": gn[:int(info[2])],
                "final_relative_residual": out3[0], "j_background": out3[1], "j_obs": out3[2]}


# ---------------------------------------------------------------- container I/O
# io.cpp:133-281 restated with nlohmann::json (rgf_oracle_io.cpp). Arrays are
# (ny, nx), x fastest, as in the containers.
def _io_check(status):
    if status != 0:
        raise OracleError(lib.rgfo_io_last_error().decode())


def load_grid(path, nx, ny):
    dx, dy = np.empty((ny, nx)), np.empty((ny, nx))
    mask = np.empty((ny, nx), dtype=np.uint8)
    g = _i64()
    _io_check(lib.rgfo_load_grid(str(path).encode(), nx, ny, _p(dx), _p(dy), _p(mask),
                                 ctypes.byref(g)))
    return dx, dy, mask.astype(bool), g.value


def save_grid(path, dx, dy, mask, ghost_width=0):
    ny, nx = np.shape(dx)
    arrs = [np.ascontiguousarray(dx, dtype=np.float64), np.ascontiguousarray(dy, dtype=np.float64),
            np.ascontiguousarray(mask, dtype=np.uint8)]
    _io_check(lib.rgfo_save_grid(str(path).encode(), nx, ny, int(ghost_width), *(_p(a) for a in arrs)))


def load_scale(path, nx, ny):
    rx, ry = np.empty((ny, nx)), np.empty((ny, nx))
    _io_check(lib.rgfo_load_scale(str(path).encode(), nx, ny, _p(rx), _p(ry)))
    return rx, ry


def save_scale(path, rx, ry):
    ny, nx = np.shape(rx)
    a, b = (np.ascontiguousarray(v, dtype=np.float64) for v in (rx, ry))
    _io_check(lib.rgfo_save_scale(str(path).encode(), nx, ny, _p(a), _p(b)))


def load_field(path, nx, ny):
    v = np.empty((ny, nx))
    _io_check(lib.rgfo_load_field(str(path).encode(), nx, ny, _p(v)))
    return v


def save_field(path, values):
    ny, nx = np.shape(values)
    v = np.ascontiguousarray(values, dtype=np.float64)
    _io_check(lib.rgfo_save_field(str(path).encode(), nx, ny, _p(v)))


# ---------------------------------------------------------------- diagnostics
def impulse_response(sigma, order, k, length, calibration=0):
    """diagnostics.cpp:69-96 -> (h, sum_h, err_h_l2, err_h_max)."""
    h = np.empty(length)
    o = np.empty(3)
    if lib.rgfo_impulse_response(float(sigma), int(order), int(k), int(length), int(calibration),
                                 _p(h), _p(o[0:]), _p(o[1:]), _p(o[2:])) != 0:
        raise OracleError(lib.rgfo_diag_last_error().decode())
    return h, o[0], o[1], o[2]


def remark1(s0, sigma, order, k, calibration=0):
    """diagnostics.cpp:102-135 -> (lhs, rhs, err_h_l2, holds)."""
    x = np.ascontiguousarray(s0, dtype=np.float64)
    o = np.empty(4)
    if lib.rgfo_remark1(_p(x), x.size, float(sigma), int(order), int(k), int(calibration),
                        _p(o)) != 0:
        raise OracleError(lib.rgfo_diag_last_error().decode())
    return o[0], o[1], o[2], bool(o[3])
