// Operator-construction kernels: validation, per-level sigma statistics,
// coefficient precompute (elementwise), and the land-mask segmentation
// scan/compaction. All run once per HorizontalCovarianceOp
// (covariance.cpp:155-220), outside the timed filter applications.
#pragma once
#include "common.cuh"

namespace rgfb {

// ------------------------------------------------------------ validation
// grid.cpp:33-34: first non-positive spacing (linear index), atomicMin.
__global__ void k_check_spacing(const double* dx, const double* dy, int64_t nh,
                                unsigned long long* first_bad) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nh;
       p += (int64_t)gridDim.x * blockDim.x)
    if (!(dx[p] > 0) || !(dy[p] > 0)) atomicMin(first_bad, (unsigned long long)p);
}

// grid.cpp:41-55 ScaleField::validate per level (first failing sea point in
// [lev][j][i] order), plus the union-of-levels sea map used for the shared
// coefficient tables.
__global__ void k_check_scales(const double* rx, const double* ry, const double* dx,
                               const double* dy, const uint8_t* mask, int64_t nh,
                               int64_t nlev, unsigned long long* first_bad,
                               uint8_t* any_sea) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nh;
       p += (int64_t)gridDim.x * blockDim.x) {
    const double sx = ddiv(rx[p], dx[p]);
    const double sy = ddiv(ry[p], dy[p]);
    const bool bad = !(rx[p] > 0) || !(ry[p] > 0) || !isfinite(sx) || !isfinite(sy);
    uint8_t s = 0;
    for (int64_t l = 0; l < nlev; ++l) {
      if (mask[l * nh + p]) {
        s = 1;
        if (bad) {
          atomicMin(first_bad, (unsigned long long)(l * nh + p));
          break;
        }
      }
    }
    any_sea[p] = s;
  }
}

// --------------------------------------------------- per-level statistics
// grid.cpp:57-67 sigma_x/sigma_y with land = 1 (mask.select) and max_sigma;
// covariance.cpp:207 uniform test (min == max). sigma > 0 everywhere, so the
// IEEE bit pattern orders like the value and integer atomics are exact.
// stats[l*4 + {0,1,2,3}] = {min sx, max sx, min sy, max sy} as bit patterns.
__global__ void k_level_stats(const double* rx, const double* ry, const double* dx,
                              const double* dy, const uint8_t* mask, int64_t nh,
                              unsigned long long* stats) {
  // grid: (blocks, nlev); blockIdx.y is the level
  const int64_t l = blockIdx.y;
  unsigned long long mnx = ~0ull, mxx = 0, mny = ~0ull, mxy = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nh;
       p += (int64_t)gridDim.x * blockDim.x) {
    const bool sea = mask[l * nh + p] != 0;
    const unsigned long long bx = __double_as_longlong(sea ? ddiv(rx[p], dx[p]) : 1.0);
    const unsigned long long by = __double_as_longlong(sea ? ddiv(ry[p], dy[p]) : 1.0);
    mnx = bx < mnx ? bx : mnx;
    mxx = bx > mxx ? bx : mxx;
    mny = by < mny ? by : mny;
    mxy = by > mxy ? by : mxy;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mnx, o);
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, mxx, o);
    const unsigned long long c = __shfl_xor_sync(0xffffffffu, mny, o);
    const unsigned long long d = __shfl_xor_sync(0xffffffffu, mxy, o);
    mnx = a < mnx ? a : mnx;
    mxx = b > mxx ? b : mxx;
    mny = c < mny ? c : mny;
    mxy = d > mxy ? d : mxy;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&stats[l * 4 + 0], mnx);
    atomicMax(&stats[l * 4 + 1], mxx);
    atomicMin(&stats[l * 4 + 2], mny);
    atomicMax(&stats[l * 4 + 3], mxy);
  }
}

// ------------------------------------------------- coefficient precompute
// covariance.cpp:182-206 `build`: sigma = r/d where any level is sea (else 1,
// the select of grid.cpp:58), then rf3_filter_scalars (+ inv_dc) or
// rf1_coefficients per point. One thread per horizontal point.
__global__ void k_coefficients(const double* r, const double* d, const uint8_t* any_sea,
                               int64_t nh, int order, int k, int calibration, int unit_dc,
                               Coef3* c3, double2* c1, double* idc) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nh;
       p += (int64_t)gridDim.x * blockDim.x) {
    const double sigma = any_sea[p] ? ddiv(r[p], d[p]) : 1.0;
    if (order == 1) {
      const double a = rf1_alpha(sigma, k);
      c1[p] = make_double2(a, dsub(1.0, a));
    } else {
      const Scal3 f = rf3_filter_scalars(sigma, calibration);
      c3[p] = Coef3{f.alpha1, f.alpha2, f.alpha3, f.beta};
      if (unit_dc) idc[p] = inv_dc(sigma);
    }
  }
}

// Scalar builders for the C ABI helpers and the 1-D entry points.
__global__ void k_scalar_coefficients(double sigma, int calibration, int k, double* out) {
  if (threadIdx.x != 0) return;
  const Poly3 t = rf3_coefficients(sigma);
  out[0] = t.a0; out[1] = t.a1; out[2] = t.a2; out[3] = t.a3;
  out[4] = t.alpha1; out[5] = t.alpha2; out[6] = t.alpha3; out[7] = t.beta;
  const Scal3 f = rf3_filter_scalars(sigma, calibration);
  out[8] = f.alpha1; out[9] = f.alpha2; out[10] = f.alpha3; out[11] = f.beta; out[12] = f.q;
  if (k >= 1) {
    const double a = rf1_alpha(sigma, k);
    out[13] = a;
    out[14] = dsub(1.0, a);
  }
}

// ---------------------------------------------------------- segmentation
// covariance.cpp:246-258: maximal sea runs [i, j] of one line. Lines of
// direction x are (lev, iy) scanning ix; of direction y (lev, ix) scanning
// iy. Pass 1 counts runs per line; a device exclusive scan gives offsets;
// pass 2 writes (start, len) descriptors in order. Indexing is exact
// integer work (bit-identical to the reference's enumeration).
__device__ __forceinline__ bool line_sea(const uint8_t* mask, int dir, int64_t nx, int64_t ny,
                                         int64_t line, int64_t k) {
  // line = lev*ny + iy (dir 0) or lev*nx + ix (dir 1)
  if (dir == 0) {
    return mask[line * nx + k] != 0;
  } else {
    const int64_t lev = line / nx, ix = line - lev * nx;
    return mask[(lev * ny + k) * nx + ix] != 0;
  }
}

__global__ void k_seg_count(const uint8_t* mask, int dir, int64_t nx, int64_t ny,
                            int64_t nlines, int64_t* counts) {
  const int64_t n = dir == 0 ? nx : ny;
  for (int64_t line = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; line < nlines;
       line += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    bool prev = false;
    for (int64_t k = 0; k < n; ++k) {
      const bool s = line_sea(mask, dir, nx, ny, line, k);
      c += (s && !prev);
      prev = s;
    }
    counts[line] = c;
  }
}

__global__ void k_seg_fill(const uint8_t* mask, int dir, int64_t nx, int64_t ny,
                           int64_t nlines, const int64_t* offsets, int2* segs,
                           int32_t* seg_line) {
  const int64_t n = dir == 0 ? nx : ny;
  for (int64_t line = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; line < nlines;
       line += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = offsets[line];
    int64_t i = 0;
    while (i < n) {
      if (!line_sea(mask, dir, nx, ny, line, i)) {
        ++i;
        continue;
      }
      int64_t j = i;
      while (j + 1 < n && line_sea(mask, dir, nx, ny, line, j + 1)) ++j;
      seg_line[o] = static_cast<int32_t>(line);  // (lev, line) of this segment
      segs[o++] = make_int2((int)i, (int)(j - i + 1));
      i = j + 1;
    }
  }
}

// Sort key of every segment for the closure pass: (line, end position, level),
// so the levels sharing a segment end are adjacent (shared closure rows).
__global__ void k_seg_keys(const int2* segs, const int32_t* seg_line, int64_t nsegs,
                           int64_t nlines, int64_t n, int64_t nlev, uint64_t* keys,
                           int64_t* idx) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nsegs;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lg = seg_line[s];
    const int64_t lev = lg / nlines, line = lg - lev * nlines;
    const int64_t j = segs[s].x + segs[s].y - 1;
    keys[s] = static_cast<uint64_t>((line * n + j) * nlev + lev);
    idx[s] = s;
  }
}

}  // namespace rgfb
