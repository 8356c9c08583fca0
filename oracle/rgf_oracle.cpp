/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY (see rgf_oracle.h).
 *
 * Restates the reference hot path without Eigen. Every function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Build: oracle/Makefile (-O3 -DNDEBUG -ffp-contract=off, no -march=native),
 * matching the reference's CMake Release build (src/CMakeLists.txt:12).
 */
#include "rgf_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <numbers>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_last_error;

using Index = int64_t;

// ---------------------------------------------------------------- rf3.hpp
// rf3.hpp:46-66 (printed table; RGF_USE_APPENDIX_A_CONSTANTS selects the
// alternate set, mirrored here by the same macro).
namespace c3 {
#ifdef RGF_USE_APPENDIX_A_CONSTANTS
constexpr double c00 = 3.738128, c01 = 5.788982, c02 = 3.382472, c11 = 5.788824,
                 c12 = 6.764946, c13 = 2.999999, c22 = -3.382472, c23 = -2.999999;
#else
constexpr double c00 = 3.738128, c01 = 5.788982, c02 = 3.382473, c11 = 5.788982,
                 c12 = 6.764946, c13 = 3.0, c22 = -3.382473, c23 = -3.0;
#endif
}  // namespace c3

struct Poly {
  double a0, a1, a2, a3, alpha1, alpha2, alpha3, beta;
};

// rf3.hpp:78-95
Poly rf3_coefficients(double sigma) {
  using namespace c3;
  if (!(sigma > 0.0)) throw std::invalid_argument("rf3_coefficients: sigma must be positive");
  const double x = sigma, x2 = x * x, x3 = x2 * x;
  Poly t;
  t.a0 = c00 + c01 * x + c02 * x2 + x3;
  t.a1 = c11 * x + c12 * x2 + c13 * x3;
  t.a2 = c22 * x2 + c23 * x3;
  t.a3 = x3;
  t.alpha1 = t.a1 / t.a0;
  t.alpha2 = t.a2 / t.a0;
  t.alpha3 = t.a3 / t.a0;
  t.beta = std::pow(2.0 * std::numbers::pi * sigma * sigma, 0.25) *
           (1.0 - (t.alpha1 + t.alpha2 + t.alpha3));
  return t;
}

// rf3.hpp:101-108
double rf3_cascade_variance(double q) {
  const Poly t = rf3_coefficients(q);
  const double a = 1.0 - (t.alpha1 + t.alpha2 + t.alpha3);
  const double s1 = t.alpha1 + 2.0 * t.alpha2 + 3.0 * t.alpha3;
  const double s2 = 2.0 * t.alpha2 + 6.0 * t.alpha3;
  return 2.0 * (s1 * s1 / (a * a) + (s1 + s2) / a);
}

// rf3.hpp:116-126
double yvv95_argument(double sigma) {
  double q;
  if (sigma >= 2.5) {
    q = 0.98711 * sigma - 0.96330;
  } else {
    const double arg = std::max(1.0 - 0.26891 * sigma, 0.0);
    q = 3.97156 - 4.14554 * std::sqrt(arg);
  }
  return std::max(q, 0.01);
}

// rf3.hpp:128-139
double variance_matched_argument(double sigma) {
  const double target = sigma * sigma;
  double lo = 1e-12;
  double hi = std::max(sigma, 1.0);
  while (rf3_cascade_variance(hi) < target) hi *= 2.0;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    (rf3_cascade_variance(mid) < target ? lo : hi) = mid;
  }
  return 0.5 * (lo + hi);
}

// rf3.hpp:143-154 (types.hpp:39: yvv95=0, variance_match=1, none=2)
double rf3_length_scale_argument(double sigma, int calibration) {
  switch (calibration) {
    case 0: return yvv95_argument(sigma);
    case 1: return variance_matched_argument(sigma);
    case 2: return sigma;
  }
  return sigma;
}

struct Scalars3 {
  double alpha1, alpha2, alpha3, beta, q;
};

// rf3.hpp:166-181
Scalars3 rf3_filter_scalars(double sigma, int calibration) {
  if (!(sigma > 0.0)) throw std::invalid_argument("rf3_filter_scalars: sigma must be positive");
  const double q = rf3_length_scale_argument(sigma, calibration);
  const Poly t = rf3_coefficients(q);
  Scalars3 f;
  f.alpha1 = t.alpha1;
  f.alpha2 = t.alpha2;
  f.alpha3 = t.alpha3;
  f.beta = std::pow(2.0 * std::numbers::pi * sigma * sigma, 0.25) *
           (1.0 - (t.alpha1 + t.alpha2 + t.alpha3));
  f.q = q;
  return f;
}

// rf3.hpp:217-239 (startup rows written out as in the reference)
void rf3_forward(double* s, const double* a1, const double* a2, const double* a3,
                 const double* b, Index m) {
  double pm1 = b[0] * s[0];
  s[0] = pm1;
  double t = b[1] * s[1] + a1[1] * pm1;
  s[1] = t;
  double pm2 = pm1;
  pm1 = t;
  t = b[2] * s[2] + a1[2] * pm1 + a2[2] * pm2;
  s[2] = t;
  double pm3 = pm2;
  pm2 = pm1;
  pm1 = t;
  for (Index i = 3; i < m; ++i) {
    t = b[i] * s[i] + a1[i] * pm1 + a2[i] * pm2 + a3[i] * pm3;
    pm3 = pm2;
    pm2 = pm1;
    pm1 = t;
    s[i] = t;
  }
}

// rf3.hpp:241-262
void rf3_backward(double* s, const double* a1, const double* a2, const double* a3,
                  const double* b, Index m) {
  double pm1 = b[m - 1] * s[m - 1];
  s[m - 1] = pm1;
  double t = b[m - 2] * s[m - 2] + a1[m - 2] * pm1;
  s[m - 2] = t;
  double pm2 = pm1;
  pm1 = t;
  t = b[m - 3] * s[m - 3] + a1[m - 3] * pm1 + a2[m - 3] * pm2;
  s[m - 3] = t;
  double pm3 = pm2;
  pm2 = pm1;
  pm1 = t;
  for (Index i = m - 4; i >= 0; --i) {
    t = b[i] * s[i] + a1[i] * pm1 + a2[i] * pm2 + a3[i] * pm3;
    pm3 = pm2;
    pm2 = pm1;
    pm1 = t;
    s[i] = t;
  }
}

// rf3.hpp:264-274
void rf3_forward_transpose(double* w, const double* a1, const double* a2,
                           const double* a3, const double* b, Index m) {
  for (Index i = m - 1; i >= 0; --i) {
    const double wi = w[i];
    if (i >= 1) w[i - 1] += a1[i] * wi;
    if (i >= 2) w[i - 2] += a2[i] * wi;
    if (i >= 3) w[i - 3] += a3[i] * wi;
    w[i] = b[i] * wi;
  }
}

// rf3.hpp:276-286
void rf3_backward_transpose(double* w, const double* a1, const double* a2,
                            const double* a3, const double* b, Index m) {
  for (Index i = 0; i < m; ++i) {
    const double wi = w[i];
    if (i + 1 < m) w[i + 1] += a1[i] * wi;
    if (i + 2 < m) w[i + 2] += a2[i] * wi;
    if (i + 3 < m) w[i + 3] += a3[i] * wi;
    w[i] = b[i] * wi;
  }
}

// ---------------------------------------------------------------- rf1.hpp
// rf1.hpp:20-29
void rf1_forward(double* s, const double* a, const double* b, Index m) {
  double prev = b[0] * s[0];
  s[0] = prev;
  for (Index i = 1; i < m; ++i) {
    prev = b[i] * s[i] + a[i] * prev;
    s[i] = prev;
  }
}
// rf1.hpp:31-39
void rf1_backward(double* s, const double* a, const double* b, Index m) {
  double prev = b[m - 1] * s[m - 1];
  s[m - 1] = prev;
  for (Index i = m - 2; i >= 0; --i) {
    prev = b[i] * s[i] + a[i] * prev;
    s[i] = prev;
  }
}
// rf1.hpp:43-52
void rf1_forward_transpose(double* w, const double* a, const double* b, Index m) {
  double prev = w[m - 1];
  w[m - 1] = b[m - 1] * prev;
  for (Index i = m - 2; i >= 0; --i) {
    const double cur = w[i] + a[i + 1] * prev;
    w[i] = b[i] * cur;
    prev = cur;
  }
}
// rf1.hpp:54-63
void rf1_backward_transpose(double* w, const double* a, const double* b, Index m) {
  double prev = w[0];
  w[0] = b[0] * prev;
  for (Index i = 1; i < m; ++i) {
    const double cur = w[i] + a[i - 1] * prev;
    w[i] = b[i] * cur;
    prev = cur;
  }
}

struct Scalars1 {
  double alpha, beta;
};
// rf1.hpp:76-85
Scalars1 rf1_coefficients(double sigma, int k) {
  if (!(sigma > 0.0)) throw std::invalid_argument("rf1_coefficients: sigma must be positive");
  if (k < 1) throw std::invalid_argument("rf1_coefficients: k must be >= 1");
  const double q = double(k) / (sigma * sigma);
  const double root = std::sqrt(q * (q + 2.0));
  const double alpha = 1.0 + q - root;
  return {alpha, 1.0 - alpha};
}

// ------------------------------------------- covariance.cpp scalar twins
// covariance.cpp:49-151 — identical arithmetic to the per-point kernels.
void rf1_forward_u(double* s, double a, double b, Index m) {
  double prev = b * s[0];
  s[0] = prev;
  for (Index i = 1; i < m; ++i) {
    prev = b * s[i] + a * prev;
    s[i] = prev;
  }
}
void rf1_backward_u(double* s, double a, double b, Index m) {
  double prev = b * s[m - 1];
  s[m - 1] = prev;
  for (Index i = m - 2; i >= 0; --i) {
    prev = b * s[i] + a * prev;
    s[i] = prev;
  }
}
void rf1_forward_transpose_u(double* w, double a, double b, Index m) {
  double prev = w[m - 1];
  w[m - 1] = b * prev;
  for (Index i = m - 2; i >= 0; --i) {
    const double cur = w[i] + a * prev;
    w[i] = b * cur;
    prev = cur;
  }
}
void rf1_backward_transpose_u(double* w, double a, double b, Index m) {
  double prev = w[0];
  w[0] = b * prev;
  for (Index i = 1; i < m; ++i) {
    const double cur = w[i] + a * prev;
    w[i] = b * cur;
    prev = cur;
  }
}
void rf3_forward_u(double* s, double a1, double a2, double a3, double b, Index m) {
  double pm1 = b * s[0];
  s[0] = pm1;
  double t = b * s[1] + a1 * pm1;
  s[1] = t;
  double pm2 = pm1;
  pm1 = t;
  t = b * s[2] + a1 * pm1 + a2 * pm2;
  s[2] = t;
  double pm3 = pm2;
  pm2 = pm1;
  pm1 = t;
  for (Index i = 3; i < m; ++i) {
    t = b * s[i] + a1 * pm1 + a2 * pm2 + a3 * pm3;
    pm3 = pm2;
    pm2 = pm1;
    pm1 = t;
    s[i] = t;
  }
}
void rf3_backward_u(double* s, double a1, double a2, double a3, double b, Index m) {
  double pm1 = b * s[m - 1];
  s[m - 1] = pm1;
  double t = b * s[m - 2] + a1 * pm1;
  s[m - 2] = t;
  double pm2 = pm1;
  pm1 = t;
  t = b * s[m - 3] + a1 * pm1 + a2 * pm2;
  s[m - 3] = t;
  double pm3 = pm2;
  pm2 = pm1;
  pm1 = t;
  for (Index i = m - 4; i >= 0; --i) {
    t = b * s[i] + a1 * pm1 + a2 * pm2 + a3 * pm3;
    pm3 = pm2;
    pm2 = pm1;
    pm1 = t;
    s[i] = t;
  }
}
void rf3_forward_transpose_u(double* w, double a1, double a2, double a3, double b,
                             Index m) {
  for (Index i = m - 1; i >= 0; --i) {
    const double wi = w[i];
    if (i >= 1) w[i - 1] += a1 * wi;
    if (i >= 2) w[i - 2] += a2 * wi;
    if (i >= 3) w[i - 3] += a3 * wi;
    w[i] = b * wi;
  }
}
void rf3_backward_transpose_u(double* w, double a1, double a2, double a3, double b,
                              Index m) {
  for (Index i = 0; i < m; ++i) {
    const double wi = w[i];
    if (i + 1 < m) w[i + 1] += a1 * wi;
    if (i + 2 < m) w[i + 2] += a2 * wi;
    if (i + 3 < m) w[i + 3] += a3 * wi;
    w[i] = b * wi;
  }
}

// ------------------------------------------------------------ parallel.hpp
// parallel.hpp:18-22
int resolve_thread_count(int requested) {
  if (requested > 0) return requested;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1 : static_cast<int>(hw);
}

// parallel.hpp:26-44: contiguous chunks, one thread per chunk, spawned per call.
template <typename F>
void parallel_for(Index n, int threads, F&& f) {
  threads = static_cast<int>(std::min<Index>(resolve_thread_count(threads), n));
  if (threads <= 1) {
    for (Index i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> pool;
  pool.reserve(threads);
  const Index chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const Index begin = t * chunk;
    const Index end = std::min(n, begin + chunk);
    if (begin >= end) break;
    pool.emplace_back([begin, end, &f] {
      for (Index i = begin; i < end; ++i) f(i);
    });
  }
  for (auto& th : pool) th.join();
}

// ------------------------------------------------------- covariance.cpp
// covariance.cpp:21-34 thread_local scratch.
struct SweepScratch {
  std::vector<double> v, a1, a2, a3, b, inv_dc;
  void resize(Index n, bool values_only) {
    v.resize(n);
    if (values_only) return;
    a1.resize(n);
    a2.resize(n);
    a3.resize(n);
    b.resize(n);
    inv_dc.resize(n);
  }
};
thread_local SweepScratch scratch;

// covariance.cpp:38-44 gather_with_ghosts: end values replicated into ghosts.
template <typename Line>
void gather_with_ghosts(std::vector<double>& dst, const Line& src, Index lo, Index len,
                        Index gl, Index gr) {
  for (Index k = 0; k < len; ++k) dst[gl + k] = src(lo + k);
  for (Index k = 0; k < gl; ++k) dst[k] = src(lo);
  for (Index k = 0; k < gr; ++k) dst[gl + len + k] = src(lo + len - 1);
}

// covariance.hpp:72-78 DirCoefficients, shared by every level (see the
// "shared tables" note in rgfo_op_create). Uniform fields are per level.
struct DirTables {
  std::vector<double> alpha1, alpha2, alpha3, beta, inv_dc;
};
struct LevelDir {
  bool uniform = false;
  double u_alpha1 = 0, u_alpha2 = 0, u_alpha3 = 0, u_beta = 0, u_inv_dc = 1;
};

}  // namespace

struct rgfo_op {
  Index nx = 0, ny = 0, nlev = 0;
  std::vector<uint8_t> mask;  // nlev*ny*nx
  int order = 3;               // 1 or 3
  int k_iterations = 1;
  bool unit_dc = true;
  int threads = 0;
  int calibration = 0;
  bool has_variance = false;
  std::vector<double> variance;  // nlev*ny*nx
  std::vector<Index> ghost;      // per level
  DirTables cx, cy;
  std::vector<LevelDir> ux, uy;  // per level

  bool sea(Index lev, Index i, Index j) const { return mask[(lev * ny + j) * nx + i] != 0; }

  // covariance.cpp:228-352 sweep_line, for level `lev`; in/out are one plane.
  void sweep_line(const double* in, double* out, int dir, bool transpose, Index line,
                  Index lev) const {
    const bool third = order == 3;
    const bool udc = third && unit_dc;
    const Index min_len = third ? 4 : 2;
    const Index n = dir == 0 ? nx : ny;
    const DirTables& c = dir == 0 ? cx : cy;
    const LevelDir& u = dir == 0 ? ux[lev] : uy[lev];
    const Index G = ghost[lev];
    // element k of this line -> plane offset
    const auto off = [&](Index k) { return dir == 0 ? line * nx + k : k * nx + line; };
    const auto mask_at = [&](Index k) {
      return dir == 0 ? sea(lev, k, line) : sea(lev, line, k);
    };
    const auto coeff_line = [&](const std::vector<double>& f) {
      return [&f, &off](Index k) { return f[off(k)]; };
    };

    Index i = 0;
    while (i < n) {
      if (!mask_at(i)) {
        ++i;
        continue;
      }
      Index j = i;
      while (j + 1 < n && mask_at(j + 1)) ++j;
      const Index len = j - i + 1;
      const Index gl = i > 0 ? G : 0;
      const Index gr = j < n - 1 ? G : 0;
      const Index ext = len + gl + gr;
      if (ext < min_len) {
        for (Index k = 0; k < len; ++k) out[off(i + k)] = in[off(i + k)];
        i = j + 1;
        continue;
      }
      scratch.resize(ext, u.uniform);
      std::fill(scratch.v.begin(), scratch.v.begin() + ext, 0.0);
      for (Index k = 0; k < len; ++k) scratch.v[gl + k] = in[off(i + k)];
      double* v = scratch.v.data();
      if (u.uniform) {
        if (!transpose) {
          if (third) {
            rf3_forward_u(v, u.u_alpha1, u.u_alpha2, u.u_alpha3, u.u_beta, ext);
            rf3_backward_u(v, u.u_alpha1, u.u_alpha2, u.u_alpha3, u.u_beta, ext);
            if (udc)
              for (Index k = 0; k < ext; ++k) v[k] *= u.u_inv_dc;
          } else {
            for (int it = 0; it < k_iterations; ++it) {
              rf1_forward_u(v, u.u_alpha1, u.u_beta, ext);
              rf1_backward_u(v, u.u_alpha1, u.u_beta, ext);
            }
          }
        } else {
          if (third) {
            if (udc)
              for (Index k = 0; k < ext; ++k) v[k] *= u.u_inv_dc;
            rf3_backward_transpose_u(v, u.u_alpha1, u.u_alpha2, u.u_alpha3, u.u_beta, ext);
            rf3_forward_transpose_u(v, u.u_alpha1, u.u_alpha2, u.u_alpha3, u.u_beta, ext);
          } else {
            for (int it = 0; it < k_iterations; ++it) {
              rf1_backward_transpose_u(v, u.u_alpha1, u.u_beta, ext);
              rf1_forward_transpose_u(v, u.u_alpha1, u.u_beta, ext);
            }
          }
        }
      } else {
        gather_with_ghosts(scratch.a1, coeff_line(c.alpha1), i, len, gl, gr);
        gather_with_ghosts(scratch.b, coeff_line(c.beta), i, len, gl, gr);
        if (third) {
          gather_with_ghosts(scratch.a2, coeff_line(c.alpha2), i, len, gl, gr);
          gather_with_ghosts(scratch.a3, coeff_line(c.alpha3), i, len, gl, gr);
          if (udc) gather_with_ghosts(scratch.inv_dc, coeff_line(c.inv_dc), i, len, gl, gr);
        }
        const double* a1 = scratch.a1.data();
        const double* a2 = scratch.a2.data();
        const double* a3 = scratch.a3.data();
        const double* b = scratch.b.data();
        if (!transpose) {
          if (third) {
            rf3_forward(v, a1, a2, a3, b, ext);
            rf3_backward(v, a1, a2, a3, b, ext);
            if (udc)
              for (Index k = 0; k < ext; ++k) v[k] *= scratch.inv_dc[k];
          } else {
            for (int it = 0; it < k_iterations; ++it) {
              rf1_forward(v, a1, b, ext);
              rf1_backward(v, a1, b, ext);
            }
          }
        } else {
          if (third) {
            if (udc)
              for (Index k = 0; k < ext; ++k) v[k] *= scratch.inv_dc[k];
            rf3_backward_transpose(v, a1, a2, a3, b, ext);
            rf3_forward_transpose(v, a1, a2, a3, b, ext);
          } else {
            for (int it = 0; it < k_iterations; ++it) {
              rf1_backward_transpose(v, a1, b, ext);
              rf1_forward_transpose(v, a1, b, ext);
            }
          }
        }
      }
      for (Index k = 0; k < len; ++k) out[off(i + k)] = scratch.v[gl + k];
      i = j + 1;
    }
  }

  // covariance.cpp:354-360: out starts zero (land stays exactly 0).
  void sweep(const double* in, double* out, int dir, bool transpose, Index lev) const {
    std::fill(out, out + nx * ny, 0.0);
    const Index lines = dir == 0 ? ny : nx;
    parallel_for(lines, threads,
                 [&](Index line) { sweep_line(in, out, dir, transpose, line, lev); });
  }
};

namespace {

int fail(const std::exception& e, int code) {
  g_last_error = e.what();
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}

}  // namespace

extern "C" {

const char* rgfo_last_error(void) { return g_last_error.c_str(); }

int rgfo_rf3_coefficients(double sigma, double out[8]) {
  return guarded([&] {
    const Poly t = rf3_coefficients(sigma);
    const double v[8] = {t.a0, t.a1, t.a2, t.a3, t.alpha1, t.alpha2, t.alpha3, t.beta};
    std::memcpy(out, v, sizeof(v));
  });
}

int rgfo_rf3_filter_scalars(double sigma, int calibration, double out[5]) {
  return guarded([&] {
    const Scalars3 f = rf3_filter_scalars(sigma, calibration);
    const double v[5] = {f.alpha1, f.alpha2, f.alpha3, f.beta, f.q};
    std::memcpy(out, v, sizeof(v));
  });
}

double rgfo_rf3_cascade_variance(double q) { return rf3_cascade_variance(q); }

double rgfo_rf3_length_scale_argument(double sigma, int calibration) {
  return rf3_length_scale_argument(sigma, calibration);
}

int rgfo_rf1_coefficients(double sigma, int k, double out[2]) {
  return guarded([&] {
    const Scalars1 c = rf1_coefficients(sigma, k);
    out[0] = c.alpha;
    out[1] = c.beta;
  });
}

// rf3.hpp:30-37
double rgfo_rational_gauss(double t) {
  const double t2 = t * t;
  return 1.0 / (2.490895 + 1.466003 * t2 + -0.024393 * t2 * t2 + 0.178257 * t2 * t2 * t2);
}

int rgfo_rf3_apply_1d_coeffs(const double* in, const double* a1, const double* a2,
                             const double* a3, const double* b, int64_t m, int transpose,
                             double* out) {
  return guarded([&] {
    // rf3.hpp:292-316
    if (m < 4) throw std::invalid_argument("rf3 filter: segment length must be >= 4");
    std::copy(in, in + m, out);
    if (!transpose) {
      rf3_forward(out, a1, a2, a3, b, m);
      rf3_backward(out, a1, a2, a3, b, m);
    } else {
      rf3_backward_transpose(out, a1, a2, a3, b, m);
      rf3_forward_transpose(out, a1, a2, a3, b, m);
    }
  });
}

int rgfo_rf3_apply_1d(const double* in, const double* sigma, int64_t m, int calibration,
                      int transpose, double* out) {
  return guarded([&] {
    // rf3.hpp:191-210 rf3_filter_coefficients
    std::vector<double> a1(m), a2(m), a3(m), b(m);
    for (Index i = 0; i < m; ++i) {
      const Scalars3 f = rf3_filter_scalars(sigma[i], calibration);
      a1[i] = f.alpha1;
      a2[i] = f.alpha2;
      a3[i] = f.alpha3;
      b[i] = f.beta;
    }
    if (m < 4) throw std::invalid_argument("rf3 filter: segment length must be >= 4");
    std::copy(in, in + m, out);
    if (!transpose) {
      rf3_forward(out, a1.data(), a2.data(), a3.data(), b.data(), m);
      rf3_backward(out, a1.data(), a2.data(), a3.data(), b.data(), m);
    } else {
      rf3_backward_transpose(out, a1.data(), a2.data(), a3.data(), b.data(), m);
      rf3_forward_transpose(out, a1.data(), a2.data(), a3.data(), b.data(), m);
    }
  });
}

int rgfo_rf1_apply_1d(const double* in, const double* sigma, int64_t m, int k,
                      int transpose, double* out) {
  return guarded([&] {
    // rf1.hpp:96-110, 113-137
    std::vector<double> a(m), b(m);
    for (Index i = 0; i < m; ++i) {
      const Scalars1 c = rf1_coefficients(sigma[i], k);
      a[i] = c.alpha;
      b[i] = c.beta;
    }
    if (m < 2) throw std::invalid_argument("rf1 filter: segment length must be >= 2");
    std::copy(in, in + m, out);
    for (int it = 0; it < k; ++it) {
      if (!transpose) {
        rf1_forward(out, a.data(), b.data(), m);
        rf1_backward(out, a.data(), b.data(), m);
      } else {
        rf1_backward_transpose(out, a.data(), b.data(), m);
        rf1_forward_transpose(out, a.data(), b.data(), m);
      }
    }
  });
}

int rgfo_op_create(int64_t nx, int64_t ny, int64_t nlev, const double* dx, const double* dy,
                   const uint8_t* mask, int64_t grid_ghost_width, const double* rx,
                   const double* ry, int order, int k_iterations, int unit_dc,
                   int64_t ghost_width, const double* variance, int threads, int calibration,
                   rgfo_op** out) {
  *out = nullptr;
  return guarded([&] {
    // grid.cpp:27-39 Grid2D::validate
    if (nx < 4 || ny < 4) throw std::invalid_argument("Grid2D: nx and ny must both be >= 4");
    if (nlev < 1) throw std::invalid_argument("Grid2D: nlev must be >= 1");
    const Index nh = nx * ny;
    for (Index p = 0; p < nh; ++p)
      if (!(dx[p] > 0) || !(dy[p] > 0))
        throw std::invalid_argument("Grid2D: grid spacing must be strictly positive");
    if (grid_ghost_width < 0) throw std::invalid_argument("Grid2D: ghost_width must be >= 0");
    // grid.cpp:41-55 ScaleField::validate, per level
    std::vector<uint8_t> any_sea(nh, 0);
    for (Index l = 0; l < nlev; ++l)
      for (Index j = 0; j < ny; ++j)
        for (Index i = 0; i < nx; ++i) {
          const Index p = j * nx + i;
          if (!mask[l * nh + p]) continue;
          any_sea[p] = 1;
          const double sx = rx[p] / dx[p];
          const double sy = ry[p] / dy[p];
          if (!(rx[p] > 0) || !(ry[p] > 0) || !std::isfinite(sx) || !std::isfinite(sy))
            throw std::invalid_argument(
                "ScaleField: non-positive or non-finite radius at sea point (" +
                std::to_string(i) + "," + std::to_string(j) + ")");
        }
    // covariance.cpp:159-168
    if (order != 1 && order != 3) throw std::invalid_argument("covariance: order must be 1 or 3");
    if (order == 1 && k_iterations < 1)
      throw std::invalid_argument("covariance: k_iterations must be >= 1");
    if (order == 3 && k_iterations != 1)
      throw std::invalid_argument(
          "covariance: the third-order filter is single-iteration by construction");

    auto op = std::make_unique<rgfo_op>();
    op->nx = nx;
    op->ny = ny;
    op->nlev = nlev;
    op->mask.assign(mask, mask + nlev * nh);
    op->order = order;
    op->k_iterations = k_iterations;
    op->unit_dc = unit_dc != 0;
    op->threads = threads;
    op->calibration = calibration;
    if (variance) {
      op->has_variance = true;
      op->variance.assign(variance, variance + nlev * nh);
    }

    // Shared tables: sigma = rx/dx wherever any level is sea, 1 elsewhere
    // (grid.cpp:57-63 select). At a level's land points the reference's
    // table holds the sigma=1 coefficients instead; sweeps never read land
    // coefficients (covariance.cpp:303-310 gathers sea points only), so
    // sharing one table across levels is arithmetic-identical.
    const auto build = [&](const double* r, const double* d, DirTables& c,
                           std::vector<LevelDir>& lu) {
      c.alpha1.resize(nh);
      c.beta.resize(nh);
      std::vector<double> sig(nh);
      for (Index p = 0; p < nh; ++p) sig[p] = any_sea[p] ? r[p] / d[p] : 1.0;
      if (order == 1) {
        for (Index p = 0; p < nh; ++p) {
          const Scalars1 ab = rf1_coefficients(sig[p], k_iterations);
          c.alpha1[p] = ab.alpha;
          c.beta[p] = ab.beta;
        }
      } else {
        c.alpha2.resize(nh);
        c.alpha3.resize(nh);
        for (Index p = 0; p < nh; ++p) {
          const Scalars3 f = rf3_filter_scalars(sig[p], calibration);
          c.alpha1[p] = f.alpha1;
          c.alpha2[p] = f.alpha2;
          c.alpha3[p] = f.alpha3;
          c.beta[p] = f.beta;
        }
        if (unit_dc) {
          // covariance.cpp:205: 1.0 / (sqrt(2 pi) * sigma), elementwise
          c.inv_dc.resize(nh);
          const double s2pi = std::sqrt(2.0 * std::numbers::pi);
          for (Index p = 0; p < nh; ++p) c.inv_dc[p] = 1.0 / (s2pi * sig[p]);
        }
      }
      // covariance.cpp:207-216 uniform fast path, per level (land sigma = 1)
      lu.resize(nlev);
      for (Index l = 0; l < nlev; ++l) {
        double mn = INFINITY, mx = -INFINITY;
        for (Index p = 0; p < nh; ++p) {
          const double s = op->mask[l * nh + p] ? r[p] / d[p] : 1.0;
          mn = std::min(mn, s);
          mx = std::max(mx, s);
        }
        LevelDir& u = lu[l];
        u.uniform = mn == mx;
        if (u.uniform) {
          if (order == 1) {
            const Scalars1 ab = rf1_coefficients(mn, k_iterations);
            u.u_alpha1 = ab.alpha;
            u.u_beta = ab.beta;
          } else {
            const Scalars3 f = rf3_filter_scalars(mn, calibration);
            u.u_alpha1 = f.alpha1;
            u.u_alpha2 = f.alpha2;
            u.u_alpha3 = f.alpha3;
            u.u_beta = f.beta;
            if (unit_dc) u.u_inv_dc = 1.0 / (std::sqrt(2.0 * std::numbers::pi) * mn);
          }
        }
      }
    };

    // covariance.cpp:173-180 ghost width, per level (max_sigma grid.cpp:65-67)
    if (ghost_width >= 0) {
      op->ghost.assign(nlev, ghost_width);
    } else if (grid_ghost_width > 0) {
      op->ghost.assign(nlev, grid_ghost_width);
    } else {
      op->ghost.resize(nlev);
      for (Index l = 0; l < nlev; ++l) {
        double mx = -INFINITY;
        for (Index p = 0; p < nh; ++p) {
          const bool s = op->mask[l * nh + p] != 0;
          mx = std::max(mx, s ? rx[p] / dx[p] : 1.0);
          mx = std::max(mx, s ? ry[p] / dy[p] : 1.0);
        }
        op->ghost[l] = static_cast<Index>(std::ceil(9.0 * mx));
      }
    }
    build(rx, dx, op->cx, op->ux);
    build(ry, dy, op->cy, op->uy);
    *out = op.release();
  });
}

void rgfo_op_destroy(rgfo_op* op) { delete op; }

int rgfo_op_apply(const rgfo_op* op, int kind, const double* in, double* out, int64_t nvar,
                  int64_t lev0, int64_t nlev_sub) {
  return guarded([&] {
    const Index nh = op->nx * op->ny;
    const Index nl = nlev_sub > 0 ? nlev_sub : op->nlev;
    if (lev0 < 0 || lev0 + nl > op->nlev) throw std::invalid_argument("apply: level range");
    std::vector<double> t1(nh), t2(nh);
    for (Index v = 0; v < nvar; ++v)
      for (Index ll = 0; ll < nl; ++ll) {
        const Index lev = lev0 + ll;
        const double* src = in + (v * nl + ll) * nh;
        double* dst = out + (v * nl + ll) * nh;
        const double* var = op->has_variance ? op->variance.data() + lev * nh : nullptr;
        // covariance.cpp:362-398
        switch (kind) {
          case 0: op->sweep(src, dst, 0, false, lev); break;
          case 1: op->sweep(src, dst, 1, false, lev); break;
          case 2: op->sweep(src, dst, 0, true, lev); break;
          case 3: op->sweep(src, dst, 1, true, lev); break;
          case 7:  // diagnostics.cpp:182 apply_gy(apply_gx(f))
            op->sweep(src, t1.data(), 0, false, lev);
            op->sweep(t1.data(), dst, 1, false, lev);
            break;
          case 4:  // apply_v
            op->sweep(src, t1.data(), 0, false, lev);
            op->sweep(t1.data(), dst, 1, false, lev);
            if (var)
              for (Index p = 0; p < nh; ++p) dst[p] *= var[p];
            break;
          case 5: {  // apply_v_transpose
            const double* s = src;
            if (var) {
              for (Index p = 0; p < nh; ++p) t2[p] = src[p] * var[p];
              s = t2.data();
            }
            op->sweep(s, t1.data(), 1, true, lev);
            op->sweep(t1.data(), dst, 0, true, lev);
            break;
          }
          case 6: {  // apply_b = apply_v(apply_v_transpose(f))
            const double* s = src;
            if (var) {
              for (Index p = 0; p < nh; ++p) t2[p] = src[p] * var[p];
              s = t2.data();
            }
            op->sweep(s, t1.data(), 1, true, lev);
            op->sweep(t1.data(), t2.data(), 0, true, lev);
            op->sweep(t2.data(), t1.data(), 0, false, lev);
            op->sweep(t1.data(), dst, 1, false, lev);
            if (var)
              for (Index p = 0; p < nh; ++p) dst[p] *= var[p];
            break;
          }
          default: throw std::invalid_argument("apply: unknown kind");
        }
      }
  });
}

int64_t rgfo_op_ghost_width(const rgfo_op* op, int64_t level) { return op->ghost[level]; }

// covariance.cpp:222-226, per 2-D level operator
uint64_t rgfo_op_coefficient_bytes(const rgfo_op* op) {
  const uint64_t per_point = op->order == 1 ? 2 : 4;
  return 2 * per_point * sizeof(double) * static_cast<uint64_t>(op->nx * op->ny);
}

int rgfo_op_uniform(const rgfo_op* op, int64_t level, int dir) {
  return dir == 0 ? op->ux[level].uniform : op->uy[level].uniform;
}

int rgfo_resolve_thread_count(int requested) { return resolve_thread_count(requested); }

}  // extern "C"

// ------------------------------------------------------------------ obs + CG
// Restatement of obs.cpp (bilinear H, scatter H^T, misfit) and solver.cpp
// (cost, control-variable CG) for a 2-D operator (level 0, one variable).
namespace {

struct Stencil {
  Index i0, j0;
  double w00, w10, w01, w11;
};

}  // namespace

struct rgfo_obs {
  Index n = 0;
  std::vector<Stencil> st;
  std::vector<double> values, r_var;
};

namespace {

// obs.cpp:18-44 bilinear_stencil
Stencil bilinear_stencil(const rgfo_op* op, double x, double y, Index row) {
  const auto fail = [row](const std::string& why) {
    throw std::invalid_argument("observation " + std::to_string(row) + ": " + why);
  };
  if (!std::isfinite(x) || !std::isfinite(y) || x < 0 || y < 0 || x > double(op->nx - 1) ||
      y > double(op->ny - 1))
    fail("position (" + std::to_string(x) + "," + std::to_string(y) + ") is outside the grid");
  Stencil st;
  st.i0 = std::min<Index>(static_cast<Index>(std::floor(x)), op->nx - 2);
  st.j0 = std::min<Index>(static_cast<Index>(std::floor(y)), op->ny - 2);
  const double fx = x - double(st.i0);
  const double fy = y - double(st.j0);
  st.w00 = (1 - fx) * (1 - fy);
  st.w10 = fx * (1 - fy);
  st.w01 = (1 - fx) * fy;
  st.w11 = fx * fy;
  const bool any_sea = op->sea(0, st.i0, st.j0) || op->sea(0, st.i0 + 1, st.j0) ||
                       op->sea(0, st.i0, st.j0 + 1) || op->sea(0, st.i0 + 1, st.j0 + 1);
  if (!any_sea) fail("all four stencil corners are land");
  return st;
}

// obs.cpp:59-71
void obs_h(const rgfo_op* op, const rgfo_obs* o, const double* f, double* out) {
  const Index nx = op->nx;
  for (Index n = 0; n < o->n; ++n) {
    const Stencil& st = o->st[n];
    const Index c = st.j0 * nx + st.i0;
    out[n] = st.w00 * f[c] + st.w10 * f[c + 1] + st.w01 * f[c + nx] + st.w11 * f[c + nx + 1];
  }
}

// obs.cpp:73-87
void obs_ht(const rgfo_op* op, const rgfo_obs* o, const double* v, double* out) {
  const Index nx = op->nx;
  std::fill(out, out + op->nx * op->ny, 0.0);
  for (Index n = 0; n < o->n; ++n) {
    const Stencil& st = o->st[n];
    const Index c = st.j0 * nx + st.i0;
    out[c] += st.w00 * v[n];
    out[c + 1] += st.w10 * v[n];
    out[c + nx] += st.w01 * v[n];
    out[c + nx + 1] += st.w11 * v[n];
  }
}

double odot(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

void validate_obs(const rgfo_obs* o) {  // obs.cpp:48-57 (positions checked at creation)
  for (Index n = 0; n < o->n; ++n)
    if (!(o->r_var[n] > 0))
      throw std::invalid_argument("observation " + std::to_string(n) +
                                  ": error variance must be positive");
}

struct CgCtx {
  const rgfo_op* op;
  const rgfo_obs* o;
  Index nh;
  std::vector<double> apply(int kind, const std::vector<double>& x) const {
    std::vector<double> y(nh);
    if (rgfo_op_apply(op, kind, x.data(), y.data(), 1, 0, 0) != 0)
      throw std::runtime_error(rgfo_last_error());
    return y;
  }
  std::vector<double> h(const std::vector<double>& f) const {
    std::vector<double> y(o->n);
    obs_h(op, o, f.data(), y.data());
    return y;
  }
  // solver.cpp:26-31: V^T H^T (v ./ r_var)
  std::vector<double> adjoint_rhs(const std::vector<double>& v) const {
    std::vector<double> s(o->n), t(nh);
    for (Index n = 0; n < o->n; ++n) s[n] = v[n] / o->r_var[n];
    obs_ht(op, o, s.data(), t.data());
    return apply(5, t);
  }
  // solver.cpp:18-22
  std::vector<double> misfit(const double* background) const {
    if (!background) return o->values;
    std::vector<double> bg(background, background + nh);
    std::vector<double> hb = h(bg), d(o->n);
    for (Index n = 0; n < o->n; ++n) d[n] = o->values[n] - hb[n];
    return d;
  }
};

void require_2d(const rgfo_op* op) {
  if (op->nlev != 1) throw std::invalid_argument("solve: the operator must have one level");
}

}  // namespace

extern "C" {

int rgfo_obs_create(const rgfo_op* op, int64_t n, const double* x, const double* y,
                    const double* values, const double* r_var, rgfo_obs** out) {
  return guarded([&] {
    require_2d(op);
    auto o = std::make_unique<rgfo_obs>();
    o->n = n;
    for (Index k = 0; k < n; ++k) o->st.push_back(bilinear_stencil(op, x[k], y[k], k));
    o->values.assign(values, values + n);
    o->r_var.assign(r_var, r_var + n);
    *out = o.release();
  });
}

void rgfo_obs_destroy(rgfo_obs* o) { delete o; }

// transpose 0: out[n] = H field; 1: out field = H^T in
int rgfo_obs_apply(const rgfo_op* op, const rgfo_obs* o, int transpose, const double* in,
                   double* out) {
  return guarded([&] {
    if (transpose)
      obs_ht(op, o, in, out);
    else
      obs_h(op, o, in, out);
  });
}

// solver.cpp:35-50; j3 = {j_total, j_background, j_obs}
int rgfo_cost(const rgfo_op* op, const rgfo_obs* o, const double* chi, const double* background,
              double* j3, double* gradient) {
  return guarded([&] {
    require_2d(op);
    validate_obs(o);
    const CgCtx cx{op, o, op->nx * op->ny};
    const std::vector<double> d = cx.misfit(background);
    const std::vector<double> c(chi, chi + cx.nh);
    const std::vector<double> hv = cx.h(cx.apply(4, c));
    std::vector<double> res(o->n);
    for (Index n = 0; n < o->n; ++n) res[n] = d[n] - hv[n];
    const double jb = 0.5 * odot(c, c);
    double jo = 0.0;
    for (Index n = 0; n < o->n; ++n) jo += res[n] * res[n] / o->r_var[n];
    jo *= 0.5;
    j3[0] = jb + jo;
    j3[1] = jb;
    j3[2] = jo;
    const std::vector<double> g = cx.adjoint_rhs(res);
    for (Index p = 0; p < cx.nh; ++p) gradient[p] = c[p] - g[p];
  });
}

// solver.cpp:52-114. gnorms: max_iter + 1 slots; info = {iterations, converged,
// number of gradient norms}; out3 = {final_relative_residual, j_background, j_obs}
int rgfo_solve(const rgfo_op* op, const rgfo_obs* o, double tol, int max_iter,
               const double* background, double* increment, double* misfit, double* gnorms,
               int64_t* info, double* out3) {
  return guarded([&] {
    if (!(tol > 0)) throw std::invalid_argument("solve: tol must be positive");
    if (max_iter < 0) throw std::invalid_argument("solve: max_iter must be >= 0");
    require_2d(op);
    validate_obs(o);
    const CgCtx cx{op, o, op->nx * op->ny};
    std::fill(increment, increment + cx.nh, 0.0);
    const std::vector<double> d = cx.misfit(background);
    std::copy(d.begin(), d.end(), misfit);
    info[0] = 0;
    info[1] = 0;
    info[2] = 0;
    out3[0] = out3[1] = out3[2] = 0.0;
    if (o->n == 0) {
      info[1] = 1;
      return;
    }
    const std::vector<double> b = cx.adjoint_rhs(d);
    const double bnorm = std::sqrt(odot(b, b));
    if (bnorm == 0) {
      info[1] = 1;
      return;
    }
    std::vector<double> chi(cx.nh, 0.0), r = b, p = r;
    double rs = odot(r, r);
    std::vector<double> gn{std::sqrt(rs)};
    bool conv = false;
    int iters = 0;
    for (int it = 0; it < max_iter; ++it) {
      std::vector<double> ap = cx.adjoint_rhs(cx.h(cx.apply(4, p)));  // solver.cpp:81-85
      for (Index q = 0; q < cx.nh; ++q) ap[q] = p[q] + ap[q];
      const double denom = odot(p, ap);
      if (denom <= 0) break;
      const double alpha = rs / denom;
      for (Index q = 0; q < cx.nh; ++q) chi[q] += alpha * p[q];
      for (Index q = 0; q < cx.nh; ++q) r[q] -= alpha * ap[q];
      const double rs_next = odot(r, r);
      iters = it + 1;
      gn.push_back(std::sqrt(rs_next));
      if (std::sqrt(rs_next) <= tol * bnorm) {
        conv = true;
        rs = rs_next;
        break;
      }
      const double beta = rs_next / rs;
      for (Index q = 0; q < cx.nh; ++q) p[q] = r[q] + beta * p[q];
      rs = rs_next;
    }
    (void)conv;
    const double rel = gn.back() / bnorm;
    const std::vector<double> inc = cx.apply(4, chi);
    std::copy(inc.begin(), inc.end(), increment);
    const std::vector<double> hi = cx.h(inc);
    double jo = 0.0;
    for (Index n = 0; n < o->n; ++n) {
      const double res = d[n] - hi[n];
      jo += res * res / o->r_var[n];
    }
    info[0] = iters;
    info[1] = rel <= tol ? 1 : 0;
    info[2] = static_cast<int64_t>(gn.size());
    std::copy(gn.begin(), gn.end(), gnorms);
    out3[0] = rel;
    out3[1] = 0.5 * odot(chi, chi);
    out3[2] = 0.5 * jo;
  });
}

}  // extern "C"
