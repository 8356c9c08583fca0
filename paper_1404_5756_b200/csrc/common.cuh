// Shared device helpers: IEEE-exact arithmetic wrappers and the coefficient
// builders of the reference (rf3.hpp:78-181, rf1.hpp:76-85,
// covariance.cpp:205), evaluated on the device.
//
// Contraction is suppressed with the __d*_rn intrinsics wherever the
// reference's result is reproduced bit-for-bit (every coefficient except beta,
// whose pow() may differ from glibc by an ulp or two).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rgfb {

#define RGFB_HD __host__ __device__ __forceinline__

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// rf3.hpp:46-66 (printed constants; RGF_USE_APPENDIX_A_CONSTANTS selects the
// alternate printing exactly as the reference's CMake option does).
#ifdef RGF_USE_APPENDIX_A_CONSTANTS
constexpr double kC00 = 3.738128, kC01 = 5.788982, kC02 = 3.382472, kC11 = 5.788824,
                 kC12 = 6.764946, kC13 = 2.999999, kC22 = -3.382472, kC23 = -2.999999;
#else
constexpr double kC00 = 3.738128, kC01 = 5.788982, kC02 = 3.382473, kC11 = 5.788982,
                 kC12 = 6.764946, kC13 = 3.0, kC22 = -3.382473, kC23 = -3.0;
#endif
constexpr double kTwoPi = 6.283185307179586;  // 2 * std::numbers::pi, exact

struct Poly3 {
  double a0, a1, a2, a3, alpha1, alpha2, alpha3, beta;
};

// (2 pi sigma sigma)^(1/4), evaluated as ((2*pi)*sigma)*sigma then pow.
__device__ __forceinline__ double amp(double sigma) {
  return pow(dmul(dmul(kTwoPi, sigma), sigma), 0.25);
}

// rf3.hpp:78-95 rf3_coefficients (left-to-right, unfused).
__device__ inline Poly3 rf3_coefficients(double x) {
  const double x2 = dmul(x, x), x3 = dmul(x2, x);
  Poly3 t;
  t.a0 = dadd(dadd(dadd(kC00, dmul(kC01, x)), dmul(kC02, x2)), x3);
  t.a1 = dadd(dadd(dmul(kC11, x), dmul(kC12, x2)), dmul(kC13, x3));
  t.a2 = dadd(dmul(kC22, x2), dmul(kC23, x3));
  t.a3 = x3;
  t.alpha1 = ddiv(t.a1, t.a0);
  t.alpha2 = ddiv(t.a2, t.a0);
  t.alpha3 = ddiv(t.a3, t.a0);
  t.beta = dmul(amp(x), dsub(1.0, dadd(dadd(t.alpha1, t.alpha2), t.alpha3)));
  return t;
}

// rf3.hpp:101-108
__device__ inline double rf3_cascade_variance(double q) {
  const Poly3 t = rf3_coefficients(q);
  const double a = dsub(1.0, dadd(dadd(t.alpha1, t.alpha2), t.alpha3));
  const double s1 = dadd(dadd(t.alpha1, dmul(2.0, t.alpha2)), dmul(3.0, t.alpha3));
  const double s2 = dadd(dmul(2.0, t.alpha2), dmul(6.0, t.alpha3));
  return dmul(2.0, dadd(ddiv(dmul(s1, s1), dmul(a, a)), ddiv(dadd(s1, s2), a)));
}

// rf3.hpp:116-126 yvv95_argument
__device__ inline double yvv95_argument(double sigma) {
  double q;
  if (sigma >= 2.5) {
    q = dsub(dmul(0.98711, sigma), 0.96330);
  } else {
    double arg = dsub(1.0, dmul(0.26891, sigma));
    arg = arg < 0.0 ? 0.0 : arg;  // std::max(arg, 0)
    q = dsub(3.97156, dmul(4.14554, __dsqrt_rn(arg)));
  }
  return q < 0.01 ? 0.01 : q;  // std::max(q, 0.01)
}

// rf3.hpp:128-139 variance_matched_argument (200-step bisection)
__device__ inline double variance_matched_argument(double sigma) {
  const double target = dmul(sigma, sigma);
  double lo = 1e-12;
  double hi = sigma < 1.0 ? 1.0 : sigma;
  while (rf3_cascade_variance(hi) < target) hi = dmul(hi, 2.0);
  for (int it = 0; it < 200; ++it) {
    const double mid = dmul(0.5, dadd(lo, hi));
    if (rf3_cascade_variance(mid) < target)
      lo = mid;
    else
      hi = mid;
  }
  return dmul(0.5, dadd(lo, hi));
}

// rf3.hpp:143-154
__device__ inline double rf3_length_scale_argument(double sigma, int calibration) {
  switch (calibration) {
    case 0: return yvv95_argument(sigma);
    case 1: return variance_matched_argument(sigma);
    default: return sigma;
  }
}

struct Scal3 {
  double alpha1, alpha2, alpha3, beta, q;
};

// rf3.hpp:166-181 rf3_filter_scalars: ratios at q, amplitude at the target sigma.
__device__ inline Scal3 rf3_filter_scalars(double sigma, int calibration) {
  const double q = rf3_length_scale_argument(sigma, calibration);
  const Poly3 t = rf3_coefficients(q);
  Scal3 f;
  f.alpha1 = t.alpha1;
  f.alpha2 = t.alpha2;
  f.alpha3 = t.alpha3;
  f.beta = dmul(amp(sigma), dsub(1.0, dadd(dadd(t.alpha1, t.alpha2), t.alpha3)));
  f.q = q;
  return f;
}

// rf1.hpp:76-85: q = K/sigma^2, alpha = (1+q) - sqrt(q(q+2)), beta = 1 - alpha.
__device__ inline double rf1_alpha(double sigma, int k) {
  const double q = ddiv(double(k), dmul(sigma, sigma));
  const double root = __dsqrt_rn(dmul(q, dadd(q, 2.0)));
  return dsub(dadd(1.0, q), root);
}

// covariance.cpp:205: 1.0 / (sqrt(2 pi) * sigma)
__device__ inline double inv_dc(double sigma) {
  return ddiv(1.0, dmul(__dsqrt_rn(kTwoPi), sigma));
}

// Per-direction coefficient tables, shared by all levels (a level's land
// points are never read, covariance.cpp:303-310).
struct Coef3 {
  double a1, a2, a3, b;  // 32 B: one sector per point
};

// Closure table addressing: [class][dir][part][nh][10] doubles
// (part 0 = forward operator, 1 = adjoint).
__host__ __device__ __forceinline__ int64_t clos_off(int cls, int dir, int part, int64_t nh,
                                                     int64_t h) {
  return ((static_cast<int64_t>(cls) * 2 + dir) * 2 + part) * nh * 10 + h * 10;
}

}  // namespace rgfb
