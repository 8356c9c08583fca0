// Batched filter diagnostics (diagnostics.cpp:69-135):
// many impulse studies and Remark-1 accuracy checks at once, one thread per
// study (a study is one 1-D line with its own sigma, filter order and K).
// The filters are the reference's 1-D recursions with the uniform-sigma
// scalars (diagnostics.cpp:18-37 builds constant tables); the reductions run
// serially inside the study's thread in the reference's order, so results do
// not depend on the batch size. exp() is the device's (the reference uses
// glibc's): the checks compare within 1e-12, not bit for bit.
#pragma once
#include "sweep_generic.cuh"

namespace rgfb {

struct UniCoef {  // constant coefficients (one sigma per line)
  double a1_, a2_, a3_, b_;
  __device__ __forceinline__ double a1(int64_t) const { return a1_; }
  __device__ __forceinline__ double a2(int64_t) const { return a2_; }
  __device__ __forceinline__ double a3(int64_t) const { return a3_; }
  __device__ __forceinline__ double b(int64_t) const { return b_; }
};

// diagnostics.cpp:18-37 apply_filter_1d, in place on v[0..m)
__device__ inline void diag_filter(double* v, int64_t m, double sigma, int order, int k,
                                   int calibration, bool unit_dc) {
  if (order == 1) {
    const double a = rf1_alpha(sigma, k);
    const UniCoef c{a, 0.0, 0.0, dsub(1.0, a)};
    for (int it = 0; it < k; ++it) {
      g_rf1_forward(v, c, m);
      g_rf1_backward(v, c, m);
    }
  } else {
    const Scal3 f = rf3_filter_scalars(sigma, calibration);
    const UniCoef c{f.alpha1, f.alpha2, f.alpha3, f.beta};
    g_rf3_forward(v, c, m);
    g_rf3_backward(v, c, m);
    if (unit_dc) {  // out /= sqrt(2 pi) sigma (diagnostics.cpp:35)
      const double d = dmul(sqrt(dmul(2.0, 3.141592653589793)), sigma);
      for (int64_t i = 0; i < m; ++i) v[i] = ddiv(v[i], d);
    }
  }
}

// diagnostics.cpp:69-96 impulse_response: h (length per study), sum_h,
// err_h_l2, err_h_max. h doubles as the study's scratch.
__global__ void k_impulse(const double* sigma, int64_t n, int order, int k, int64_t length,
                          int calibration, double* h, double* sum_h, double* err_l2,
                          double* err_max) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    double* v = h + s * length;
    const int64_t c = length / 2;
    for (int64_t i = 0; i < length; ++i) v[i] = i == c ? 1.0 : 0.0;
    const double sg = sigma[s];
    diag_filter(v, length, sg, order, k, calibration, false);
    double sh = 0.0, sgs = 0.0;
    for (int64_t i = 0; i < length; ++i) sh = dadd(sh, v[i]);
    const double den = dmul(dmul(2.0, sg), sg);
    for (int64_t i = 0; i < length; ++i) {
      const double o = static_cast<double>(i - c);
      sgs = dadd(sgs, exp(ddiv(-dmul(o, o), den)));
    }
    double l2 = 0.0, mx = 0.0;
    for (int64_t i = 0; i < length; ++i) {
      const double o = static_cast<double>(i - c);
      const double d = dsub(ddiv(v[i], sh), ddiv(exp(ddiv(-dmul(o, o), den)), sgs));
      l2 = dadd(l2, dmul(d, d));
      mx = fmax(mx, fabs(d));
    }
    sum_h[s] = sh;
    err_l2[s] = sqrt(l2);
    err_max[s] = mx;
  }
}

// diagnostics.cpp:102-135 remark1_bound_check for study s: input s0 (m), its
// own sigma; scratch 3*m per study. out4 = {lhs, rhs, err_h_l2, holds}.
__global__ void k_remark1(const double* s0, const double* sigma, int64_t n, int64_t m, int order,
                          int k, int calibration, double* scratch, double* out4) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    const double* x = s0 + s * m;
    double* h = scratch + s * 3 * m;
    double* kern = h + m;
    double* f = h + 2 * m;
    const double sg = sigma[s];
    const int64_t c = m / 2;
    int64_t radius = static_cast<int64_t>(ceil(dmul(8.0, sg)));
    radius = radius < c ? radius : c;
    radius = radius < m - 1 - c ? radius : m - 1 - c;
    // gaussian_kernel (diagnostics.cpp:40-46): unit-sum sampled Gaussian
    double ks = 0.0;
    const double den = dmul(dmul(2.0, sg), sg);
    for (int64_t o = -radius; o <= radius; ++o) {
      kern[o + radius] = exp(ddiv(-static_cast<double>(o * o), den));
      ks = dadd(ks, kern[o + radius]);
    }
    for (int64_t o = 0; o <= 2 * radius; ++o) kern[o] = ddiv(kern[o], ks);
    for (int64_t i = 0; i < m; ++i) h[i] = i == c ? 1.0 : 0.0;
    diag_filter(h, m, sg, order, k, calibration, true);
    double e2 = 0.0;  // ||g_centered - h||
    for (int64_t i = 0; i < m; ++i) {
      const double g = (i >= c - radius && i <= c + radius) ? kern[i - c + radius] : 0.0;
      const double d = dsub(g, h[i]);
      e2 = dadd(e2, dmul(d, d));
    }
    for (int64_t i = 0; i < m; ++i) f[i] = x[i];
    diag_filter(f, m, sg, order, k, calibration, true);
    double l2 = 0.0, n2 = 0.0;
    for (int64_t i = 0; i < m; ++i) {  // convolve_same (diagnostics.cpp:49-60) on the fly
      const int64_t lo = i - radius > 0 ? i - radius : 0;
      const int64_t hi = i + radius < m - 1 ? i + radius : m - 1;
      double acc = 0.0;
      for (int64_t j = lo; j <= hi; ++j) acc = dadd(acc, dmul(kern[i - j + radius], x[j]));
      const double d = dsub(acc, f[i]);
      l2 = dadd(l2, dmul(d, d));
      n2 = dadd(n2, dmul(x[i], x[i]));
    }
    const double lhs = sqrt(l2), err = sqrt(e2), rhs = dmul(err, sqrt(n2));
    out4[4 * s + 0] = lhs;
    out4[4 * s + 1] = rhs;
    out4[4 * s + 2] = err;
    out4[4 * s + 3] = lhs <= dmul(rhs, dadd(1.0, 1e-9)) ? 1.0 : 0.0;
  }
}

}  // namespace rgfb
