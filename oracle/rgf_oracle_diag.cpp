// Oracle restatement of the reference's batched-diagnostics targets (test
// infrastructure only): diagnostics.cpp:18-60 (apply_filter_1d,
// gaussian_kernel, convolve_same), :69-96 impulse_response and :102-135
// remark1_bound_check, on the oracle's own 1-D filters (rgf_oracle.cpp).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numbers>
#include <stdexcept>
#include <string>
#include <vector>

#include "rgf_oracle.h"

namespace {
thread_local std::string g_diag_error;

std::vector<double> apply_filter_1d(const std::vector<double>& s0, double sigma, int order, int k,
                                    int calibration, bool unit_dc) {  // diagnostics.cpp:18-37
  const int64_t m = static_cast<int64_t>(s0.size());
  const std::vector<double> sig(static_cast<size_t>(m), sigma);
  std::vector<double> out(static_cast<size_t>(m));
  int st;
  if (order == 1) {
    st = rgfo_rf1_apply_1d(s0.data(), sig.data(), m, k, 0, out.data());
  } else {
    if (k != 1)
      throw std::invalid_argument("the third-order filter is single-iteration by construction");
    st = rgfo_rf3_apply_1d(s0.data(), sig.data(), m, calibration, 0, out.data());
    if (st == 0 && unit_dc)
      for (double& v : out) v /= std::sqrt(2.0 * std::numbers::pi) * sigma;
  }
  if (st != 0) throw std::invalid_argument(rgfo_last_error());
  return out;
}

double norm(const std::vector<double>& v) {
  double s = 0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}
}  // namespace

extern "C" {

const char* rgfo_diag_last_error(void) { return g_diag_error.c_str(); }

int rgfo_impulse_response(double sigma, int order, int k, int64_t length, int calibration,
                          double* h, double* sum_h, double* err_l2, double* err_max) {
  try {
    if (length < 4) throw std::invalid_argument("impulse_response: length must be >= 4");
    if (!(sigma > 0)) throw std::invalid_argument("impulse_response: sigma must be positive");
    const int64_t c = length / 2;
    std::vector<double> dirac(static_cast<size_t>(length), 0.0);
    dirac[static_cast<size_t>(c)] = 1.0;
    const std::vector<double> r = apply_filter_1d(dirac, sigma, order, k, calibration, false);
    std::vector<double> g(static_cast<size_t>(length));
    for (int64_t i = 0; i < length; ++i)
      g[static_cast<size_t>(i)] = std::exp(-double((i - c) * (i - c)) / (2 * sigma * sigma));
    double sh = 0, sg = 0;
    for (int64_t i = 0; i < length; ++i) {
      sh += r[static_cast<size_t>(i)];
      sg += g[static_cast<size_t>(i)];
    }
    std::vector<double> diff(static_cast<size_t>(length));
    double mx = 0;
    for (int64_t i = 0; i < length; ++i) {
      diff[static_cast<size_t>(i)] = r[static_cast<size_t>(i)] / sh - g[static_cast<size_t>(i)] / sg;
      mx = std::max(mx, std::abs(diff[static_cast<size_t>(i)]));
      h[i] = r[static_cast<size_t>(i)];
    }
    *sum_h = sh;
    *err_l2 = norm(diff);
    *err_max = mx;
    return 0;
  } catch (const std::exception& e) {
    g_diag_error = e.what();
    return 1;
  }
}

int rgfo_remark1(const double* s0p, int64_t m, double sigma, int order, int k, int calibration,
                 double* out4) {
  try {
    if (m < 4) throw std::invalid_argument("remark1_bound_check: input too short");
    const std::vector<double> s0(s0p, s0p + m);
    const int64_t c = m / 2;
    const int64_t radius =
        std::min<int64_t>(static_cast<int64_t>(std::ceil(8 * sigma)), std::min(c, m - 1 - c));
    std::vector<double> kernel(static_cast<size_t>(2 * radius + 1));  // :40-46
    double ks = 0;
    for (int64_t o = -radius; o <= radius; ++o) {
      kernel[static_cast<size_t>(o + radius)] = std::exp(-double(o * o) / (2 * sigma * sigma));
      ks += kernel[static_cast<size_t>(o + radius)];
    }
    for (double& v : kernel) v /= ks;
    std::vector<double> dirac(static_cast<size_t>(m), 0.0);
    dirac[static_cast<size_t>(c)] = 1.0;
    const std::vector<double> h = apply_filter_1d(dirac, sigma, order, k, calibration, true);
    std::vector<double> gd(static_cast<size_t>(m), 0.0);
    for (int64_t i = c - radius; i <= c + radius; ++i)
      gd[static_cast<size_t>(i)] = kernel[static_cast<size_t>(i - c + radius)] - h[static_cast<size_t>(i)];
    for (int64_t i = 0; i < m; ++i)
      if (i < c - radius || i > c + radius) gd[static_cast<size_t>(i)] = -h[static_cast<size_t>(i)];
    const double err = norm(gd);
    std::vector<double> st(static_cast<size_t>(m), 0.0);  // convolve_same :49-60
    for (int64_t i = 0; i < m; ++i) {
      const int64_t lo = std::max<int64_t>(0, i - radius), hi = std::min<int64_t>(m - 1, i + radius);
      double acc = 0;
      for (int64_t j = lo; j <= hi; ++j)
        acc += kernel[static_cast<size_t>(i - j + radius)] * s0[static_cast<size_t>(j)];
      st[static_cast<size_t>(i)] = acc;
    }
    const std::vector<double> sf = apply_filter_1d(s0, sigma, order, k, calibration, true);
    for (int64_t i = 0; i < m; ++i) st[static_cast<size_t>(i)] -= sf[static_cast<size_t>(i)];
    out4[0] = norm(st);
    out4[1] = err * norm(s0);
    out4[2] = err;
    out4[3] = out4[0] <= out4[1] * (1.0 + 1e-9) ? 1.0 : 0.0;
    return 0;
  } catch (const std::exception& e) {
    g_diag_error = e.what();
    return 1;
  }
}

}  // extern "C"
