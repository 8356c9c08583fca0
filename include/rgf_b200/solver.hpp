// C++ facade over the C ABI for the observation operator and the 3D-VAR
// analysis: the reference's obs.hpp:15-46 and solver.hpp:19-55 with the same
// names, arguments and exceptions, running on the device (SURVEY.md §8f rows
// 1-2). Header-only; include after (or instead of) rgf_b200/covariance.hpp.
#pragma once

#include <cmath>
#include <string>
#include <vector>

#include "rgf_b200/covariance.hpp"

namespace rgf {

#ifdef RGF_B200_USE_EIGEN
}  // namespace rgf
#include "rgf/obs.hpp"  // the reference's ObsSet, obs_operator(_transpose), misfit (obs.cpp)
namespace rgf {
#else
// column vector (Eigen::VectorXd stand-in)
class Vector {
 public:
  Vector() = default;
  explicit Vector(Index n) : v_(static_cast<size_t>(n), 0.0) {}
  Index size() const { return static_cast<Index>(v_.size()); }
  void resize(Index n) { v_.assign(static_cast<size_t>(n), 0.0); }
  Scalar& operator[](Index i) { return v_[static_cast<size_t>(i)]; }
  const Scalar& operator[](Index i) const { return v_[static_cast<size_t>(i)]; }
  Scalar* data() { return v_.data(); }
  const Scalar* data() const { return v_.data(); }

 private:
  std::vector<Scalar> v_;
};
// n x 2 column-major positions (Eigen::ArrayX2d stand-in): (n, 0) = x, (n, 1) = y
using Positions = Array2<Scalar>;

// obs.hpp:15-25
struct ObsSet {
  Positions positions;
  Vector values;
  Vector r_var;
  Index size() const { return values.size(); }
};
#endif

// solver.hpp:19-40
struct SolveOptions {
  Scalar tol = 1e-6;
  int max_iter = 30;
};
struct Analysis {
  StateField increment;
  Vector misfit;
  int cg_iterations = 0;
  std::vector<Scalar> gradient_norms;
  bool converged = false;
  Scalar final_relative_residual = 0;
  Scalar j_background = 0;
  Scalar j_obs = 0;
};
struct CostReport {
  Scalar j_total;
  Scalar j_background;
  Scalar j_obs;
  Field gradient;
};

namespace detail {
// device ObsSet bound to a grid (stencils validated on creation, obs.cpp:18-57)
class DeviceObs {
 public:
  DeviceObs(const Grid2D& g, const ObsSet& obs, int device = 0) {
    if (obs.positions.rows() != obs.values.size() || obs.positions.rows() != obs.r_var.size())
      throw std::invalid_argument("ObsSet: inconsistent column lengths");
    const Index n = obs.size();
    std::vector<double> x(static_cast<size_t>(n)), y(static_cast<size_t>(n));
    for (Index k = 0; k < n; ++k) {
      x[static_cast<size_t>(k)] = obs.positions(k, 0);
      y[static_cast<size_t>(k)] = obs.positions(k, 1);
    }
    mask_.resize(static_cast<size_t>(g.nx * g.ny));
    for (Index j = 0; j < g.ny; ++j)
      for (Index i = 0; i < g.nx; ++i)
        mask_[static_cast<size_t>(j * g.nx + i)] = g.mask(i, j) ? 1 : 0;
    const rgf_grid_desc d{g.nx, g.ny, 1, g.dx.data(), g.dy.data(), mask_.data(), g.ghost_width};
    check(rgf_obs_create(&d, device, n, x.data(), y.data(), obs.values.data(), obs.r_var.data(),
                         &h_));
  }
  DeviceObs(const DeviceObs&) = delete;
  DeviceObs& operator=(const DeviceObs&) = delete;
  ~DeviceObs() {
    if (h_) rgf_obs_destroy(h_);
  }
  rgf_obs* get() const { return h_; }

 private:
  std::vector<std::uint8_t> mask_;
  rgf_obs* h_ = nullptr;
};

// Field (nx x ny column-major) <-> the C ABI's ny*nx x-fastest layout: the
// same memory order (element (i, j) at j*nx + i), so data() passes through.
inline const double* flat(const Field& f) { return f.data(); }
}  // namespace detail

#ifndef RGF_B200_USE_EIGEN  // the drop-in keeps the reference's obs.cpp for these
// obs.hpp:41-43: H, bilinear interpolation at each observation
inline Vector obs_operator(const StateField& field, const ObsSet& obs) {
  if (!field.grid) throw std::invalid_argument("obs_operator: field has no grid");
  detail::DeviceObs d(*field.grid, obs);
  Vector out(obs.size());
  if (obs.size() > 0)
    detail::check(rgf_obs_apply(d.get(), 0, detail::flat(field.values), out.data(), RGF_HOST,
                                nullptr));
  return out;
}

// obs.hpp:45-46: H^T, scatter with the same weights
inline StateField obs_operator_transpose(const Vector& vec, const ObsSet& obs,
                                         const Grid2D& grid) {
  if (vec.size() != obs.size())
    throw std::invalid_argument("obs_operator_transpose: vector length mismatch");
  detail::DeviceObs d(grid, obs);
  StateField out = StateField::zeros(grid);
  double dummy = 0.0;
  detail::check(rgf_obs_apply(d.get(), 1, vec.size() ? vec.data() : &dummy, out.values.data(),
                              RGF_HOST, nullptr));
  return out;
}

// obs.hpp:48-49
inline Vector misfit(const Vector& background_at_obs, const ObsSet& obs) {
  if (background_at_obs.size() != obs.size())
    throw std::invalid_argument("misfit: vector length mismatch");
  Vector d(obs.size());
  for (Index k = 0; k < obs.size(); ++k) d[k] = obs.values[k] - background_at_obs[k];
  return d;
}

#endif

// solver.hpp:45-47
inline CostReport cost(const StateField& chi, const ObsSet& obs, const HorizontalCovarianceOp& op,
                       const StateField* background = nullptr) {
  require_on_grid(chi, op.grid(), "cost");
  if (background) require_on_grid(*background, op.grid(), "solve");
  detail::DeviceObs d(op.grid(), obs, op.options().device);
  double j3[3];
  CostReport r{0, 0, 0, Field(op.grid().nx, op.grid().ny)};
  detail::check(rgf_cost(op.handle(), d.get(), chi.values.data(),
                         background ? background->values.data() : nullptr, j3,
                         r.gradient.data()));
  r.j_total = j3[0];
  r.j_background = j3[1];
  r.j_obs = j3[2];
  return r;
}

// solver.hpp:49-55
inline Analysis solve(const ObsSet& obs, const HorizontalCovarianceOp& op,
                      SolveOptions options = {}, const StateField* background = nullptr) {
  if (!(options.tol > 0)) throw std::invalid_argument("solve: tol must be positive");
  if (options.max_iter < 0) throw std::invalid_argument("solve: max_iter must be >= 0");
  if (background) require_on_grid(*background, op.grid(), "solve");
  detail::DeviceObs d(op.grid(), obs, op.options().device);
  Analysis an;
  an.increment = StateField::zeros(op.grid());
  an.misfit = Vector(obs.size());
  std::vector<double> gn(static_cast<size_t>(options.max_iter) + 1);
  rgf_analysis a{};
  detail::check(rgf_solve(op.handle(), d.get(), options.tol, options.max_iter,
                          background ? background->values.data() : nullptr,
                          an.increment.values.data(), obs.size() ? an.misfit.data() : nullptr,
                          gn.data(), &a));
  an.cg_iterations = a.cg_iterations;
  an.converged = a.converged != 0;
  an.gradient_norms.assign(gn.begin(), gn.begin() + a.n_gradient_norms);
  an.final_relative_residual = a.final_relative_residual;
  an.j_background = a.j_background;
  an.j_obs = a.j_obs;
  return an;
}

}  // namespace rgf
