// C++ facade over the rgf_b200 C ABI with the reference's names and
// semantics (/root/reference/proj/include/rgf/{types,grid,covariance,rf1,rf3}.hpp).
//
// A caller of rgf::HorizontalCovarianceOp switches by including this header
// instead of rgf/covariance.hpp and linking librgf_b200.so: the types,
// constructors, the seven const apply_* methods, effective_ghost_width(),
// coefficient_bytes() and the std::invalid_argument messages are the same.
// The only representational difference is that Eigen is optional: Field is a
// minimal column-major (x fastest) array with the Eigen accessors the
// reference's callers use (operator()(i,j), rows(), cols(), data(), size(),
// Constant/Zero/Ones). Where Eigen is available, define
// RGF_B200_USE_EIGEN before including to get the reference's exact
// Eigen::Array typedefs instead; the facade only touches .data().
//
// Header-only; every arithmetic operation on field values happens in the
// sm_100a kernels behind rgf_op_apply.
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../rgf_b200.h"

#ifdef RGF_B200_USE_EIGEN
#include <Eigen/Dense>
#endif

namespace rgf {

using Scalar = double;            // types.hpp:14
using Index = std::ptrdiff_t;     // Eigen::Index

#ifdef RGF_B200_USE_EIGEN
using Field = Eigen::Array<Scalar, Eigen::Dynamic, Eigen::Dynamic>;
using MaskField = Eigen::Array<bool, Eigen::Dynamic, Eigen::Dynamic>;
#else
// Column-major nx x ny array (types.hpp:25-28: x along rows, contiguous).
template <typename T>
class Array2 {
 public:
  Array2() = default;
  Array2(Index rows, Index cols) : r_(rows), c_(cols), v_(static_cast<size_t>(rows * cols)) {}
  static Array2 Constant(Index rows, Index cols, T v) {
    Array2 a(rows, cols);
    for (auto& x : a.v_) x = v;
    return a;
  }
  static Array2 Zero(Index rows, Index cols) { return Constant(rows, cols, T(0)); }
  static Array2 Ones(Index rows, Index cols) { return Constant(rows, cols, T(1)); }
  T& operator()(Index i, Index j) { return v_[static_cast<size_t>(j * r_ + i)]; }
  const T& operator()(Index i, Index j) const { return v_[static_cast<size_t>(j * r_ + i)]; }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  T* data() { return v_.data(); }
  const T* data() const { return v_.data(); }
  void resize(Index rows, Index cols) {
    r_ = rows;
    c_ = cols;
    v_.assign(static_cast<size_t>(rows * cols), T(0));
  }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<T> v_;
};
using Field = Array2<Scalar>;
using MaskField = Array2<std::uint8_t>;
#endif

enum class FilterOrder { first = RGF_ORDER_FIRST, third = RGF_ORDER_THIRD };  // types.hpp:30
enum class Rf3Calibration {                                                    // types.hpp:39
  yvv95 = RGF_CAL_YVV95,
  variance_match = RGF_CAL_VARIANCE_MATCH,
  none = RGF_CAL_NONE
};

namespace detail {
inline void check(int status) {
  if (status == RGF_OK) return;
  const std::string msg = rgf_last_error();
  if (status == RGF_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
}  // namespace detail

// grid.hpp:20-37
struct Grid2D {
  Index nx = 0;
  Index ny = 0;
  Field dx;
  Field dy;
  MaskField mask;  // true / nonzero = sea
  Index ghost_width = 0;

  static Grid2D uniform(Index nx, Index ny, Scalar dx, Scalar dy, Index ghost_width = 0) {
    Grid2D g;
    g.nx = nx;
    g.ny = ny;
    g.dx = Field::Constant(nx, ny, dx);
    g.dy = Field::Constant(nx, ny, dy);
    g.mask = MaskField::Constant(nx, ny, 1);
    g.ghost_width = ghost_width;
    if (nx < 4 || ny < 4) throw std::invalid_argument("Grid2D: nx and ny must both be >= 4");
    return g;
  }
  Index size() const { return nx * ny; }
  bool same_shape(const Grid2D& o) const { return nx == o.nx && ny == o.ny; }
};

// grid.hpp:40-52
struct ScaleField {
  Field rx;
  Field ry;
};

inline ScaleField uniform_scale(const Grid2D& grid, Scalar r) {  // grid.cpp:69-76
  if (!(r > 0)) throw std::invalid_argument("uniform_scale: radius must be positive");
  return {Field::Constant(grid.nx, grid.ny, r), Field::Constant(grid.nx, grid.ny, r)};
}

// grid.hpp:59-71
struct StateField {
  const Grid2D* grid = nullptr;
  Field values;
  static StateField zeros(const Grid2D& g) { return {&g, Field::Zero(g.nx, g.ny)}; }
  static StateField from(const Grid2D& g, Field v) {
    if (v.rows() != g.nx || v.cols() != g.ny)
      throw std::invalid_argument("StateField: values shape does not match grid");
    return {&g, std::move(v)};
  }
};

inline void require_on_grid(const StateField& f, const Grid2D& g, const std::string& what) {
  if (f.grid == nullptr || !f.grid->same_shape(g) || f.values.rows() != g.nx ||
      f.values.cols() != g.ny)
    throw std::invalid_argument(what + ": field is not on the expected grid");
}

// covariance.hpp:17-25
struct CovarianceOptions {
  FilterOrder order = FilterOrder::third;
  int k_iterations = 1;
  bool unit_dc = true;
  std::optional<Index> ghost_width;
  std::optional<Field> variance;
  int threads = 0;  // accepted; the GPU path ignores it
  Rf3Calibration calibration = Rf3Calibration::yvv95;
  int device = 0;   // CUDA device ordinal (extension)
};

// covariance.hpp:35-79
class HorizontalCovarianceOp {
 public:
  HorizontalCovarianceOp(const Grid2D& grid, const ScaleField& scales,
                         CovarianceOptions options = {})
      : grid_(&grid), options_(std::move(options)) {
    if (grid.dx.rows() != grid.nx || grid.dx.cols() != grid.ny || grid.dy.rows() != grid.nx ||
        grid.dy.cols() != grid.ny)
      throw std::invalid_argument("Grid2D: spacing field shape mismatch");
    if (grid.mask.rows() != grid.nx || grid.mask.cols() != grid.ny)
      throw std::invalid_argument("Grid2D: mask shape mismatch");
    if (scales.rx.rows() != grid.nx || scales.rx.cols() != grid.ny ||
        scales.ry.rows() != grid.nx || scales.ry.cols() != grid.ny)
      throw std::invalid_argument("ScaleField: shape does not match grid");
    if (options_.variance &&
        (options_.variance->rows() != grid.nx || options_.variance->cols() != grid.ny))
      throw std::invalid_argument("covariance: variance field shape mismatch");
    if (options_.ghost_width && *options_.ghost_width < 0)
      throw std::invalid_argument("covariance: ghost_width < 0");
    mask_.resize(static_cast<size_t>(grid.nx * grid.ny));
    for (Index j = 0; j < grid.ny; ++j)
      for (Index i = 0; i < grid.nx; ++i)
        mask_[static_cast<size_t>(j * grid.nx + i)] = grid.mask(i, j) ? 1 : 0;
    rgf_grid_desc g{grid.nx, grid.ny, 1, grid.dx.data(), grid.dy.data(), mask_.data(),
                    grid.ghost_width};
    rgf_options o;
    rgf_options_default(&o);
    o.order = static_cast<int32_t>(options_.order);
    o.k_iterations = options_.k_iterations;
    o.unit_dc = options_.unit_dc ? 1 : 0;
    o.calibration = static_cast<int32_t>(options_.calibration);
    o.ghost_width = options_.ghost_width ? static_cast<int64_t>(*options_.ghost_width) : -1;
    o.variance = options_.variance ? options_.variance->data() : nullptr;
    o.threads = options_.threads;
    o.device = options_.device;
    detail::check(rgf_op_create(&g, scales.rx.data(), scales.ry.data(), &o, &op_));
  }
  HorizontalCovarianceOp(const HorizontalCovarianceOp&) = delete;
  HorizontalCovarianceOp& operator=(const HorizontalCovarianceOp&) = delete;
  ~HorizontalCovarianceOp() {
    if (op_) rgf_op_destroy(op_);
  }

  StateField apply_gx(const StateField& f) const { return run(RGF_GX, f, "apply_gx"); }
  StateField apply_gy(const StateField& f) const { return run(RGF_GY, f, "apply_gy"); }
  StateField apply_gx_transpose(const StateField& f) const {
    return run(RGF_GXT, f, "apply_gx_transpose");
  }
  StateField apply_gy_transpose(const StateField& f) const {
    return run(RGF_GYT, f, "apply_gy_transpose");
  }
  StateField apply_v(const StateField& f) const { return run(RGF_V, f, "apply_v"); }
  StateField apply_v_transpose(const StateField& f) const {
    return run(RGF_VT, f, "apply_v_transpose");
  }
  StateField apply_b(const StateField& f) const { return run(RGF_B, f, "apply_v_transpose"); }

  const Grid2D& grid() const { return *grid_; }
  const CovarianceOptions& options() const { return options_; }
  rgf_op* handle() const { return op_; }  // the C-ABI operator (solver.hpp)
  Index effective_ghost_width() const {
    int64_t g = 0;
    detail::check(rgf_op_ghost_width(op_, 0, &g));
    return static_cast<Index>(g);
  }
  std::size_t coefficient_bytes() const {
    uint64_t b = 0;
    detail::check(rgf_op_coefficient_bytes(op_, &b));
    return static_cast<std::size_t>(b);
  }

 private:
  StateField run(int kind, const StateField& f, const char* what) const {
    require_on_grid(f, *grid_, what);
    StateField out{grid_, Field(grid_->nx, grid_->ny)};
    detail::check(rgf_op_apply(op_, kind, RGF_F64, f.values.data(), out.values.data(), 1,
                               RGF_HOST, nullptr));
    return out;
  }

  const Grid2D* grid_;
  CovarianceOptions options_;
  std::vector<std::uint8_t> mask_;
  rgf_op* op_ = nullptr;
};

// rf3.hpp:71-76, 159-164 and rf1.hpp:403-407 scalar coefficient sets,
// evaluated by the device builders.
template <typename S>
struct Rf3PolynomialSet {
  S a0, a1, a2, a3;
  S alpha1, alpha2, alpha3;
  S beta;
};
inline Rf3PolynomialSet<double> rf3_coefficients(double sigma) {
  double o[8];
  detail::check(rgf_rf3_coefficients(sigma, o));
  return {o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7]};
}
template <typename S>
struct Rf3Scalars {
  S alpha1, alpha2, alpha3;
  S beta;
  S q;
};
inline Rf3Scalars<double> rf3_filter_scalars(double sigma,
                                             Rf3Calibration c = Rf3Calibration::yvv95) {
  double o[5];
  detail::check(rgf_rf3_filter_scalars(sigma, static_cast<int>(c), o));
  return {o[0], o[1], o[2], o[3], o[4]};
}
template <typename S>
struct Rf1Scalars {
  S alpha;
  S beta;
};
inline Rf1Scalars<double> rf1_coefficients(double sigma, int k) {
  double o[2];
  detail::check(rgf_rf1_coefficients(sigma, k, o));
  return {o[0], o[1]};
}

}  // namespace rgf
