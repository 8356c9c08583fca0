// C++ facade over the rgf_b200 C ABI with the reference's names and
// semantics (/root/reference/proj/include/rgf/{types,grid,covariance,rf1,rf3}.hpp).
//
// Two configurations:
//
//  * RGF_B200_USE_EIGEN (the drop-in): the reference's own
//    rgf/types.hpp and rgf/grid.hpp are included, so Scalar, Index, Field,
//    MaskField, FilterOrder, Rf3Calibration, Grid2D, ScaleField, StateField,
//    uniform_scale and require_on_grid stay the reference's (grid.cpp is still
//    compiled from the reference). This header defines only what
//    rgf/covariance.hpp declares: CovarianceOptions and
//    HorizontalCovarianceOp, whose applies run on the device. The reference
//    include graph (diagnostics.hpp:13-14 includes covariance, then grid)
//    therefore compiles unchanged: include/rgf_b200/dropin/rgf/covariance.hpp
//    shadows the reference's header on the include path
//    (tests/test_boundary.py::test_dropin_compiles_with_reference_headers).
//    The 1-D entry points with coefficient tables are in namespace rgf::b200
//    (the reference's header-only rf1.hpp / rf3.hpp keep their names).
//
//  * default (no Eigen in this container): Eigen-free stand-ins with the
//    reference's names, members, validation and messages; Field is a
//    column-major (x fastest) nx x ny array with the accessors the
//    reference's callers use. The 1-D entry points are in namespace rgf
//    with the reference's names.
//
// Header-only; every arithmetic operation on field values happens in the
// sm_100a kernels behind the C ABI (include/rgf_b200.h).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../rgf_b200.h"

#ifdef RGF_B200_USE_EIGEN
#include "rgf/grid.hpp"   // the reference's (rgfvar include path)
#include "rgf/types.hpp"
#endif

namespace rgf {

namespace detail {
inline void check(int status) {
  if (status == RGF_OK) return;
  const std::string msg = rgf_last_error();
  if (status == RGF_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
}  // namespace detail

#ifndef RGF_B200_USE_EIGEN
using Scalar = double;         // types.hpp:14
using Index = std::ptrdiff_t;  // Eigen::Index

// Column-major rows x cols array (types.hpp:25-28: x along rows, contiguous).
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
  T& operator[](Index i) { return v_[static_cast<size_t>(i)]; }
  const T& operator[](Index i) const { return v_[static_cast<size_t>(i)]; }
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
  void resize(Index n) { resize(n, 1); }
  bool all() const {
    for (const T& x : v_)
      if (!x) return false;
    return true;
  }
  T maxCoeff() const { return *std::max_element(v_.begin(), v_.end()); }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<T> v_;
};
using Field = Array2<Scalar>;
using MaskField = Array2<std::uint8_t>;
template <typename S>
using ArrayX = Array2<S>;   // n x 1 (types.hpp:19-20)
template <typename S>
using VectorX = Array2<S>;  // n x 1 (types.hpp:17-18)

enum class FilterOrder { first, third };                   // types.hpp:30
enum class Rf3Calibration { yvv95, variance_match, none };  // types.hpp:39

struct Grid2D;
// grid.hpp:40-52 (grid.cpp:40-67)
struct ScaleField {
  Field rx;
  Field ry;
  void validate(const Grid2D& grid) const;
  Field sigma_x(const Grid2D& grid) const;
  Field sigma_y(const Grid2D& grid) const;
  Scalar max_sigma(const Grid2D& grid) const;
};

// grid.hpp:20-37 (grid.cpp:7-38)
struct Grid2D {
  Index nx = 0;
  Index ny = 0;
  Field dx;
  Field dy;
  MaskField mask;  // nonzero = sea
  Index ghost_width = 0;

  static Grid2D uniform(Index nx, Index ny, Scalar dx, Scalar dy, Index ghost_width = 0) {
    Grid2D g;
    g.nx = nx;
    g.ny = ny;
    g.dx = Field::Constant(nx, ny, dx);
    g.dy = Field::Constant(nx, ny, dy);
    g.mask = MaskField::Constant(nx, ny, 1);
    g.ghost_width = ghost_width;
    g.validate();
    return g;
  }
  void validate() const {
    if (nx < 4 || ny < 4) throw std::invalid_argument("Grid2D: nx and ny must both be >= 4");
    if (dx.rows() != nx || dx.cols() != ny || dy.rows() != nx || dy.cols() != ny)
      throw std::invalid_argument("Grid2D: spacing field shape mismatch");
    if (mask.rows() != nx || mask.cols() != ny)
      throw std::invalid_argument("Grid2D: mask shape mismatch");
    for (Index p = 0; p < nx * ny; ++p)
      if (!(dx[p] > 0) || !(dy[p] > 0))
        throw std::invalid_argument("Grid2D: grid spacing must be strictly positive");
    if (ghost_width < 0) throw std::invalid_argument("Grid2D: ghost_width must be >= 0");
  }
  bool all_sea() const { return mask.all(); }
  Index size() const { return nx * ny; }
  bool same_shape(const Grid2D& o) const { return nx == o.nx && ny == o.ny; }
};

inline void ScaleField::validate(const Grid2D& grid) const {
  if (rx.rows() != grid.nx || rx.cols() != grid.ny || ry.rows() != grid.nx ||
      ry.cols() != grid.ny)
    throw std::invalid_argument("ScaleField: shape does not match grid");
  for (Index j = 0; j < grid.ny; ++j)
    for (Index i = 0; i < grid.nx; ++i) {
      if (!grid.mask(i, j)) continue;
      const Scalar sx = rx(i, j) / grid.dx(i, j);
      const Scalar sy = ry(i, j) / grid.dy(i, j);
      if (!(rx(i, j) > 0) || !(ry(i, j) > 0) || !std::isfinite(sx) || !std::isfinite(sy))
        throw std::invalid_argument("ScaleField: non-positive or non-finite radius at sea point (" +
                                    std::to_string(i) + "," + std::to_string(j) + ")");
    }
}
// grid.cpp:57-63: sigma = R / d at sea, 1 on land (the values the operator's
// coefficient kernels compute on the device; host copies for callers)
inline Field ScaleField::sigma_x(const Grid2D& grid) const {
  Field s(grid.nx, grid.ny);
  for (Index p = 0; p < grid.nx * grid.ny; ++p) s[p] = grid.mask[p] ? rx[p] / grid.dx[p] : 1.0;
  return s;
}
inline Field ScaleField::sigma_y(const Grid2D& grid) const {
  Field s(grid.nx, grid.ny);
  for (Index p = 0; p < grid.nx * grid.ny; ++p) s[p] = grid.mask[p] ? ry[p] / grid.dy[p] : 1.0;
  return s;
}
inline Scalar ScaleField::max_sigma(const Grid2D& grid) const {  // grid.cpp:65-67
  return std::max(sigma_x(grid).maxCoeff(), sigma_y(grid).maxCoeff());
}

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
#endif  // !RGF_B200_USE_EIGEN

// covariance.hpp:17-25
struct CovarianceOptions {
  FilterOrder order = FilterOrder::third;
  int k_iterations = 1;
  bool unit_dc = true;
  std::optional<Index> ghost_width;
  std::optional<Field> variance;
  int threads = 0;  // accepted; the GPU path ignores it
  Rf3Calibration calibration = Rf3Calibration::yvv95;
  int device = 0;   // CUDA device ordinal (extension; defaulted, so aggregate use is unchanged)
};

// covariance.hpp:35-79 (covariance.cpp:155-398 on the device)
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
    o.order = options_.order == FilterOrder::first ? RGF_ORDER_FIRST : RGF_ORDER_THIRD;
    o.k_iterations = options_.k_iterations;
    o.unit_dc = options_.unit_dc ? 1 : 0;
    o.calibration = options_.calibration == Rf3Calibration::yvv95            ? RGF_CAL_YVV95
                    : options_.calibration == Rf3Calibration::variance_match ? RGF_CAL_VARIANCE_MATCH
                                                                             : RGF_CAL_NONE;
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

// ------------------------------------------------------------------ 1-D
// Scalar builders and the 1-D entry points (rf3.hpp:71-334, rf1.hpp:64-155),
// device-backed. Drop-in: namespace rgf::b200 (the reference's rf1.hpp /
// rf3.hpp own the names in rgf); stand-in: namespace rgf.
#ifdef RGF_B200_USE_EIGEN
namespace b200 {
#endif

inline int cal_abi(Rf3Calibration c) {
  return c == Rf3Calibration::yvv95 ? RGF_CAL_YVV95
         : c == Rf3Calibration::variance_match ? RGF_CAL_VARIANCE_MATCH : RGF_CAL_NONE;
}

template <typename S>
struct Rf3PolynomialSet {  // rf3.hpp:71-76
  S a0, a1, a2, a3;
  S alpha1, alpha2, alpha3;
  S beta;
};
inline Rf3PolynomialSet<double> rf3_coefficients(double sigma) {  // rf3.hpp:78-95
  double o[8];
  detail::check(rgf_rf3_coefficients(sigma, o));
  return {o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7]};
}
template <typename S>
struct Rf3Scalars {  // rf3.hpp:159-164
  S alpha1, alpha2, alpha3;
  S beta;
  S q;
};
inline Rf3Scalars<double> rf3_filter_scalars(double sigma,  // rf3.hpp:166-181
                                             Rf3Calibration c = Rf3Calibration::yvv95) {
  double o[5];
  detail::check(rgf_rf3_filter_scalars(sigma, cal_abi(c), o));
  return {o[0], o[1], o[2], o[3], o[4]};
}
inline double rf3_cascade_variance(double q) {  // rf3.hpp:101-108
  double v = 0.0;
  detail::check(rgf_rf3_cascade_variance(q, &v));
  return v;
}
inline double rf3_length_scale_argument(double sigma, Rf3Calibration c) {  // rf3.hpp:143-154
  double v = 0.0;
  detail::check(rgf_rf3_length_scale_argument(sigma, cal_abi(c), &v));
  return v;
}
template <typename S>
struct Rf1Scalars {  // rf1.hpp:66-70
  S alpha;
  S beta;
};
inline Rf1Scalars<double> rf1_coefficients(double sigma, int k) {  // rf1.hpp:76-85
  double o[2];
  detail::check(rgf_rf1_coefficients(sigma, k, o));
  return {o[0], o[1]};
}

// Coefficient tables (rf3.hpp:183-189, rf1.hpp:87-92). Container: anything
// with resize(n), size() and data() over doubles (the stand-in arrays,
// Eigen::ArrayXd, std::vector<double>).
template <typename A>
struct Rf3TablesT {
  A alpha1, alpha2, alpha3, beta;
};
template <typename A>
struct Rf1TablesT {
  A alpha, beta;
  int k_iterations = 1;
};
#ifndef RGF_B200_USE_EIGEN
using Rf3Coefficients = Rf3TablesT<ArrayX<double>>;  // rf3.hpp:189
using Rf1Coefficients = Rf1TablesT<ArrayX<double>>;  // rf1.hpp:94
template <typename S>
using Rf3CoefficientsT = Rf3TablesT<ArrayX<S>>;
template <typename S>
using Rf1CoefficientsT = Rf1TablesT<ArrayX<S>>;
#endif

// rf3.hpp:191-210 rf3_filter_coefficients(sigma table, calibration)
template <typename Tab = Rf3TablesT<ArrayX<double>>, typename Sigma>
Tab rf3_filter_coefficients(const Sigma& sigma, Rf3Calibration c = Rf3Calibration::yvv95) {
  Tab t;
  const auto m = static_cast<Index>(sigma.size());
  t.alpha1.resize(m);
  t.alpha2.resize(m);
  t.alpha3.resize(m);
  t.beta.resize(m);
  detail::check(rgf_rf3_filter_coefficients(sigma.data(), m, cal_abi(c), t.alpha1.data(),
                                            t.alpha2.data(), t.alpha3.data(), t.beta.data()));
  return t;
}
// rf1.hpp:96-110 table overload
template <typename Tab = Rf1TablesT<ArrayX<double>>, typename Sigma,
          typename = std::enable_if_t<!std::is_arithmetic_v<Sigma>>>
Tab rf1_coefficients(const Sigma& sigma, int k) {
  Tab t;
  const auto m = static_cast<Index>(sigma.size());
  t.k_iterations = k;
  t.alpha.resize(m);
  t.beta.resize(m);
  detail::check(rgf_rf1_coefficients_table(sigma.data(), m, k, t.alpha.data(), t.beta.data()));
  return t;
}

// rf3.hpp:292-316: one forward+backward cascade (or its transpose), in place
template <typename Seg, typename Tab>
void rf3_filter_in_place(Seg& seg, const Tab& c) {
  const auto m = static_cast<Index>(seg.size());
  if (m < 4) throw std::invalid_argument("rf3 filter: segment length must be >= 4");
  if (static_cast<Index>(c.alpha1.size()) != m || static_cast<Index>(c.beta.size()) != m)
    throw std::invalid_argument("rf3 filter: coefficient length mismatch");
  detail::check(rgf_rf3_filter(seg.data(), c.alpha1.data(), c.alpha2.data(), c.alpha3.data(),
                               c.beta.data(), m, 1, 0, seg.data()));
}
template <typename Seg, typename Tab>
void rf3_filter_transpose_in_place(Seg& seg, const Tab& c) {
  const auto m = static_cast<Index>(seg.size());
  if (m < 4) throw std::invalid_argument("rf3 filter: segment length must be >= 4");
  if (static_cast<Index>(c.alpha1.size()) != m || static_cast<Index>(c.beta.size()) != m)
    throw std::invalid_argument("rf3 filter: coefficient length mismatch");
  detail::check(rgf_rf3_filter(seg.data(), c.alpha1.data(), c.alpha2.data(), c.alpha3.data(),
                               c.beta.data(), m, 1, 1, seg.data()));
}
// rf3.hpp:318-334 (out of place)
template <typename Seg, typename Tab>
Seg rf3_apply_1d(const Seg& segment, const Tab& c) {
  Seg out = segment;
  rf3_filter_in_place(out, c);
  return out;
}
template <typename Seg, typename Tab>
Seg rf3_apply_transpose_1d(const Seg& segment, const Tab& c) {
  Seg out = segment;
  rf3_filter_transpose_in_place(out, c);
  return out;
}
// rf1.hpp:113-137: K x {forward, backward} (or the transposes), in place
template <typename Seg, typename Tab>
void rf1_filter_in_place(Seg& seg, const Tab& c) {
  const auto m = static_cast<Index>(seg.size());
  if (m < 2) throw std::invalid_argument("rf1 filter: segment length must be >= 2");
  if (static_cast<Index>(c.alpha.size()) != m || static_cast<Index>(c.beta.size()) != m)
    throw std::invalid_argument("rf1 filter: coefficient length mismatch");
  detail::check(rgf_rf1_filter(seg.data(), c.alpha.data(), c.beta.data(), m, 1, c.k_iterations, 0,
                               seg.data()));
}
template <typename Seg, typename Tab>
void rf1_filter_transpose_in_place(Seg& seg, const Tab& c) {
  const auto m = static_cast<Index>(seg.size());
  if (m < 2) throw std::invalid_argument("rf1 filter: segment length must be >= 2");
  if (static_cast<Index>(c.alpha.size()) != m || static_cast<Index>(c.beta.size()) != m)
    throw std::invalid_argument("rf1 filter: coefficient length mismatch");
  detail::check(rgf_rf1_filter(seg.data(), c.alpha.data(), c.beta.data(), m, 1, c.k_iterations, 1,
                               seg.data()));
}
// rf1.hpp:139-155 (out of place)
template <typename Seg, typename Tab>
Seg rf1_apply_1d(const Seg& segment, const Tab& c) {
  Seg out = segment;
  rf1_filter_in_place(out, c);
  return out;
}
template <typename Seg, typename Tab>
Seg rf1_apply_transpose_1d(const Seg& segment, const Tab& c) {
  Seg out = segment;
  rf1_filter_transpose_in_place(out, c);
  return out;
}

#ifdef RGF_B200_USE_EIGEN
}  // namespace b200
#endif

}  // namespace rgf
