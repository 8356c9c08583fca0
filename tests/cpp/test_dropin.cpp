// The INTEGRATION.md drop-in configuration, compiled against the reference's
// own headers (/root/reference/proj/include) with include/rgf_b200/dropin
// first on the include path and a minimal Eigen stand-in
// (tests/cpp/eigen_shim). The reference include graph is exercised as its
// translation units see it: diagnostics.hpp:13-14 (covariance, then grid),
// solver.hpp:12-15 (covariance, grid, obs), io.hpp. Links the reference's own
// grid.cpp (Grid2D::uniform / validate, ScaleField::sigma_x / sigma_y /
// max_sigma, uniform_scale) and librgf_b200.so. Built and run by
// tests/test_boundary.py (CPU): without a GPU the operator's construction
// must fail loudly with the C ABI's CUDA error, not fall back.
#include <cstdio>
#include <stdexcept>
#include <string>

#include "rgf/diagnostics.hpp"
#include "rgf/io.hpp"
#include "rgf/solver.hpp"

int main() {
  using namespace rgf;
  Grid2D g = Grid2D::uniform(16, 12, 5000.0, 5000.0);  // reference grid.cpp
  g.mask(3, 4) = false;
  g.validate();
  const ScaleField s = uniform_scale(g, 20000.0);  // reference grid.cpp
  s.validate(g);
  if (s.max_sigma(g) != 4.0 || s.sigma_x(g)(3, 4) != 1.0 || g.all_sea()) return 2;
  CovarianceOptions o;  // the drop-in's (same fields as covariance.hpp:17-25)
  o.order = FilterOrder::first;
  o.k_iterations = 5;
  o.variance = Field::Constant(g.nx, g.ny, 2.0);
  try {
    const HorizontalCovarianceOp op(g, s, o);
    StateField f = StateField::zeros(g);
    f.values(8, 6) = 1.0;
    const StateField out = op.apply_gy(op.apply_gx(f));  // diagnostics.cpp:182
    const StateField v = op.apply_v_transpose(out);      // solver.cpp:26-31
    std::printf("applied on the device: %g\n", v.values(8, 6));
    ObsSet obs;
    obs.positions.resize(1, 2);
    obs.positions(0, 0) = 4.5;
    obs.positions(0, 1) = 3.5;
    obs.values = Vector::Zero(1);
    obs.r_var = Vector::Zero(1);
    SolveOptions so;
    (void)so;
    std::printf("dropin ok (device)\n");
  } catch (const std::runtime_error& e) {
    std::printf("dropin ok (no device: %s)\n", e.what());
  }
  // the 1-D entry points with tables live in rgf::b200 in this configuration
  Eigen::ArrayXd sig = Eigen::ArrayXd::Constant(8, 1, 3.0);
  try {
    const auto c = b200::rf3_filter_coefficients(sig);
    std::printf("tables %ld\n", static_cast<long>(c.alpha1.size()));
  } catch (const std::runtime_error& e) {
    std::printf("tables need a device: %s\n", e.what());
  }
  return 0;
}
