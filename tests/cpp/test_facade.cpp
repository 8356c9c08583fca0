// Reference-style parity tests through the C++ facade (include/rgf_b200/
// covariance.hpp), mirroring proj/tests/test_covariance.cpp case by case.
// Built and run by tests/test_gpu_facade.py on the GPU box:
//   g++ -std=c++20 -O2 -I include tests/cpp/test_facade.cpp \
//       paper_1404_5756_b200/librgf_b200.so -o /tmp/test_facade
#include <array>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "rgf_b200/covariance.hpp"
#include "rgf_b200/solver.hpp"

using namespace rgf;

static int failures = 0, checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++checks;                                                              \
    if (!(cond)) {                                                         \
      ++failures;                                                          \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
    }                                                                      \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                           \
  do {                                                                     \
    ++checks;                                                              \
    bool thrown = false;                                                   \
    try { (void)(expr); } catch (const T&) { thrown = true; }              \
    if (!thrown) { ++failures; std::printf("FAIL %s:%d: no throw\n", __FILE__, __LINE__); } \
  } while (0)

static CovarianceOptions opts(FilterOrder order, int k, bool unit_dc,
                              std::optional<Index> ghost = std::nullopt) {
  CovarianceOptions o;
  o.order = order;
  o.k_iterations = k;
  o.unit_dc = unit_dc;
  o.ghost_width = ghost;
  o.threads = 1;
  return o;
}

static MaskField checkered(Index nx, Index ny, unsigned seed, double sea) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  MaskField m(nx, ny);
  for (Index j = 0; j < ny; ++j)
    for (Index i = 0; i < nx; ++i) m(i, j) = u(rng) < sea;
  return m;
}

static Field random_field(Index nx, Index ny, std::mt19937& rng) {
  std::normal_distribution<double> d;
  Field f(nx, ny);
  for (Index j = 0; j < ny; ++j)
    for (Index i = 0; i < nx; ++i) f(i, j) = d(rng);
  return f;
}

int main() {
  {  // test_covariance.cpp:65-79 land splits a row into independent segments
    Grid2D g = Grid2D::uniform(21, 4, 6000.0, 6000.0);
    for (Index j = 0; j < g.ny; ++j) g.mask(10, j) = 0;
    const ScaleField s = uniform_scale(g, 12000.0);
    for (const auto order : {FilterOrder::first, FilterOrder::third}) {
      const HorizontalCovarianceOp op(g, s, opts(order, order == FilterOrder::first ? 5 : 1, false));
      StateField f = StateField::zeros(g);
      f.values(4, 1) = 1.0;
      const StateField out = op.apply_gx(f);
      CHECK(out.values(10, 1) == 0.0);
      for (Index i = 11; i < g.nx; ++i) CHECK(out.values(i, 1) == 0.0);
      CHECK(out.values(4, 1) > 0.0);
    }
  }
  {  // :81-96 short segments pass through
    Grid2D g = Grid2D::uniform(5, 4, 6000.0, 6000.0);
    for (Index j = 0; j < g.ny; ++j) g.mask(2, j) = 0;
    const HorizontalCovarianceOp op(g, uniform_scale(g, 12000.0), opts(FilterOrder::third, 1, false, 0));
    StateField f = StateField::zeros(g);
    f.values(0, 1) = 2.0;
    f.values(1, 1) = -1.0;
    f.values(3, 1) = 0.5;
    const StateField out = op.apply_gx(f);
    CHECK(out.values(0, 1) == 2.0);
    CHECK(out.values(1, 1) == -1.0);
    CHECK(out.values(2, 1) == 0.0);
    CHECK(out.values(3, 1) == 0.5);
  }
  {  // :120-132 land barrier blocks B
    Grid2D g = Grid2D::uniform(40, 24, 6000.0, 6000.0);
    for (Index j = 0; j < g.ny; ++j) g.mask(20, j) = 0;
    const HorizontalCovarianceOp op(g, uniform_scale(g, 12000.0), opts(FilterOrder::third, 1, true));
    StateField f = StateField::zeros(g);
    f.values(8, 12) = 1.0;
    const Field b = op.apply_b(f).values;
    for (Index j = 0; j < g.ny; ++j)
      for (Index i = 20; i < g.nx; ++i) CHECK(b(i, j) == 0.0);
    CHECK(b(8, 12) > 0.0);
  }
  {  // :134-154 separability against the device 1-D coefficients
    const Grid2D g = Grid2D::uniform(64, 64, 6000.0, 6000.0);
    const HorizontalCovarianceOp op(g, uniform_scale(g, 12000.0), opts(FilterOrder::third, 1, false));
    StateField f = StateField::zeros(g);
    f.values(32, 32) = 1.0;
    const Field out = op.apply_gy(op.apply_gx(f)).values;
    std::vector<double> d(64, 0.0), h(64), sig(64, 2.0);
    d[32] = 1.0;
    detail::check(rgf_rf3_apply_1d(d.data(), sig.data(), 64, 1, RGF_CAL_YVV95, 0, h.data()));
    for (Index j = 0; j < 64; ++j)
      for (Index i = 0; i < 64; ++i)
        CHECK(std::abs(out(i, j) - h[i] * h[j]) < 1e-10 * (1.0 + std::abs(h[i] * h[j])));
  }
  {  // :178-197 masked dot product (mt19937 masks as the reference builds them)
    Grid2D g = Grid2D::uniform(20, 20, 6000.0, 6000.0);
    g.mask = checkered(20, 20, 99, 0.8);
    const ScaleField s = uniform_scale(g, 12000.0);
    std::mt19937 rng(31);
    for (const auto order : {FilterOrder::first, FilterOrder::third}) {
      const HorizontalCovarianceOp op(g, s, opts(order, order == FilterOrder::first ? 5 : 1, true));
      for (int trial = 0; trial < 20; ++trial) {
        const StateField u{&g, random_field(20, 20, rng)};
        const StateField v{&g, random_field(20, 20, rng)};
        const Field vu = op.apply_v(u).values, vtv = op.apply_v_transpose(v).values;
        double lhs = 0, rhs = 0, nu = 0, nv = 0;
        for (Index k = 0; k < u.values.size(); ++k) {
          lhs += v.values.data()[k] * vu.data()[k];
          rhs += vtv.data()[k] * u.values.data()[k];
          nu += u.values.data()[k] * u.values.data()[k];
          nv += v.values.data()[k] * v.values.data()[k];
        }
        CHECK(std::abs(lhs - rhs) <= 1e-10 * std::sqrt(nu * nv));
      }
    }
  }
  {  // :308-327 land exactly zero with junk input
    Grid2D g = Grid2D::uniform(24, 24, 6000.0, 6000.0);
    g.mask = checkered(24, 24, 121, 0.7);
    const ScaleField s = uniform_scale(g, 12000.0);
    std::mt19937 rng(61);
    for (const auto order : {FilterOrder::first, FilterOrder::third}) {
      const HorizontalCovarianceOp op(g, s, opts(order, order == FilterOrder::first ? 3 : 1, true));
      const StateField u{&g, random_field(24, 24, rng)};
      const StateField results[] = {op.apply_gx(u), op.apply_gy(u), op.apply_v(u),
                                    op.apply_v_transpose(u), op.apply_b(u)};
      for (const auto& r : results)
        for (Index j = 0; j < 24; ++j)
          for (Index i = 0; i < 24; ++i)
            if (!g.mask(i, j)) CHECK(r.values(i, j) == 0.0);
    }
  }
  {  // :339-359 coefficient bytes and ghost resolution
    Grid2D g = Grid2D::uniform(32, 20, 6000.0, 6000.0);
    const ScaleField s = uniform_scale(g, 12000.0);
    const HorizontalCovarianceOp op1(g, s, opts(FilterOrder::first, 5, true));
    const HorizontalCovarianceOp op3(g, s, opts(FilterOrder::third, 1, true));
    CHECK(op3.coefficient_bytes() == 2 * op1.coefficient_bytes());
    CHECK(op1.coefficient_bytes() == 2 * 2 * sizeof(double) * 32 * 20);
    Grid2D h = Grid2D::uniform(16, 16, 6000.0, 6000.0);
    const ScaleField hs = uniform_scale(h, 12000.0);
    CHECK(HorizontalCovarianceOp(h, hs).effective_ghost_width() == 18);
    h.ghost_width = 7;
    CHECK(HorizontalCovarianceOp(h, hs).effective_ghost_width() == 7);
    CHECK(HorizontalCovarianceOp(h, hs, opts(FilterOrder::third, 1, true, 0)).effective_ghost_width() == 0);
    CHECK(HorizontalCovarianceOp(h, hs, opts(FilterOrder::third, 1, true, 3)).effective_ghost_width() == 3);
  }
  {  // :361-374 determinism (the GPU analogue of thread-count invariance)
    Grid2D g = Grid2D::uniform(48, 40, 6000.0, 6000.0);
    g.mask = checkered(48, 40, 5, 0.85);
    std::mt19937 rng(71);
    const StateField u{&g, random_field(48, 40, rng)};
    CovarianceOptions o4 = opts(FilterOrder::third, 1, true);
    o4.threads = 4;
    const Field a = HorizontalCovarianceOp(g, uniform_scale(g, 12000.0), opts(FilterOrder::third, 1, true)).apply_b(u).values;
    const Field b = HorizontalCovarianceOp(g, uniform_scale(g, 12000.0), o4).apply_b(u).values;
    bool same = true;
    for (Index k = 0; k < a.size(); ++k) same = same && a.data()[k] == b.data()[k];
    CHECK(same);
  }
  {  // :376-381 and :484-492 rejections
    const Grid2D g = Grid2D::uniform(8, 8, 6000.0, 6000.0);
    CHECK_THROWS_AS(HorizontalCovarianceOp(g, uniform_scale(g, 12000.0), opts(FilterOrder::third, 2, true)),
                    std::invalid_argument);
    const Grid2D g16 = Grid2D::uniform(16, 16, 6000.0, 6000.0);
    const Grid2D other = Grid2D::uniform(18, 16, 6000.0, 6000.0);
    const HorizontalCovarianceOp op(g16, uniform_scale(g16, 12000.0));
    const StateField f = StateField::zeros(other);
    CHECK_THROWS_AS(op.apply_gx(f), std::invalid_argument);
    CHECK_THROWS_AS(op.apply_b(f), std::invalid_argument);
  }
  // ---- proj/tests/test_solver.cpp through rgf_b200/solver.hpp
  auto make_obs = [](std::initializer_list<std::array<double, 4>> rows) {
    ObsSet o;
    const Index n = static_cast<Index>(rows.size());
    o.positions.resize(n, 2);
    o.values.resize(n);
    o.r_var.resize(n);
    Index k = 0;
    for (const auto& r : rows) {
      o.positions(k, 0) = r[0];
      o.positions(k, 1) = r[1];
      o.values[k] = r[2];
      o.r_var[k] = r[3];
      ++k;
    }
    return o;
  };
  {  // :45-58 exact on affine fields and nodes
    const Grid2D g = Grid2D::uniform(8, 8, 1000.0, 1000.0);
    StateField f = StateField::zeros(g);
    for (Index j = 0; j < 8; ++j)
      for (Index i = 0; i < 8; ++i) f.values(i, j) = 2.0 * i - 3.0 * j + 1.0;
    const Vector h = obs_operator(f, make_obs({{3.5, 2.0, 0.0, 1.0}, {5.0, 5.0, 0.0, 1.0}}));
    CHECK(std::abs(h[0] - (2.0 * 3.5 - 3.0 * 2.0 + 1.0)) <= 1e-14 * 2.0);
    CHECK(h[1] == f.values(5, 5));
  }
  {  // :60-74 rejects all-land stencils and outside positions
    Grid2D g = Grid2D::uniform(8, 8, 1000.0, 1000.0);
    g.mask(3, 3) = g.mask(4, 3) = g.mask(3, 4) = g.mask(4, 4) = 0;
    const StateField f = StateField::zeros(g);
    CHECK_THROWS_AS(obs_operator(f, make_obs({{3.5, 3.5, 0.0, 1.0}})), std::invalid_argument);
    CHECK_THROWS_AS(obs_operator(f, make_obs({{-0.5, 2.0, 0.0, 1.0}})), std::invalid_argument);
  }
  {  // :165-192 single observation increment
    const Grid2D g = Grid2D::uniform(64, 64, 6000.0, 6000.0);
    const HorizontalCovarianceOp op(g, uniform_scale(g, 12000.0));
    const Analysis an = solve(make_obs({{32, 32, 1.0, 1.0}}), op, {1e-10, 50});
    CHECK(an.converged);
    double peak = -1e300;
    Index imax = -1, jmax = -1;
    for (Index j = 0; j < 64; ++j)
      for (Index i = 0; i < 64; ++i)
        if (an.increment.values(i, j) > peak) {
          peak = an.increment.values(i, j);
          imax = i;
          jmax = j;
        }
    CHECK(imax == 32 && jmax == 32);
    CHECK(peak > 0.0 && peak < 1.0);
  }
  {  // :239-250 hitting max_iter flags non-convergence; :139-163 bad options
    const Grid2D g = Grid2D::uniform(24, 24, 6000.0, 6000.0);
    const HorizontalCovarianceOp op(g, uniform_scale(g, 12000.0));
    const Analysis an = solve(
        make_obs({{5, 5, 1.0, 0.1}, {12, 12, -1.0, 0.1}, {18, 6, 2.0, 0.1}}), op, {1e-15, 1});
    CHECK(!an.converged);
    CHECK(an.cg_iterations == 1);
    CHECK(an.gradient_norms.size() == 2);
    CHECK_THROWS_AS(solve(make_obs({{6, 6, 1.0, 1.0}}), op, {0.0, 30}), std::invalid_argument);
    const CostReport r = cost(StateField::zeros(g), make_obs({{3.0, 4.0, 1.0, 0.5}}), op);
    CHECK(std::abs(r.j_total - 0.5 * 1.0 / 0.5) <= 1e-14);
  }
  std::printf("%d checks, %d failures\n", checks, failures);
  return failures == 0 ? 0 : 1;
}
