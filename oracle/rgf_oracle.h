/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * An Eigen-free C++ restatement of the reference hot path (rgfvar,
 * /root/reference/proj): rf1.hpp, rf3.hpp, grid.cpp, covariance.cpp and
 * parallel.hpp, kept in the reference's evaluation order and compiled with
 * -ffp-contract=off so that it reproduces the reference's IEEE arithmetic.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the timed CPU baseline. The product (paper_1404_5756_b200) never links it.
 *
 * Parity is pinned against the reference's own golden tables and known-answer
 * tests (tests/test_oracle_*.py restate test_rf1.cpp, test_rf3.cpp,
 * test_covariance.cpp and acceptance.cpp cases). The reference itself cannot
 * be compiled here (Eigen3 / CLI11 / doctest are absent).
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: 0 ok, 1 invalid argument, 2 runtime error */
const char* rgfo_last_error(void);

/* rf3.hpp:78-95 -> out = {a0, a1, a2, a3, alpha1, alpha2, alpha3, beta} */
int rgfo_rf3_coefficients(double sigma, double out[8]);
/* rf3.hpp:166-181 -> out = {alpha1, alpha2, alpha3, beta, q} */
int rgfo_rf3_filter_scalars(double sigma, int calibration, double out[5]);
/* rf3.hpp:101-108 */
double rgfo_rf3_cascade_variance(double q);
/* rf3.hpp:143-154 */
double rgfo_rf3_length_scale_argument(double sigma, int calibration);
/* rf1.hpp:76-85 -> out = {alpha, beta} */
int rgfo_rf1_coefficients(double sigma, int k, double out[2]);
/* rf3.hpp:12-37 rational_gauss */
double rgfo_rational_gauss(double t);

/* 1-D entry points (rf3.hpp:292-334, rf1.hpp:113-155): per-point sigma,
 * coefficients built as rf3_filter_coefficients / rf1_coefficients do. */
int rgfo_rf3_apply_1d(const double* in, const double* sigma, int64_t m,
                      int calibration, int transpose, double* out);
int rgfo_rf1_apply_1d(const double* in, const double* sigma, int64_t m, int k,
                      int transpose, double* out);
/* Same, with explicit coefficient arrays (alpha2/alpha3 unused for rf1). */
int rgfo_rf3_apply_1d_coeffs(const double* in, const double* a1, const double* a2,
                             const double* a3, const double* b, int64_t m,
                             int transpose, double* out);

/* Batched covariance operator: nlev independent 2-D HorizontalCovarianceOp
 * instances sharing dx, dy, rx, ry; per-level masks (nlev*ny*nx, x fastest,
 * 1 = sea). ghost_width < 0 = unset. variance: NULL or nlev*ny*nx. */
typedef struct rgfo_op rgfo_op;
int rgfo_op_create(int64_t nx, int64_t ny, int64_t nlev, const double* dx,
                   const double* dy, const uint8_t* mask, int64_t grid_ghost_width,
                   const double* rx, const double* ry, int order, int k_iterations,
                   int unit_dc, int64_t ghost_width, const double* variance,
                   int threads, int calibration, rgfo_op** out);
void rgfo_op_destroy(rgfo_op* op);
/* kind: 0 gx, 1 gy, 2 gxT, 3 gyT, 4 v, 5 vT, 6 b, 7 gy(gx(.)) ;
 * in/out: nvar*nlev*ny*nx doubles. Levels [lev0, lev0+nlev_sub) only when
 * nlev_sub > 0 (bounded CPU-baseline samples); the arrays then hold
 * nvar*nlev_sub planes. */
int rgfo_op_apply(const rgfo_op* op, int kind, const double* in, double* out,
                  int64_t nvar, int64_t lev0, int64_t nlev_sub);
int64_t rgfo_op_ghost_width(const rgfo_op* op, int64_t level);
uint64_t rgfo_op_coefficient_bytes(const rgfo_op* op);
int rgfo_op_uniform(const rgfo_op* op, int64_t level, int dir);
int rgfo_resolve_thread_count(int requested);

/* Observation operator and CG analysis (obs.cpp, solver.cpp) on a one-level
 * operator: positions x, y in fractional grid indices; fields ny*nx. */
typedef struct rgfo_obs rgfo_obs;
int rgfo_obs_create(const rgfo_op* op, int64_t n, const double* x, const double* y,
                    const double* values, const double* r_var, rgfo_obs** out);
void rgfo_obs_destroy(rgfo_obs* o);
int rgfo_obs_apply(const rgfo_op* op, const rgfo_obs* o, int transpose, const double* in,
                   double* out);
int rgfo_cost(const rgfo_op* op, const rgfo_obs* o, const double* chi, const double* background,
              double* j3, double* gradient);
int rgfo_solve(const rgfo_op* op, const rgfo_obs* o, double tol, int max_iter,
               const double* background, double* increment, double* misfit, double* gnorms,
               int64_t* info, double* out3);

/* io.cpp:133-281 binary containers (rgf_oracle_io.cpp, nlohmann::json) */
const char* rgfo_io_last_error(void);
int rgfo_load_grid(const char* path, int64_t nx, int64_t ny, double* dx, double* dy,
                   uint8_t* mask, int64_t* ghost_width);
int rgfo_save_grid(const char* path, int64_t nx, int64_t ny, int64_t ghost_width,
                   const double* dx, const double* dy, const uint8_t* mask);
int rgfo_load_scale(const char* path, int64_t nx, int64_t ny, double* rx, double* ry);
int rgfo_save_scale(const char* path, int64_t nx, int64_t ny, const double* rx, const double* ry);
int rgfo_load_field(const char* path, int64_t nx, int64_t ny, double* values);
int rgfo_save_field(const char* path, int64_t nx, int64_t ny, const double* values);

/* diagnostics.cpp:69-135 (rgf_oracle_diag.cpp) */
const char* rgfo_diag_last_error(void);
int rgfo_impulse_response(double sigma, int order, int k, int64_t length, int calibration,
                          double* h, double* sum_h, double* err_l2, double* err_max);
int rgfo_remark1(const double* s0, int64_t m, double sigma, int order, int k, int calibration,
                 double* out4);

#ifdef __cplusplus
}
#endif
