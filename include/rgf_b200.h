/*
 * rgf_b200 — C ABI of the B200-native recursive-filter covariance operator.
 *
 * Drop-in boundary for the hot path of rgfvar (arXiv 1404.5756, OceanVar
 * 3D-VAR horizontal covariance). Every entry point replaces a reference C++
 * interface; the reference file:line it stands for is given beside it (paths
 * relative to the reference's proj/ directory). Plain pointers and sizes
 * only; no torch or Eigen types cross this boundary.
 *
 * Memory layout (types.hpp:25-28, io.hpp:18-22): x fastest. A 2-D field is
 * nx*ny doubles with element (ix,iy) at iy*nx+ix. The batched 3-D extension
 * is [var][lev][iy][ix]; every level carries its own land mask and hence its
 * own segments and ghost width, exactly as a loop of independent 2-D
 * HorizontalCovarianceOp instances.
 *
 * Errors: every function returns RGF_OK (0) or a nonzero status and sets a
 * thread-local message, read with rgf_last_error(). RGF_EINVAL corresponds to
 * the reference's std::invalid_argument with the same message text; the C++
 * facade (rgf_b200/covariance.hpp) rethrows it as such.
 *
 * There is no CPU fallback: every apply runs sm_100a kernels; without a CUDA
 * device the calls fail with RGF_ECUDA.
 */
#ifndef RGF_B200_H
#define RGF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RGF_OK 0
#define RGF_EINVAL 1   /* std::invalid_argument in the reference */
#define RGF_ERUNTIME 2 /* std::runtime_error */
#define RGF_ECUDA 3    /* device error (no reference counterpart) */

/* types.hpp:30 FilterOrder */
#define RGF_ORDER_FIRST 1
#define RGF_ORDER_THIRD 3
/* types.hpp:39 Rf3Calibration */
#define RGF_CAL_YVV95 0
#define RGF_CAL_VARIANCE_MATCH 1
#define RGF_CAL_NONE 2

/* covariance.hpp:40-47 apply_* methods; RGF_GYGX is diagnostics.cpp:182's
 * timed unit apply_gy(apply_gx(f)). */
#define RGF_GX 0
#define RGF_GY 1
#define RGF_GXT 2
#define RGF_GYT 3
#define RGF_V 4
#define RGF_VT 5
#define RGF_B 6
#define RGF_GYGX 7

#define RGF_F64 0 /* reference Scalar = double (types.hpp:14) */
#define RGF_F32 1 /* fp32 storage, fp64 coefficients and recursion registers */

#define RGF_HOST 0   /* in/out are host pointers: H2D, kernels, D2H */
#define RGF_DEVICE 1 /* in/out are device pointers on the op's device */

/* grid.hpp:20-37 Grid2D, with the level axis added. */
typedef struct rgf_grid_desc {
  int64_t nx, ny;        /* nx, ny >= 4 (grid.cpp:28) */
  int64_t nlev;          /* independent levels, >= 1 */
  const double* dx;      /* nx*ny metres, > 0 */
  const double* dy;      /* nx*ny metres, > 0 */
  const uint8_t* mask;   /* nlev*ny*nx, nonzero = sea */
  int64_t ghost_width;   /* Grid2D::ghost_width, 0 = derive from sigma */
} rgf_grid_desc;

/* covariance.hpp:17-25 CovarianceOptions. */
typedef struct rgf_options {
  int32_t order;          /* RGF_ORDER_FIRST | RGF_ORDER_THIRD (default 3) */
  int32_t k_iterations;   /* default 1 */
  int32_t unit_dc;        /* default 1 */
  int32_t calibration;    /* default RGF_CAL_YVV95 */
  int64_t ghost_width;    /* < 0: unset (std::optional), default -1 */
  const double* variance; /* NULL or nlev*ny*nx (std::optional<Field>) */
  int32_t threads;        /* accepted for ABI parity; the GPU ignores it */
  int32_t device;         /* CUDA device ordinal, default 0 */
} rgf_options;

typedef struct rgf_op rgf_op;

const char* rgf_last_error(void);

/* CovarianceOptions{} defaults (covariance.hpp:17-25). */
void rgf_options_default(rgf_options* opt);

/* HorizontalCovarianceOp::HorizontalCovarianceOp (covariance.hpp:37-38,
 * covariance.cpp:155-220): validates grid/scales/options with the reference's
 * messages, resolves the per-level ghost width, builds the per-point
 * coefficient tables on the device (coefficient-precompute kernel) and the
 * sea-segment descriptors (segmentation scan/compaction kernels).
 * rx, ry: nx*ny metres (grid.hpp:40-52 ScaleField). */
int rgf_op_create(const rgf_grid_desc* grid, const double* rx, const double* ry,
                  const rgf_options* opt, rgf_op** out);
int rgf_op_destroy(rgf_op* op);

/* apply_gx / apply_gy / apply_gx_transpose / apply_gy_transpose / apply_v /
 * apply_v_transpose / apply_b (covariance.cpp:362-398), out of place.
 * in/out hold nvar*nlev*ny*nx elements of `dtype`. memory = RGF_HOST or
 * RGF_DEVICE. stream: a cudaStream_t or NULL (the legacy default stream).
 * Device applies are asynchronous on `stream`; host applies return after the
 * result is in `out`. */
int rgf_op_apply(rgf_op* op, int kind, int dtype, const void* in, void* out, int64_t nvar,
                 int memory, void* stream);

/* HorizontalCovarianceOp::effective_ghost_width (covariance.hpp:51), per level. */
int rgf_op_ghost_width(const rgf_op* op, int64_t level, int64_t* out);
/* HorizontalCovarianceOp::coefficient_bytes (covariance.cpp:222-226): the
 * reference's per-2-D-operator accounting 2 * {2|4} * 8 * nx*ny. */
int rgf_op_coefficient_bytes(const rgf_op* op, uint64_t* out);
/* Device bytes actually held by the operator (tables, descriptors, scratch). */
int rgf_op_device_bytes(const rgf_op* op, uint64_t* out);
/* Number of kernels this op has launched so far (bench evidence). */
int rgf_op_launch_count(const rgf_op* op, uint64_t* out);

/* Sea-segment descriptors built by the segmentation kernel, for bit-exact
 * checks against covariance.cpp:246-269. dir 0 = x lines (nlev*ny lines),
 * 1 = y lines (nlev*nx lines). offsets: nlines+1 entries (prefix sums);
 * segs: 2*nsegs int32 (start, len). Pass NULL to query sizes. */
int rgf_op_segments(const rgf_op* op, int dir, int64_t* nlines, int64_t* nsegs,
                    int64_t* offsets, int32_t* segs);

/* Per-point coefficient tables (device-computed), for parity checks of the
 * coefficient-precompute kernel against rf3.hpp:166-210 / rf1.hpp:96-110 /
 * covariance.cpp:182-206. dir 0 = x, 1 = y. out_* are nx*ny doubles; pass
 * NULL for tables the order does not have. */
int rgf_op_coefficients(const rgf_op* op, int dir, double* alpha1, double* alpha2,
                        double* alpha3, double* beta, double* inv_dc);

/* Scalar coefficient builders evaluated on the device.
 * rf3.hpp:78-95 rf3_coefficients -> {a0,a1,a2,a3,alpha1,alpha2,alpha3,beta} */
int rgf_rf3_coefficients(double sigma, double out[8]);
/* rf3.hpp:166-181 rf3_filter_scalars -> {alpha1,alpha2,alpha3,beta,q} */
int rgf_rf3_filter_scalars(double sigma, int calibration, double out[5]);
/* rf1.hpp:76-85 rf1_coefficients -> {alpha, beta} */
int rgf_rf1_coefficients(double sigma, int k, double out[2]);

/* rf3.hpp:101-108 rf3_cascade_variance(q) */
int rgf_rf3_cascade_variance(double q, double* out);
/* rf3.hpp:143-154 rf3_length_scale_argument(sigma, calibration) */
int rgf_rf3_length_scale_argument(double sigma, int calibration, double* out);

/* 1-D entry points over a batch of `nlines` contiguous host vectors of
 * length m (one coefficient table, shared by the batch).
 *
 * Per-point sigma (m doubles) turned into coefficients on the device:
 * rf3_apply_1d / rf3_apply_transpose_1d (rf3.hpp:318-334 with
 * rf3_filter_coefficients, rf3.hpp:191-210) and rf1_apply_1d /
 * rf1_apply_transpose_1d (rf1.hpp:139-155 with the table overload of
 * rf1_coefficients, rf1.hpp:96-110). */
int rgf_rf3_apply_1d(const double* in, const double* sigma, int64_t m, int64_t nlines,
                     int calibration, int transpose, double* out);
int rgf_rf1_apply_1d(const double* in, const double* sigma, int64_t m, int64_t nlines,
                     int k, int transpose, double* out);

/* Coefficient tables (the reference's Rf3CoefficientsT / Rf1CoefficientsT):
 * rf3_filter_coefficients(sigma, calibration) (rf3.hpp:191-210) and the
 * table overload rf1_coefficients(sigma, k) (rf1.hpp:96-110), m points. */
int rgf_rf3_filter_coefficients(const double* sigma, int64_t m, int calibration,
                                double* alpha1, double* alpha2, double* alpha3, double* beta);
int rgf_rf1_coefficients_table(const double* sigma, int64_t m, int k, double* alpha,
                               double* beta);

/* Filters with caller-supplied tables: rf3_filter_in_place /
 * rf3_filter_transpose_in_place / rf3_apply_1d(segment, coefficients)
 * (rf3.hpp:292-334) and rf1_filter_in_place / rf1_filter_transpose_in_place /
 * rf1_apply_1d(segment, coefficients) (rf1.hpp:113-155). `in` may equal
 * `out` (in place). Errors as the reference: "rf3 filter: segment length must
 * be >= 4", "rf1 filter: segment length must be >= 2". */
int rgf_rf3_filter(const double* in, const double* alpha1, const double* alpha2,
                   const double* alpha3, const double* beta, int64_t m, int64_t nlines,
                   int transpose, double* out);
int rgf_rf1_filter(const double* in, const double* alpha, const double* beta, int64_t m,
                   int64_t nlines, int k, int transpose, double* out);


/* ------------------------------------------------------------------------
 * Batched diagnostics (diagnostics.cpp:69-135), one
 * device thread per study, host arrays.
 * impulse_response(sigma[s], order, k, length, calibration) for n studies:
 * h is n x length (raw response to a Dirac at length/2), and per study
 * sum_h, err_h_l2, err_h_max (vs the unit-sum sampled Gaussian). */
int rgf_impulse_responses(const double* sigma, int64_t n, int order, int k, int64_t length,
                          int calibration, double* h, double* sum_h, double* err_h_l2,
                          double* err_h_max);
/* remark1_bound_check(s0[s], sigma[s], order, k, calibration) for n inputs of
 * length m (s0 is n x m): out4[4*s..] = {lhs, rhs, err_h_l2, holds (0/1)} */
int rgf_remark1_checks(const double* s0, const double* sigma, int64_t n, int64_t m, int order,
                       int k, int calibration, double* out4);

/* ------------------------------------------------------------------------
 * Container I/O (io.cpp:133-281, proj/README.md "File
 * formats"): rgf-grid / rgf-scale / rgf-field binary containers (one JSON
 * header line, then raw little-endian f64 sections in header order, x
 * fastest; masks one byte per point). Errors: RGF_ERUNTIME with io.cpp's
 * messages ("cannot open <path>", "expected a \"rgf-field\" container",
 * "field file dimensions do not match the grid", "payload section \"values\"
 * is truncated (dimension mismatch?)", ...), RGF_EINVAL for grid.cpp's
 * validation. Headers are written as nlohmann::json::dump() writes them, so
 * a save/load round trip is byte-identical. */
/* header of any container: format (<= 31 chars + NUL), nx, ny, ghost_width
 * (0 if absent), nlev (1 if absent; rgf-field level stacks, an extension) */
int rgf_container_info(const char* path, char* format, int64_t* nx, int64_t* ny,
                       int64_t* ghost_width, int64_t* nlev);
/* rgf-grid -> caller buffers (nx*ny each); validated as Grid2D::validate */
int rgf_grid_load(const char* path, int64_t nx, int64_t ny, double* dx, double* dy,
                  uint8_t* mask, int64_t* ghost_width);
int rgf_grid_save(const char* path, const rgf_grid_desc* grid); /* level 0 of the mask */
/* rgf-scale -> rx, ry (nx*ny each), validated against the grid (grid.cpp:40-55) */
int rgf_scale_load(const char* path, const rgf_grid_desc* grid, double* rx, double* ry);
int rgf_scale_save(const char* path, int64_t nx, int64_t ny, const double* rx, const double* ry);
/* rgf-field (nlev levels) streamed straight into / out of `memory`
 * (RGF_HOST or RGF_DEVICE, the latter through two pinned chunks overlapping
 * the file I/O with the copies on `stream`); dtype RGF_F32 converts on the
 * device (payloads are f64). */
int rgf_field_load(const char* path, int64_t nx, int64_t ny, int64_t nlev, int dtype, void* dst,
                   int memory, void* stream);
int rgf_field_save(const char* path, int64_t nx, int64_t ny, int64_t nlev, int dtype,
                   const void* src, int memory, void* stream);

/* ------------------------------------------------------------------------
 * Observation operator and 3D-VAR analysis, on an
 * operator with one level. Replaces obs.hpp:15-46 (ObsSet, obs_operator,
 * obs_operator_transpose, misfit) and solver.hpp:19-55 (SolveOptions,
 * Analysis, cost, solve). Positions are fractional grid indices (x, y);
 * fields are ny*nx doubles, x fastest. Errors: RGF_EINVAL with the
 * reference's messages ("observation n: ...", "solve: tol must be
 * positive", "solve: max_iter must be >= 0").
 * ------------------------------------------------------------------------ */
typedef struct rgf_obs rgf_obs;

typedef struct rgf_analysis {
  int32_t cg_iterations;
  int32_t converged;
  int64_t n_gradient_norms; /* initial residual + one per iteration */
  double final_relative_residual;
  double j_background;
  double j_obs;
} rgf_analysis;

/* obs.cpp:18-57: an ObsSet bound to a grid (level-0 mask) on a device;
 * stencils validated here (bilinear_stencil messages) */
int rgf_obs_create(const rgf_grid_desc* grid, int32_t device, int64_t n, const double* x,
                   const double* y, const double* values, const double* r_var,
                   rgf_obs** out);
int rgf_obs_destroy(rgf_obs* obs);
/* transpose 0: out[n] = H in (field, obs.cpp:59-71); 1: out (field) = H^T
 * in[n] (obs.cpp:73-87); memory RGF_HOST | RGF_DEVICE */
int rgf_obs_apply(rgf_obs* obs, int transpose, const double* in, double* out, int memory,
                  void* stream);
/* solver.cpp:35-50 (host arrays): j3 = {J, J_b, J_o}; background may be NULL */
int rgf_cost(rgf_op* op, rgf_obs* obs, const double* chi, const double* background,
             double* j3, double* gradient);
/* solver.cpp:52-114 (host arrays): increment (field), misfit (n, may be
 * NULL), gradient_norms (max_iter + 1 slots); background may be NULL */
int rgf_solve(rgf_op* op, rgf_obs* obs, double tol, int32_t max_iter,
              const double* background, double* increment, double* misfit,
              double* gradient_norms, rgf_analysis* out);

#ifdef __cplusplus
}
#endif

#endif /* RGF_B200_H */
