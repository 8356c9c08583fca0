// Device kernels of the observation operator and the CG analysis
// (reference obs.cpp, solver.cpp).
//
//  * H (obs.cpp:59-71): one thread per observation, the four-corner bilinear
//    sum in the reference's order, unfused (bit-identical).
//  * H^T (obs.cpp:73-87): the reference scatters observation by observation;
//    here every touched grid cell gathers its contributions from a CSR list
//    built in observation order, so each cell's sum has the reference's
//    order and no atomics are needed (deterministic, bit-identical).
//  * dot products: fixed-shape two-stage tree reductions (deterministic; the
//    order differs from Eigen's vectorised sum, ~1 ulp).
//  * CG updates (solver.cpp:87-104): elementwise, unfused like Eigen's
//    expression evaluation.
#pragma once
#include "common.cuh"

namespace rgfb {

// obs: cell c = j0*nx + i0 and weights w[4] = (w00, w10, w01, w11)
__global__ void k_obs_h(const double* __restrict__ f, int64_t n, int64_t nx,
                        const int64_t* __restrict__ cell, const double4* __restrict__ w,
                        double* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cell[k];
    const double4 q = w[k];
    out[k] = dadd(dadd(dadd(dmul(q.x, f[c]), dmul(q.y, f[c + 1])), dmul(q.z, f[c + nx])),
                  dmul(q.w, f[c + nx + 1]));
  }
}

// d - H f (misfit / residual) fused with H
__global__ void k_obs_residual(const double* __restrict__ d, const double* __restrict__ hf,
                               int64_t n, double* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = dsub(d[k], hf[k]);
}

// out (zeroed by the caller) at each touched cell: sum over its contributions
// (obs o, corner q) in observation order of w[o][q] * (v[o] / r_var[o])
// (solver.cpp:27 scales by 1/r_var first; rvar == nullptr: no scaling)
__global__ void k_obs_ht(const double* __restrict__ v, const double* __restrict__ rvar,
                         int64_t ncell, const int64_t* __restrict__ cells,
                         const int64_t* __restrict__ ptr, const int32_t* __restrict__ ent,
                         const double* __restrict__ w, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ncell;
       t += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int64_t e = ptr[t]; e < ptr[t + 1]; ++e) {
      const int32_t oq = ent[e];  // obs * 4 + corner
      const int32_t o = oq >> 2;
      const double s = rvar ? ddiv(v[o], rvar[o]) : v[o];
      acc = dadd(acc, dmul(w[oq], s));
    }
    out[cells[t]] = acc;
  }
}

constexpr int kDotBlocks = 296, kDotThreads = 256;

// partial[b] = sum over this block's grid-stride share of a[i]*b[i]
// (or of a[i]*a[i]/r[i] when r != nullptr)
__global__ void __launch_bounds__(kDotThreads) k_dot1(const double* __restrict__ a,
                                                      const double* __restrict__ b,
                                                      const double* __restrict__ r, int64_t n,
                                                      double* __restrict__ partial) {
  __shared__ double sh[kDotThreads];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s = dadd(s, r ? ddiv(dmul(a[i], a[i]), r[i]) : dmul(a[i], b[i]));
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int k = kDotThreads / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) sh[threadIdx.x] = dadd(sh[threadIdx.x], sh[threadIdx.x + k]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}
__global__ void __launch_bounds__(kDotThreads) k_dot2(const double* __restrict__ partial, int nb,
                                                      double* __restrict__ out) {
  __shared__ double sh[kDotThreads];
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += kDotThreads) s = dadd(s, partial[i]);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int k = kDotThreads / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) sh[threadIdx.x] = dadd(sh[threadIdx.x], sh[threadIdx.x + k]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// y = a + s*x (solver.cpp:84 x + adjoint_rhs: s = 1; :92 chi += alpha p;
// :93 r -= alpha ap with s = -alpha... kept as a subtraction, see k_axmy)
__global__ void k_axpy(double* __restrict__ y, const double* __restrict__ a,
                       const double* __restrict__ x, double s, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = dadd(a[i], dmul(s, x[i]));
}
// y = a - s*x
__global__ void k_axmy(double* __restrict__ y, const double* __restrict__ a,
                       const double* __restrict__ x, double s, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = dsub(a[i], dmul(s, x[i]));
}
// y = a + x
__global__ void k_add(double* __restrict__ y, const double* __restrict__ a,
                      const double* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = dadd(a[i], x[i]);
}

}  // namespace rgfb
