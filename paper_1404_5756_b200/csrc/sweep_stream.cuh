// Streaming 3rd-RF sweeps (forward G_dir and adjoint G_dir^T).
//
// One thread per (plane, line); adjacent threads own adjacent lines, so a
// y-sweep (lines = columns) reads and writes every row as one coalesced
// 256 B warp access, and an x-sweep reads 32 B sectors per lane. Each line
// is processed as the reference does segment by segment
// (covariance.cpp:228-352), fused into two streaming passes:
//
//   A (ascending k): zero-state causal recursion inside every sea segment
//     (rf3.hpp:217-239; the reference's startup rows are exactly a zero
//     initial state), intermediate stored to `out`; land stores 0.
//   D (descending k): at each segment end j the anti-causal recursion is
//     entered through the right-ghost closure (below), then runs down the
//     segment (rf3.hpp:241-262), scales by inv_dc (covariance.cpp:317) and
//     the optional variance, and overwrites `out`. Land stays exactly 0.
//
// The adjoint (rf3.hpp:264-286, applied as backward_transpose then
// forward_transpose, covariance.cpp:325-333) is run in the equivalent
// register-resident gather form with the reference's accumulation order
// (alpha3 term, then alpha2, then alpha1).
//
// Right-ghost closure: the G imaginary points beyond a segment end carry zero
// input and the end point's replicated coefficients (covariance.cpp:38-44),
// so "continue the causal pass G steps, restart the anti-causal pass at the
// far end, come back G steps" is a fixed linear map from the 3-value causal
// state at j to the 3-value anti-causal state entering j. It depends only on
// (coefficients at j, G) and is precomputed per point and per distinct ghost
// width at construction (k_closures). Left ghosts provably never affect a
// 3rd-RF segment (zero input, zero state), so they cost
// nothing. The recursion uses FMA with the alpha1 term last, so one DFMA
// sits on the loop-carried path (11 cycles/step measured vs 33 for the
// reference's unfused order; profiles/r01_machine_probe.log).
#pragma once
#include "common.cuh"

namespace rgfb {

struct StreamArgs {
  int dir, transpose, unit_dc;
  int64_t nx, ny, nlev, nvar;
  const Coef3* c3;
  const double* idc;
  const uint64_t* bits;     // bit-packed masks for this direction
  int64_t words;            // 64-bit words per line
  const int* ghost;         // per level
  const int* cls;           // per level closure class (-1: no right ghosts)
  const double* clos;       // [class][dir][nh][18]: M (9) then M^T-closure (9)
  const double* pre_scale;  // optional (nlev*nh) input multiplier (variance)
  const double* post_scale; // optional (nlev*nh) output multiplier
};

__device__ __forceinline__ int mbit(const uint64_t* w, int64_t k, int64_t n) {
  if (k < 0 || k >= n) return 0;
  return static_cast<int>((__ldg(reinterpret_cast<const unsigned long long*>(w) + (k >> 6)) >>
                           (k & 63)) & 1ull);
}

template <typename T>
__device__ __forceinline__ double ldv(const T* p) {
  return static_cast<double>(*p);
}

__device__ __forceinline__ Coef3 ldc(const Coef3* p) {
  const double2 lo = __ldg(reinterpret_cast<const double2*>(p));
  const double2 hi = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return Coef3{lo.x, lo.y, hi.x, hi.y};
}

template <typename T, int DIR, bool TR>
__global__ void __launch_bounds__(128) k_stream(const T* __restrict__ in, T* __restrict__ out,
                                                StreamArgs a) {
  const int64_t n = DIR == 0 ? a.nx : a.ny;
  const int64_t nlines = DIR == 0 ? a.ny : a.nx;
  const int64_t nh = a.nx * a.ny;
  const int64_t stride = DIR == 0 ? 1 : a.nx;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t planes = a.nvar * a.nlev;
  if (tid >= planes * nlines) return;
  const int64_t plane = tid / nlines;
  const int64_t line = tid - plane * nlines;
  const int64_t lev = plane % a.nlev;
  const int64_t hb = DIR == 0 ? line * a.nx : line;  // horizontal index of k=0
  const T* src = in + plane * nh + hb;
  T* dst = out + plane * nh + hb;
  const Coef3* C = a.c3 + hb;
  const double* IDC = a.idc ? a.idc + hb : nullptr;
  const double* PRE = a.pre_scale ? a.pre_scale + lev * nh + hb : nullptr;
  const double* POST = a.post_scale ? a.post_scale + lev * nh + hb : nullptr;
  const uint64_t* W = a.bits + (lev * nlines + line) * a.words;
  const int G = a.ghost[lev];
  const int cl = a.cls[lev];
  const double* CL = cl >= 0 ? a.clos + ((int64_t)(cl * 2 + DIR) * nh + hb) * 18 : nullptr;

  if (!TR) {
    // ---------------- pass A: causal, zero state per segment
    double p1 = 0.0, p2 = 0.0, p3 = 0.0;
    uint64_t wcur = 0;
    for (int64_t k = 0; k < n; ++k) {
      if ((k & 63) == 0) wcur = __ldg(reinterpret_cast<const unsigned long long*>(W) + (k >> 6));
      const bool sea = (wcur >> (k & 63)) & 1ull;
      const Coef3 c = ldc(C + k * stride);
      const double s = ldv(src + k * stride);
      const double t = fma(c.a1, p1, fma(c.a2, p2, fma(c.a3, p3, c.b * s)));
      p3 = sea ? p2 : 0.0;
      p2 = sea ? p1 : 0.0;
      p1 = sea ? t : 0.0;
      dst[k * stride] = static_cast<T>(p1);
    }
    // ---------------- pass D: anti-causal, entered through the closure
    double q1 = 0.0, q2 = 0.0, q3 = 0.0;
    int sea_next = 0;  // sea(k+1)
    wcur = 0;
    double z0 = ldv(dst + (n - 1) * stride);
    double zm1 = n >= 2 ? ldv(dst + (n - 2) * stride) : 0.0;
    for (int64_t k = n - 1; k >= 0; --k) {
      if (k == n - 1 || (k & 63) == 63)
        wcur = __ldg(reinterpret_cast<const unsigned long long*>(W) + (k >> 6));
      const int sea = static_cast<int>((wcur >> (k & 63)) & 1ull);
      const double zm2 = k >= 2 ? ldv(dst + (k - 2) * stride) : 0.0;  // read-ahead
      const Coef3 c = ldc(C + k * stride);
      if (sea && !sea_next) {  // segment end j = k
        q1 = q2 = q3 = 0.0;
        if (k < n - 1 && G > 0) {
          const int s1 = mbit(W, k - 1, n);
          const int s2 = s1 ? mbit(W, k - 2, n) : 0;
          const double x0 = z0, x1 = s1 ? zm1 : 0.0, x2 = s2 ? zm2 : 0.0;
          const double* M = CL + k * stride * 18;
          q1 = fma(M[0], x0, fma(M[1], x1, M[2] * x2));
          q2 = fma(M[3], x0, fma(M[4], x1, M[5] * x2));
          q3 = fma(M[6], x0, fma(M[7], x1, M[8] * x2));
        }
      }
      const double q = fma(c.a1, q1, fma(c.a2, q2, fma(c.a3, q3, c.b * z0)));
      double o = q;
      if (IDC) o *= __ldg(IDC + k * stride);
      if (POST) o *= __ldg(POST + k * stride);
      dst[k * stride] = static_cast<T>(sea ? o : 0.0);
      q3 = q2;
      q2 = q1;
      q1 = q;
      sea_next = sea;
      z0 = zm1;
      zm1 = zm2;
    }
  } else {
    // ---------------- pass A: transpose of the anti-causal pass (gather form)
    double u1 = 0.0, x1 = 0.0, y21 = 0.0, y22 = 0.0, y31 = 0.0, y32 = 0.0, y33 = 0.0;
    uint64_t wcur = 0;
    for (int64_t k = 0; k < n; ++k) {
      if ((k & 63) == 0) wcur = __ldg(reinterpret_cast<const unsigned long long*>(W) + (k >> 6));
      const bool sea = (wcur >> (k & 63)) & 1ull;
      const Coef3 c = ldc(C + k * stride);
      double w = ldv(src + k * stride);
      if (PRE) w *= __ldg(PRE + k * stride);
      if (IDC) w *= __ldg(IDC + k * stride);
      double u = fma(x1, u1, (w + y33) + y22);
      if (!sea) {
        u = 0.0;
        y31 = y32 = 0.0;
        y21 = 0.0;
      }
      y33 = y32;
      y32 = y31;
      y31 = c.a3 * u;
      y22 = y21;
      y21 = c.a2 * u;
      x1 = c.a1;
      u1 = u;
      dst[k * stride] = static_cast<T>(u);
    }
    // ---------------- pass D: transpose of the causal pass (gather form)
    double U1 = 0.0, X1 = 0.0, Y21 = 0.0, Y22 = 0.0, Y31 = 0.0, Y32 = 0.0, Y33 = 0.0;
    int sea_next = 0;
    wcur = 0;
    double z0 = ldv(dst + (n - 1) * stride);
    double zm1 = n >= 2 ? ldv(dst + (n - 2) * stride) : 0.0;
    for (int64_t k = n - 1; k >= 0; --k) {
      if (k == n - 1 || (k & 63) == 63)
        wcur = __ldg(reinterpret_cast<const unsigned long long*>(W) + (k >> 6));
      const int sea = static_cast<int>((wcur >> (k & 63)) & 1ull);
      const double zm2 = k >= 2 ? ldv(dst + (k - 2) * stride) : 0.0;
      const Coef3 c = ldc(C + k * stride);
      if (sea && !sea_next) {  // segment end j = k
        U1 = X1 = Y21 = Y22 = Y31 = Y32 = Y33 = 0.0;
        if (k < n - 1 && G > 0) {
          const int s1 = mbit(W, k - 1, n);
          const int s2 = s1 ? mbit(W, k - 2, n) : 0;
          const double uj = z0, ujm1 = s1 ? zm1 : 0.0, ujm2 = s2 ? zm2 : 0.0;
          const Coef3 cm1 = s1 ? ldc(C + (k - 1) * stride) : Coef3{0, 0, 0, 0};
          const Coef3 cm2 = s2 ? ldc(C + (k - 2) * stride) : Coef3{0, 0, 0, 0};
          // pending causal-transpose contributions into the ghosts
          const double P1 = fma(c.a1, uj, fma(cm1.a2, ujm1, cm2.a3 * ujm2));
          const double P2 = fma(c.a2, uj, cm1.a3 * ujm1);
          const double P3 = c.a3 * uj;
          const double* M = CL + k * stride * 18 + 9;
          const double g1 = fma(M[0], P1, fma(M[1], P2, M[2] * P3));
          const double g2 = fma(M[3], P1, fma(M[4], P2, M[5] * P3));
          const double g3 = fma(M[6], P1, fma(M[7], P2, M[8] * P3));
          U1 = g1;
          X1 = c.a1;
          Y21 = c.a2 * g1;
          Y22 = c.a2 * g2;
          Y31 = c.a3 * g1;
          Y32 = c.a3 * g2;
          Y33 = c.a3 * g3;
        }
      }
      const double v = c.b * z0;
      const double u = fma(X1, U1, (v + Y33) + Y22);
      double o = c.b * u;
      if (POST) o *= __ldg(POST + k * stride);
      dst[k * stride] = static_cast<T>(sea ? o : 0.0);
      Y33 = Y32;
      Y32 = Y31;
      Y31 = c.a3 * u;
      Y22 = Y21;
      Y21 = c.a2 * u;
      X1 = c.a1;
      U1 = u;
      sea_next = sea;
      z0 = zm1;
      zm1 = zm2;
    }
  }
}

// ------------------------------------------------------------ closures
// Per point p (horizontal), ghost width G, coefficients c = c3[p]:
//  M (forward op): state (p_j, p_{j-1}, p_{j-2}) -> (q_{j+1}, q_{j+2}, q_{j+3})
//    by G causal ghost steps with zero input, then the anti-causal pass from
//    the far end with zero state (the reference's startup rows).
//  Mt (adjoint): pending contributions (P1, P2, P3) into u_{j+1..j+3} ->
//    (u'_{j+1}, u'_{j+2}, u'_{j+3}) by the causal-transpose gather over the
//    ghosts, beta scaling, and the anti-causal-transpose gather back.
// Ghost recursions use the reference's unfused left-to-right order.
__global__ void k_closures(const Coef3* c3, int64_t nh, int G, double* out, double* scratch,
                           int64_t slab) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double* g = scratch + tid * slab;
  for (int64_t p = tid; p < nh; p += (int64_t)gridDim.x * blockDim.x) {
    const Coef3 c = c3[p];
    double* o = out + p * 18;
    for (int m = 0; m < 3; ++m) {
      // forward closure, basis state e_m over (p_j, p_{j-1}, p_{j-2})
      double pm1 = m == 0, pm2 = m == 1, pm3 = m == 2;
      for (int k = 0; k < G; ++k) {
        const double t = dadd(dadd(dmul(c.a1, pm1), dmul(c.a2, pm2)), dmul(c.a3, pm3));
        pm3 = pm2;
        pm2 = pm1;
        pm1 = t;
        g[k] = t;
      }
      double q1 = 0.0, q2 = 0.0, q3 = 0.0;
      double r[3] = {0.0, 0.0, 0.0};
      for (int k = G - 1; k >= 0; --k) {
        const double t = dadd(dadd(dadd(dmul(c.b, g[k]), dmul(c.a1, q1)), dmul(c.a2, q2)),
                              dmul(c.a3, q3));
        q3 = q2;
        q2 = q1;
        q1 = t;
        if (k < 3) r[k] = t;
      }
      o[0 + m] = r[0];
      o[3 + m] = r[1];
      o[6 + m] = r[2];

      // adjoint closure, basis pending contributions e_m over (P1, P2, P3)
      const double P1 = m == 0, P2 = m == 1, P3 = m == 2;
      double u1 = 0.0, u2 = 0.0, u3 = 0.0;  // u_{k-1}, u_{k-2}, u_{k-3} (ghosts)
      for (int k = 0; k < G; ++k) {
        double u;
        if (k == 0)
          u = P1;
        else if (k == 1)
          u = dadd(P2, dmul(c.a1, u1));
        else if (k == 2)
          u = dadd(dadd(P3, dmul(c.a2, u2)), dmul(c.a1, u1));
        else
          u = dadd(dadd(dmul(c.a3, u3), dmul(c.a2, u2)), dmul(c.a1, u1));
        u3 = u2;
        u2 = u1;
        u1 = u;
        g[k] = dmul(c.b, u);  // v_{j+1+k}
      }
      double w1 = 0.0, w2 = 0.0, w3 = 0.0;  // u'_{k+1}, u'_{k+2}, u'_{k+3}
      double s[3] = {0.0, 0.0, 0.0};
      for (int k = G - 1; k >= 0; --k) {
        const double u = dadd(dadd(dadd(g[k], dmul(c.a3, w3)), dmul(c.a2, w2)), dmul(c.a1, w1));
        w3 = w2;
        w2 = w1;
        w1 = u;
        if (k < 3) s[k] = u;
      }
      o[9 + 0 + m] = s[0];
      o[9 + 3 + m] = s[1];
      o[9 + 6 + m] = s[2];
    }
  }
}

// Bit-packed masks per direction: dir 0 words[(lev*ny+iy)*W + ix/64],
// dir 1 words[(lev*nx+ix)*W + iy/64]; bit k = sea at line position k.
__global__ void k_pack_bits(const uint8_t* mask, int dir, int64_t nx, int64_t ny, int64_t nlev,
                            int64_t words, uint64_t* bits) {
  const int64_t nlines = dir == 0 ? ny : nx;
  const int64_t n = dir == 0 ? nx : ny;
  const int64_t total = nlev * nlines * words;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t wi = t % words;
    const int64_t ln = t / words;  // lev*nlines + line
    const int64_t lev = ln / nlines, line = ln - lev * nlines;
    uint64_t v = 0;
    for (int b = 0; b < 64; ++b) {
      const int64_t k = wi * 64 + b;
      if (k >= n) break;
      const int64_t idx = dir == 0 ? (lev * ny + line) * nx + k : (lev * ny + k) * nx + line;
      if (mask[idx]) v |= (1ull << b);
    }
    bits[t] = v;
  }
}

template <typename T>
int launch_stream_sweep(const T* in, T* out, const StreamArgs& a, cudaStream_t st) {
  const int64_t nlines = a.dir == 0 ? a.ny : a.nx;
  const int64_t total = a.nvar * a.nlev * nlines;
  const int threads = 128;
  const int64_t blocks = (total + threads - 1) / threads;
  if (a.dir == 0) {
    if (a.transpose)
      k_stream<T, 0, true><<<blocks, threads, 0, st>>>(in, out, a);
    else
      k_stream<T, 0, false><<<blocks, threads, 0, st>>>(in, out, a);
  } else {
    if (a.transpose)
      k_stream<T, 1, true><<<blocks, threads, 0, st>>>(in, out, a);
    else
      k_stream<T, 1, false><<<blocks, threads, 0, st>>>(in, out, a);
  }
  return 1;
}

}  // namespace rgfb
