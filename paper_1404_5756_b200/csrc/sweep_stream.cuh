// Streaming 3rd-RF sweeps (forward G_dir and adjoint G_dir^T).
//
// Each chain is one (plane, line) of the field; the reference processes it
// segment by segment (covariance.cpp:228-352). Here every chain runs two
// streaming passes over the whole line:
//
//   A (ascending k): zero-state causal recursion inside every sea segment
//     (rf3.hpp:217-239 — the reference's startup rows are exactly a zero
//     initial state); the intermediate is stored to `out`, land stores 0.
//   D (descending k): at each segment end j the anti-causal recursion is
//     entered through the right-ghost closure (closures.cuh), runs down the
//     segment (rf3.hpp:241-262), is scaled by inv_dc (covariance.cpp:317)
//     and the optional variance, and overwrites `out`. Land stays exactly 0.
//
// The adjoint (rf3.hpp:264-286, backward_transpose then forward_transpose,
// covariance.cpp:325-333) runs in the equivalent register-resident gather
// form with the reference's accumulation order (alpha3 term, then alpha2,
// then alpha1).
//
// Left ghosts never affect a 3rd-RF segment (zero input, zero state;
// SURVEY.md §8a) and cost nothing. The recursion uses FMA with the alpha1
// term last, so one DFMA sits on the loop-carried path (11 cycles/step vs
// 33 for the reference's unfused order, profiles/r01_machine_probe.log).
//
// Thread mappings (memory-system driven):
//   y-sweep (lines = columns): lanes own adjacent columns, so every row step
//     is one coalesced warp access; each thread carries L planes of its
//     column (ILP, and one coefficient load serves L chains).
//   x-sweep (lines = rows): lanes own the same row of consecutive planes, so
//     the coefficient loads are warp-uniform broadcasts; each lane streams
//     its row in 8-element vector batches (64 B fp64 / 32 B fp32).
#pragma once
#include <type_traits>

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
  const int* cls;           // per level closure class
  const double* clos;       // [class][dir][nh][18]: M (9) then adjoint closure (9)
  const double* pre_scale;  // optional (nlev*nh) input multiplier (variance)
  const double* post_scale; // optional (nlev*nh) output multiplier
};

__device__ __forceinline__ int mbit(const uint64_t* w, int64_t k, int64_t n) {
  if (k < 0 || k >= n) return 0;
  return static_cast<int>((__ldg(reinterpret_cast<const unsigned long long*>(w) + (k >> 6)) >>
                           (k & 63)) & 1ull);
}
__device__ __forceinline__ uint64_t ldw(const uint64_t* w, int64_t i) {
  return __ldg(reinterpret_cast<const unsigned long long*>(w) + i);
}
__device__ __forceinline__ Coef3 ldc(const Coef3* p) {
  const double2 lo = __ldg(reinterpret_cast<const double2*>(p));
  const double2 hi = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return Coef3{lo.x, lo.y, hi.x, hi.y};
}
template <typename T>
__device__ __forceinline__ double ldv(const T* p) {  // coherent: reads this thread's writes
  return static_cast<double>(*p);
}

// ---------------------------------------------------------- chain states
struct FwdA {  // causal: p_{k-1}, p_{k-2}, p_{k-3}
  double p1 = 0.0, p2 = 0.0, p3 = 0.0;
  __device__ __forceinline__ double step(const Coef3& c, double s, bool sea) {
    const double t = fma(c.a1, p1, fma(c.a2, p2, fma(c.a3, p3, c.b * s)));
    p3 = sea ? p2 : 0.0;
    p2 = sea ? p1 : 0.0;
    p1 = sea ? t : 0.0;
    return p1;
  }
};
struct FwdD {  // anti-causal: q_{k+1}, q_{k+2}, q_{k+3}
  double q1 = 0.0, q2 = 0.0, q3 = 0.0;
  __device__ __forceinline__ void enter(const double* M, double x0, double x1, double x2) {
    q1 = fma(M[0], x0, fma(M[1], x1, M[2] * x2));
    q2 = fma(M[3], x0, fma(M[4], x1, M[5] * x2));
    q3 = fma(M[6], x0, fma(M[7], x1, M[8] * x2));
  }
  __device__ __forceinline__ double step(const Coef3& c, double z) {
    const double q = fma(c.a1, q1, fma(c.a2, q2, fma(c.a3, q3, c.b * z)));
    q3 = q2;
    q2 = q1;
    q1 = q;
    return q;
  }
};
struct AdjA {  // transpose of the anti-causal pass, gather form
  double u1 = 0.0, x1 = 0.0, y21 = 0.0, y22 = 0.0, y31 = 0.0, y32 = 0.0, y33 = 0.0;
  __device__ __forceinline__ double step(const Coef3& c, double w, bool sea) {
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
    return u;
  }
};
struct AdjD {  // transpose of the causal pass, gather form
  double U1 = 0.0, X1 = 0.0, Y21 = 0.0, Y22 = 0.0, Y31 = 0.0, Y32 = 0.0, Y33 = 0.0;
  __device__ __forceinline__ void reset() { U1 = X1 = Y21 = Y22 = Y31 = Y32 = Y33 = 0.0; }
  // P1..P3: pending causal-transpose contributions of u_j, u_{j-1}, u_{j-2}
  // into the first three ghosts; the closure returns u'_{j+1..j+3}.
  __device__ __forceinline__ void enter(const double* M, const Coef3& c, const Coef3& cm1,
                                        const Coef3& cm2, double uj, double ujm1, double ujm2) {
    const double P1 = fma(c.a1, uj, fma(cm1.a2, ujm1, cm2.a3 * ujm2));
    const double P2 = fma(c.a2, uj, cm1.a3 * ujm1);
    const double P3 = c.a3 * uj;
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
  __device__ __forceinline__ double step(const Coef3& c, double z) {
    const double v = c.b * z;
    const double u = fma(X1, U1, (v + Y33) + Y22);
    Y33 = Y32;
    Y32 = Y31;
    Y31 = c.a3 * u;
    Y22 = Y21;
    Y21 = c.a2 * u;
    X1 = c.a1;
    U1 = u;
    return c.b * u;
  }
};

// Segment-end entry of pass D for chain data (dst: this chain's line, W: its
// mask words, CL: its closure row, C: coefficient line, stride along k).
template <bool TR, typename T, typename DState>
__device__ __forceinline__ void enter_segment(DState& st, int64_t k, int64_t n, int G,
                                              const T* dst, const uint64_t* W, const double* CL,
                                              const Coef3* C, int64_t stride, const Coef3& c,
                                              double z0) {
  if constexpr (TR) st.reset();
  else st.q1 = st.q2 = st.q3 = 0.0;
  if (k < n - 1 && G > 0) {
    const int s1 = mbit(W, k - 1, n);
    const int s2 = s1 ? mbit(W, k - 2, n) : 0;
    const double z1 = s1 ? ldv(dst + (k - 1) * stride) : 0.0;
    const double z2 = s2 ? ldv(dst + (k - 2) * stride) : 0.0;
    const double* M = CL + k * stride * 18;
    if constexpr (!TR) {
      st.enter(M, z0, z1, z2);
    } else {
      const Coef3 cm1 = s1 ? ldc(C + (k - 1) * stride) : Coef3{0, 0, 0, 0};
      const Coef3 cm2 = s2 ? ldc(C + (k - 2) * stride) : Coef3{0, 0, 0, 0};
      st.enter(M + 9, c, cm1, cm2, z0, z1, z2);
    }
  }
}

// ================================================================ y-sweep
template <typename T, bool TR, int L, int U>
__global__ void __launch_bounds__(128) k_sweep_y(const T* __restrict__ in, T* __restrict__ out,
                                                 StreamArgs a) {
  const int64_t nx = a.nx, n = a.ny, nh = nx * n;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t groups = (planes + L - 1) / L;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= groups * nx) return;
  const int64_t g = tid / nx, ix = tid - g * nx;
  const Coef3* C = a.c3 + ix;
  const double* IDC = a.idc ? a.idc + ix : nullptr;

  const T* src[L];
  T* dst[L];
  const uint64_t* W[L];
  const double* CL[L];
  const double* PRE[L];
  const double* POST[L];
  int G[L];
  bool on[L];
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const int64_t p = g * L + l;
    on[l] = p < planes;
    const int64_t pp = on[l] ? p : planes - 1;
    const int64_t lev = pp % a.nlev;
    src[l] = in + pp * nh + ix;
    dst[l] = out + pp * nh + ix;
    W[l] = a.bits + (lev * nx + ix) * a.words;
    G[l] = a.ghost[lev];
    const int cl = a.cls[lev];
    CL[l] = a.clos + ((int64_t)(cl * 2 + 1) * nh + ix) * 18;
    PRE[l] = a.pre_scale ? a.pre_scale + lev * nh + ix : nullptr;
    POST[l] = a.post_scale ? a.post_scale + lev * nh + ix : nullptr;
  }

  // ------------------------------ pass A
  {
    typename std::conditional<TR, AdjA, FwdA>::type st[L];
    uint64_t wc[L];
    for (int64_t k0 = 0; k0 < n; k0 += U) {
      if ((k0 & 63) == 0) {
#pragma unroll
        for (int l = 0; l < L; ++l) wc[l] = ldw(W[l], k0 >> 6);
      }
      Coef3 c[U];
      double s[L][U];
      double id[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = k0 + u;
        if (k < n) {
          c[u] = ldc(C + k * nx);
          if (TR) id[u] = IDC ? __ldg(IDC + k * nx) : 1.0;
#pragma unroll
          for (int l = 0; l < L; ++l) {
            s[l][u] = on[l] ? ldv(src[l] + k * nx) : 0.0;
            if (TR && PRE[l]) s[l][u] *= __ldg(PRE[l] + k * nx);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = k0 + u;
        if (k < n) {
#pragma unroll
          for (int l = 0; l < L; ++l) {
            const bool sea = (wc[l] >> (k & 63)) & 1ull;
            const double w = TR ? s[l][u] * id[u] : s[l][u];
            const double r = st[l].step(c[u], w, sea);
            if (on[l]) dst[l][k * nx] = static_cast<T>(r);
          }
        }
      }
    }
  }
  // ------------------------------ pass D
  {
    typename std::conditional<TR, AdjD, FwdD>::type st[L];
    uint64_t wc[L];
    int nxt[L];
#pragma unroll
    for (int l = 0; l < L; ++l) nxt[l] = 0;
    int64_t widx = -1;
    for (int64_t k0 = n - 1; k0 >= 0; k0 -= U) {
      Coef3 c[U];
      double z[L][U];
      double id[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = k0 - u;
        if (k >= 0) {
          c[u] = ldc(C + k * nx);
          id[u] = (!TR && IDC) ? __ldg(IDC + k * nx) : 1.0;
#pragma unroll
          for (int l = 0; l < L; ++l) z[l][u] = on[l] ? ldv(dst[l] + k * nx) : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = k0 - u;
        if (k >= 0) {
          if ((k >> 6) != widx) {
            widx = k >> 6;
#pragma unroll
            for (int l = 0; l < L; ++l) wc[l] = ldw(W[l], widx);
          }
#pragma unroll
          for (int l = 0; l < L; ++l) {
            const int sea = static_cast<int>((wc[l] >> (k & 63)) & 1ull);
            if (sea && !nxt[l] && on[l])
              enter_segment<TR>(st[l], k, n, G[l], dst[l], W[l], CL[l], C, nx, c[u], z[l][u]);
            double o = st[l].step(c[u], z[l][u]);
            if (!TR && IDC) o *= id[u];
            if (POST[l]) o *= __ldg(POST[l] + k * nx);
            if (on[l]) dst[l][k * nx] = static_cast<T>(sea ? o : 0.0);
            nxt[l] = sea;
          }
        }
      }
    }
  }
}

// ================================================================ x-sweep
// Vector batch of 8 consecutive elements of one lane's row.
template <typename T, bool VEC>
__device__ __forceinline__ void ld8(const T* p, double (&v)[8], int cnt) {
  if (VEC && cnt == 8) {
    if constexpr (sizeof(T) == 8) {
      const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double2 t = q[i];
        v[2 * i] = t.x;
        v[2 * i + 1] = t.y;
      }
    } else {
      const float4* q = reinterpret_cast<const float4*>(p);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const float4 t = q[i];
        v[4 * i] = t.x;
        v[4 * i + 1] = t.y;
        v[4 * i + 2] = t.z;
        v[4 * i + 3] = t.w;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = i < cnt ? static_cast<double>(p[i]) : 0.0;
  }
}
template <typename T, bool VEC>
__device__ __forceinline__ void st8(T* p, const double (&v)[8], int cnt) {
  if (VEC && cnt == 8) {
    if constexpr (sizeof(T) == 8) {
      double2* q = reinterpret_cast<double2*>(p);
#pragma unroll
      for (int i = 0; i < 4; ++i) q[i] = make_double2(v[2 * i], v[2 * i + 1]);
    } else {
      float4* q = reinterpret_cast<float4*>(p);
#pragma unroll
      for (int i = 0; i < 2; ++i)
        q[i] = make_float4(static_cast<float>(v[4 * i]), static_cast<float>(v[4 * i + 1]),
                           static_cast<float>(v[4 * i + 2]), static_cast<float>(v[4 * i + 3]));
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < cnt) p[i] = static_cast<T>(v[i]);
  }
}
__device__ __forceinline__ void ld8d(const double* p, double (&v)[8], int cnt, bool vec) {
  if (vec && cnt == 8) {
    const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double2 t = __ldg(q + i);
      v[2 * i] = t.x;
      v[2 * i + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = i < cnt ? __ldg(p + i) : 0.0;
  }
}

template <typename T, bool TR, bool VEC>
__global__ void __launch_bounds__(128) k_sweep_x(const T* __restrict__ in, T* __restrict__ out,
                                                 StreamArgs a) {
  const int64_t n = a.nx, ny = a.ny, nh = n * ny;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= planes * ny) return;
  const int64_t iy = tid / planes, p = tid - iy * planes;
  const int64_t lev = p % a.nlev;
  const int64_t hb = iy * n;
  const T* src = in + p * nh + hb;
  T* dst = out + p * nh + hb;
  const Coef3* C = a.c3 + hb;
  const double* IDC = a.idc ? a.idc + hb : nullptr;
  const double* PRE = a.pre_scale ? a.pre_scale + lev * nh + hb : nullptr;
  const double* POST = a.post_scale ? a.post_scale + lev * nh + hb : nullptr;
  const uint64_t* W = a.bits + (lev * ny + iy) * a.words;
  const int G = a.ghost[lev];
  const double* CL = a.clos + ((int64_t)(a.cls[lev] * 2 + 0) * nh + hb) * 18;
  const int64_t nb = (n + 7) / 8;

  // ------------------------------ pass A
  {
    typename std::conditional<TR, AdjA, FwdA>::type st;
    uint64_t wc = 0;
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t k0 = b * 8;
      const int cnt = static_cast<int>(n - k0 < 8 ? n - k0 : 8);
      if ((k0 & 63) == 0) wc = ldw(W, k0 >> 6);
      double s[8], id[8], pr[8];
      Coef3 c[8];
      ld8<T, VEC>(src + k0, s, cnt);
      if (TR) {
        if (IDC) ld8d(IDC + k0, id, cnt, VEC);
        if (PRE) ld8d(PRE + k0, pr, cnt, VEC);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (u < cnt) c[u] = ldc(C + k0 + u);
      double r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (u < cnt) {
          const bool sea = (wc >> ((k0 + u) & 63)) & 1ull;
          double w = s[u];
          if (TR) {
            if (PRE) w *= pr[u];
            if (IDC) w *= id[u];
          }
          r[u] = st.step(c[u], w, sea);
        }
      }
      st8<T, VEC>(dst + k0, r, cnt);
    }
  }
  // ------------------------------ pass D
  {
    typename std::conditional<TR, AdjD, FwdD>::type st;
    uint64_t wc = 0;
    int nxt = 0;
    for (int64_t b = nb - 1; b >= 0; --b) {
      const int64_t k0 = b * 8;
      const int cnt = static_cast<int>(n - k0 < 8 ? n - k0 : 8);
      wc = ldw(W, k0 >> 6);
      double z[8], id[8], po[8], r[8];
      Coef3 c[8];
      ld8<T, VEC>(dst + k0, z, cnt);
      if (!TR && IDC) ld8d(IDC + k0, id, cnt, VEC);
      if (POST) ld8d(POST + k0, po, cnt, VEC);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (u < cnt) c[u] = ldc(C + k0 + u);
#pragma unroll
      for (int u = 7; u >= 0; --u) {
        if (u < cnt) {
          const int64_t k = k0 + u;
          const int sea = static_cast<int>((wc >> (k & 63)) & 1ull);
          if (sea && !nxt) enter_segment<TR>(st, k, n, G, dst, W, CL, C, 1, c[u], z[u]);
          double o = st.step(c[u], z[u]);
          if (!TR && IDC) o *= id[u];
          if (POST) o *= po[u];
          r[u] = sea ? o : 0.0;
          nxt = sea;
        }
      }
      st8<T, VEC>(dst + k0, r, cnt);
    }
  }
}

template <typename T>
int launch_stream_sweep(const T* in, T* out, const StreamArgs& a, cudaStream_t st) {
  const int threads = 128;
  const int64_t planes = a.nvar * a.nlev;
  if (a.dir == 1) {
    constexpr int L = 4, U = 4;
    const int64_t total = ((planes + L - 1) / L) * a.nx;
    const int64_t blocks = (total + threads - 1) / threads;
    if (a.transpose)
      k_sweep_y<T, true, L, U><<<blocks, threads, 0, st>>>(in, out, a);
    else
      k_sweep_y<T, false, L, U><<<blocks, threads, 0, st>>>(in, out, a);
  } else {
    const int64_t total = planes * a.ny;
    const int64_t blocks = (total + threads - 1) / threads;
    // 16 B vector access needs every row start 16 B aligned
    const int64_t vec_elems = 16 / static_cast<int64_t>(sizeof(T));
    const bool vec = (a.nx % vec_elems == 0) &&
                     (reinterpret_cast<uintptr_t>(in) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    if (vec) {
      if (a.transpose)
        k_sweep_x<T, true, true><<<blocks, threads, 0, st>>>(in, out, a);
      else
        k_sweep_x<T, false, true><<<blocks, threads, 0, st>>>(in, out, a);
    } else {
      if (a.transpose)
        k_sweep_x<T, true, false><<<blocks, threads, 0, st>>>(in, out, a);
      else
        k_sweep_x<T, false, false><<<blocks, threads, 0, st>>>(in, out, a);
    }
  }
  return 1;
}

}  // namespace rgfb
