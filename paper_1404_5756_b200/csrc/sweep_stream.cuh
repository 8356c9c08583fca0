// Streaming 3rd-RF sweeps (forward G_dir and adjoint G_dir^T).
//
// A chain is one (plane, line) of the field; the reference filters it
// segment by segment (covariance.cpp:228-352). Here every chain is swept by
// three kernels:
//
//   A  (ascending k): zero-state causal recursion inside every sea segment
//      (rf3.hpp:217-239 — the reference's startup rows are exactly a zero
//      initial state); the intermediate is stored to `out`, land stores 0.
//   E  (one thread per chain, loop over its segments): the right-ghost
//      closure turns the causal state at each segment end j into the
//      anti-causal state entering j (closures.cuh); stored per segment.
//   D  (descending k): at each segment end the anti-causal recursion starts
//      from its (prefetched) entry state, runs down the segment
//      (rf3.hpp:241-262), is scaled by inv_dc (covariance.cpp:317) and the
//      optional variance, and overwrites `out`. Land stays exactly 0.
//
// Keeping the closure out of pass D removes every dependent load from the
// descending loop: a segment end costs three register moves and one
// prefetch issued a whole segment ahead.
//
// The adjoint (rf3.hpp:264-286: backward_transpose then forward_transpose,
// covariance.cpp:325-333) runs in the equivalent register-resident gather
// form with the reference's accumulation order (alpha3 term, then alpha2,
// then alpha1). Left ghosts never affect a 3rd-RF segment
// (zero input, zero state) and cost nothing. The recursion
// uses FMA with the alpha1 term last, so one DFMA sits on the loop-carried
// path (11 cycles/step vs 33 for the reference's unfused order;
// profiles/r01_machine_probe.log).
//
// Thread mappings:
//   y-sweep (lines = columns): lanes own adjacent columns, so every row step
//     is one coalesced 256 B warp access; each thread carries L planes of its
//     column (ILP; one coefficient load serves L chains).
//   x-sweep (lines = rows): lanes own the same row of consecutive planes, so
//     coefficient loads are warp-uniform broadcasts; the field is staged
//     through shared memory in [32 chains x 32 elements] tiles moved by
//     warp-cooperative cp.async (each instruction one 256 B row segment)
//     and read back per lane from a bank-conflict-free padded tile.
#pragma once
#include <type_traits>

#include "common.cuh"

namespace rgfb {

struct StreamArgs {
  int dir, transpose, unit_dc;
  int64_t nx, ny, nlev, nvar;
  int64_t pitch;            // field row stride in elements (>= nx; checkpointed kernels)
  int64_t lev0;             // first global level of this launch
  int64_t nlev_all;         // levels of the operator (bitsT stride)
  const Coef3* c3;
  const double* c3s;        // y direction only: SoA rows [ny][4][nx] (checkpointed sweeps)
  const double* idc;
  const double* idcp;       // idc with rows `ipitch` apart (16 B multiple; TMA maps)
  int64_t ipitch;
  const uint64_t* bits;     // bit-packed masks for this direction
  const uint64_t* bitsT;    // same words, chain-minor: x [iy][word][lev], y [lev][word][ix]
  int64_t words;            // 64-bit words per line
  const int* ghost;         // per level
  const int* cls;           // per level closure class
  int nclass;               // distinct ghost widths (classes)
  const double* clos;       // [class][dir][nh][18]: M (9) then adjoint closure (9)
  const int64_t* seg_off;   // per (lev, line) segment prefix offsets
  const int2* segs;         // (start, len)
  const int32_t* seg_line;  // per segment: lev*nlines + line
  const int64_t* close_order;  // segments sorted by (line, end, level)
  int64_t nsegs;            // segments of this direction (all levels)
  double4* entry;           // [var][nsegs] anti-causal entry states
  const double* pre_scale;  // optional (nlev*nh) input multiplier (variance)
  const double* post_scale; // optional (nlev*nh) output multiplier
  int box_planes;           // planes per TMA field box of the y kernels (<= the shape's)
};

__device__ __forceinline__ uint64_t ldw(const uint64_t* w, int64_t i) {
  return __ldg(reinterpret_cast<const unsigned long long*>(w) + i);
}
__device__ __forceinline__ Coef3 ldc(const Coef3* p) {
  const double2 lo = __ldg(reinterpret_cast<const double2*>(p));
  const double2 hi = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return Coef3{lo.x, lo.y, hi.x, hi.y};
}
template <typename T>
__device__ __forceinline__ double ldv(const T* p) {  // coherent load
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
  __device__ __forceinline__ void enter(const double4& e, const Coef3&) {
    q1 = e.x;
    q2 = e.y;
    q3 = e.z;
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
  // entry (u'_{j+1}, u'_{j+2}, u'_{j+3}); the ghost coefficients are c_j's
  __device__ __forceinline__ void enter(const double4& e, const Coef3& c) {
    U1 = e.x;
    X1 = c.a1;
    Y21 = c.a2 * e.x;
    Y22 = c.a2 * e.y;
    Y31 = c.a3 * e.x;
    Y32 = c.a3 * e.y;
    Y33 = c.a3 * e.z;
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

// ============================================================ kernel E
// Entry states of every segment of every chain. Forward: M (p_j, p_{j-1},
// p_{j-2}). Adjoint: M' (P1, P2, P3) with P the pending causal-transpose
// contributions of u_j, u_{j-1}, u_{j-2} into the first three ghosts.
// Chains are enumerated in the same order as the sweep kernels.
template <typename T, int DIR, bool TR>
__global__ void __launch_bounds__(128) k_entries(const T* __restrict__ z, StreamArgs a) {
  const int64_t n = DIR == 0 ? a.nx : a.ny;
  const int64_t nlines = DIR == 0 ? a.ny : a.nx;
  const int64_t nh = a.nx * a.ny;
  const int64_t stride = DIR == 0 ? 1 : a.nx;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= planes * nlines) return;
  // plane-fastest: the planes of one line share its closure rows in L2
  const int64_t line = tid / planes;
  const int64_t p = tid - line * planes;
  const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
  const int64_t hb = DIR == 0 ? line * a.nx : line;
  const T* zl = z + p * nh + hb;
  const Coef3* C = a.c3 + hb;
  const int G = a.ghost[lev];
  const double* CL = a.clos + clos_off(a.cls[lev], DIR, TR ? 1 : 0, nh, hb);
  const int64_t s0 = a.seg_off[lev * nlines + line], s1 = a.seg_off[lev * nlines + line + 1];
  double4* E = a.entry + var * a.nsegs;
  for (int64_t s = s0; s < s1; ++s) {
    const int2 sg = __ldg(a.segs + s);
    const int64_t j = sg.x + sg.y - 1;
    double4 e = make_double4(0.0, 0.0, 0.0, 0.0);
    if (j < n - 1 && G > 0) {
      const double z0 = ldv(zl + j * stride);
      const double z1 = sg.y >= 2 ? ldv(zl + (j - 1) * stride) : 0.0;
      const double z2 = sg.y >= 3 ? ldv(zl + (j - 2) * stride) : 0.0;
      const double* M = CL + j * stride * 10;
      double x0 = z0, x1 = z1, x2 = z2;
      if (TR) {
        const Coef3 c = ldc(C + j * stride);
        const Coef3 cm1 = sg.y >= 2 ? ldc(C + (j - 1) * stride) : Coef3{0, 0, 0, 0};
        const Coef3 cm2 = sg.y >= 3 ? ldc(C + (j - 2) * stride) : Coef3{0, 0, 0, 0};
        x0 = fma(c.a1, z0, fma(cm1.a2, z1, cm2.a3 * z2));
        x1 = fma(c.a2, z0, cm1.a3 * z1);
        x2 = c.a3 * z0;
      }
      e.x = fma(__ldg(M + 0), x0, fma(__ldg(M + 1), x1, __ldg(M + 2) * x2));
      e.y = fma(__ldg(M + 3), x0, fma(__ldg(M + 4), x1, __ldg(M + 5) * x2));
      e.z = fma(__ldg(M + 6), x0, fma(__ldg(M + 7), x1, __ldg(M + 8) * x2));
    }
    E[s] = e;
  }
}

// ============================================================ y-sweep
template <typename T, bool TR, int L, int U>
__global__ void __launch_bounds__(128) k_y_pass_a(const T* __restrict__ in, T* __restrict__ out,
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
  const double* PRE[L];
  bool on[L];
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const int64_t p = g * L + l;
    on[l] = p < planes;
    const int64_t pp = on[l] ? p : planes - 1;
    const int64_t lev = a.lev0 + pp % a.nlev;
    src[l] = in + pp * nh + ix;
    dst[l] = out + pp * nh + ix;
    W[l] = a.bits + (lev * nx + ix) * a.words;
    PRE[l] = (TR && a.pre_scale) ? a.pre_scale + lev * nh + ix : nullptr;
  }
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
        id[u] = (TR && IDC) ? __ldg(IDC + k * nx) : 1.0;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          s[l][u] = on[l] ? ldv(src[l] + k * nx) : 0.0;
          if (PRE[l]) s[l][u] *= __ldg(PRE[l] + k * nx);
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
          const double r = st[l].step(c[u], TR ? s[l][u] * id[u] : s[l][u], sea);
          if (on[l]) dst[l][k * nx] = static_cast<T>(r);
        }
      }
    }
  }
}

template <typename T, bool TR, int L, int U>
__global__ void __launch_bounds__(128) k_y_pass_d(T* __restrict__ out, StreamArgs a) {
  const int64_t nx = a.nx, n = a.ny, nh = nx * n;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t groups = (planes + L - 1) / L;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tid >= groups * nx) return;
  const int64_t g = tid / nx, ix = tid - g * nx;
  const Coef3* C = a.c3 + ix;
  const double* IDC = (!TR && a.idc) ? a.idc + ix : nullptr;
  T* dst[L];
  const uint64_t* W[L];
  const double* POST[L];
  const double4* E[L];
  int64_t sidx[L], sfirst[L];
  double4 ent[L];
  bool on[L];
  int nxt[L];
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const int64_t p = g * L + l;
    on[l] = p < planes;
    const int64_t pp = on[l] ? p : planes - 1;
    const int64_t var = pp / a.nlev, lev = a.lev0 + (pp - var * a.nlev);
    dst[l] = out + pp * nh + ix;
    W[l] = a.bits + (lev * nx + ix) * a.words;
    POST[l] = a.post_scale ? a.post_scale + lev * nh + ix : nullptr;
    E[l] = a.entry + var * a.nsegs;
    sfirst[l] = a.seg_off[lev * nx + ix];
    sidx[l] = a.seg_off[lev * nx + ix + 1] - 1;
    ent[l] = sidx[l] >= sfirst[l] ? E[l][sidx[l]] : make_double4(0, 0, 0, 0);
    nxt[l] = 0;
  }
  typename std::conditional<TR, AdjD, FwdD>::type st[L];
  uint64_t wc[L];
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
        id[u] = IDC ? __ldg(IDC + k * nx) : 1.0;
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
          if (sea && !nxt[l]) {  // segment end: enter, prefetch the next entry
            st[l].enter(ent[l], c[u]);
            --sidx[l];
            if (sidx[l] >= sfirst[l]) ent[l] = E[l][sidx[l]];
          }
          double o = st[l].step(c[u], z[l][u]);
          if (IDC) o *= id[u];
          if (POST[l]) o *= __ldg(POST[l] + k * nx);
          if (on[l]) dst[l][k * nx] = static_cast<T>(sea ? o : 0.0);
          nxt[l] = sea;
        }
      }
    }
  }
}

// ============================================================ x-sweep
// Warp-cooperative staging of a [32 chains x 32 elements] tile. Chain c of
// the warp is lane c's (plane, row); element e of its row segment goes to
// tile[c][e] (row pitch 33 elements: conflict-free per-lane row reads).
constexpr int XB = 32;       // elements per batch
constexpr int XP = XB + 1;   // padded pitch

__device__ __forceinline__ void cp_async_elem(void* smem, const void* gmem, int bytes, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int src = pred ? bytes : 0;  // zero-fill when predicated off
  if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// issue the loads of batch [k0, k0+XB) of all 32 chains of this warp;
// lane_row: this lane's row base (nullptr for an inactive chain),
// dummy: any valid global address (source of zero-filled copies)
template <typename T>
__device__ __forceinline__ void x_stage(T* tile, const T* lane_row, const T* dummy, int64_t k0,
                                        int64_t n, int lane) {
#pragma unroll 4
  for (int c = 0; c < 32; ++c) {
    const T* row = reinterpret_cast<const T*>(static_cast<uintptr_t>(__shfl_sync(
        0xffffffffu, static_cast<unsigned long long>(reinterpret_cast<uintptr_t>(lane_row)), c)));
    const int64_t k = k0 + lane;
    const bool ok = row != nullptr && k < n;
    cp_async_elem(tile + c * XP + lane, ok ? row + k : dummy, static_cast<int>(sizeof(T)), ok);
  }
}

template <typename T, bool TR>
__global__ void __launch_bounds__(128) k_x_pass_a(const T* __restrict__ in, T* __restrict__ out,
                                                  StreamArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* const sm = reinterpret_cast<T*>(smraw);
  const int64_t n = a.nx, ny = a.ny, nh = n * ny;
  const int64_t planes = a.nvar * a.nlev;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool on = tid < planes * ny;
  const int64_t t = on ? tid : planes * ny - 1;
  const int64_t iy = t / planes, p = t - iy * planes;
  const int64_t lev = a.lev0 + p % a.nlev;
  const int64_t hb = iy * n;
  const T* src = on ? in + p * nh + hb : nullptr;
  T* dst = out + p * nh + hb;
  const Coef3* C = a.c3 + hb;
  const double* IDC = (TR && a.idc) ? a.idc + hb : nullptr;
  const double* PRE = (TR && a.pre_scale) ? a.pre_scale + lev * nh + hb : nullptr;
  const uint64_t* W = a.bits + (lev * ny + iy) * a.words;
  T* const tiles = sm + wid * 2 * 32 * XP;
  const int64_t nb = (n + XB - 1) / XB;

  typename std::conditional<TR, AdjA, FwdA>::type st;
  x_stage<T>(tiles, src, in, 0, n, lane);
  cp_async_commit();
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t k0 = b * XB;
    T* cur = tiles + (b & 1) * 32 * XP;
    if (b + 1 < nb) x_stage<T>(tiles + ((b + 1) & 1) * 32 * XP, src, in, k0 + XB, n, lane);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    uint64_t wc = ldw(W, k0 >> 6);
    T* row = cur + lane * XP;
#pragma unroll
    for (int u0 = 0; u0 < XB; u0 += 8) {
      Coef3 c[8];
      double id[8], pr[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t k = k0 + u0 + u;
        const int64_t kk = k < n ? k : n - 1;
        c[u] = ldc(C + kk);
        if (IDC) id[u] = __ldg(IDC + kk);
        if (PRE) pr[u] = __ldg(PRE + kk);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t k = k0 + u0 + u;
        if (k < n) {
          const bool sea = (wc >> (k & 63)) & 1ull;
          double w = static_cast<double>(row[u0 + u]);
          if (PRE) w *= pr[u];
          if (IDC) w *= id[u];
          row[u0 + u] = static_cast<T>(st.step(c[u], w, sea));
        }
      }
    }
    __syncwarp();
    // cooperative coalesced store of the tile
#pragma unroll 4
    for (int c = 0; c < 32; ++c) {
      const int64_t tc = blockIdx.x * (int64_t)blockDim.x + wid * 32 + c;
      if (tc >= planes * ny) break;
      T* drow = reinterpret_cast<T*>(static_cast<uintptr_t>(__shfl_sync(
          0xffffffffu, static_cast<unsigned long long>(reinterpret_cast<uintptr_t>(dst)), c)));
      const int64_t k = k0 + lane;
      if (k < n) drow[k] = cur[c * XP + lane];
    }
    __syncwarp();
  }
  cp_async_wait<0>();
}

template <typename T, bool TR>
__global__ void __launch_bounds__(128) k_x_pass_d(T* __restrict__ out, StreamArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* const sm = reinterpret_cast<T*>(smraw);
  const int64_t n = a.nx, ny = a.ny, nh = n * ny;
  const int64_t planes = a.nvar * a.nlev;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool on = tid < planes * ny;
  const int64_t t = on ? tid : planes * ny - 1;
  const int64_t iy = t / planes, p = t - iy * planes;
  const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
  const int64_t hb = iy * n;
  T* dst = on ? out + p * nh + hb : nullptr;
  const Coef3* C = a.c3 + hb;
  const double* IDC = (!TR && a.idc) ? a.idc + hb : nullptr;
  const double* POST = a.post_scale ? a.post_scale + lev * nh + hb : nullptr;
  const uint64_t* W = a.bits + (lev * ny + iy) * a.words;
  const double4* E = a.entry + var * a.nsegs;
  const int64_t sfirst = a.seg_off[lev * ny + iy];
  int64_t sidx = a.seg_off[lev * ny + iy + 1] - 1;
  double4 ent = sidx >= sfirst ? E[sidx] : make_double4(0, 0, 0, 0);
  T* const tiles = sm + wid * 2 * 32 * XP;
  const int64_t nb = (n + XB - 1) / XB;

  typename std::conditional<TR, AdjD, FwdD>::type st;
  int nxt = 0;
  x_stage<T>(tiles + ((nb - 1) & 1) * 32 * XP, dst, out, (nb - 1) * XB, n, lane);
  cp_async_commit();
  for (int64_t b = nb - 1; b >= 0; --b) {
    const int64_t k0 = b * XB;
    T* cur = tiles + (b & 1) * 32 * XP;
    if (b > 0) x_stage<T>(tiles + ((b - 1) & 1) * 32 * XP, dst, out, k0 - XB, n, lane);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    uint64_t wc = ldw(W, k0 >> 6);
    T* row = cur + lane * XP;
#pragma unroll
    for (int u0 = XB - 8; u0 >= 0; u0 -= 8) {
      Coef3 c[8];
      double id[8], po[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t k = k0 + u0 + u;
        const int64_t kk = k < n ? k : n - 1;
        c[u] = ldc(C + kk);
        if (IDC) id[u] = __ldg(IDC + kk);
        if (POST) po[u] = __ldg(POST + kk);
      }
#pragma unroll
      for (int u = 7; u >= 0; --u) {
        const int64_t k = k0 + u0 + u;
        if (k < n) {
          const int sea = static_cast<int>((wc >> (k & 63)) & 1ull);
          if (sea && !nxt) {
            st.enter(ent, c[u]);
            --sidx;
            if (sidx >= sfirst) ent = E[sidx];
          }
          double o = st.step(c[u], static_cast<double>(row[u0 + u]));
          if (IDC) o *= id[u];
          if (POST) o *= po[u];
          row[u0 + u] = static_cast<T>(sea ? o : 0.0);
          nxt = sea;
        }
      }
    }
    __syncwarp();
#pragma unroll 4
    for (int c = 0; c < 32; ++c) {
      T* drow = reinterpret_cast<T*>(static_cast<uintptr_t>(__shfl_sync(
          0xffffffffu, static_cast<unsigned long long>(reinterpret_cast<uintptr_t>(dst)), c)));
      const int64_t k = k0 + lane;
      if (drow && k < n) drow[k] = cur[c * XP + lane];
    }
    __syncwarp();
  }
  cp_async_wait<0>();
}

template <typename T>
int launch_stream_sweep(const T* in, T* out, const StreamArgs& a, cudaStream_t st) {
  const int threads = 128;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t nlines = a.dir == 0 ? a.ny : a.nx;
  const int64_t chains = planes * nlines;
  const int64_t eblocks = (chains + threads - 1) / threads;
  if (a.dir == 1) {
    constexpr int L = 4, U = 4;
    const int64_t total = ((planes + L - 1) / L) * a.nx;
    const int64_t blocks = (total + threads - 1) / threads;
    if (a.transpose) {
      k_y_pass_a<T, true, L, U><<<blocks, threads, 0, st>>>(in, out, a);
      k_entries<T, 1, true><<<eblocks, threads, 0, st>>>(out, a);
      k_y_pass_d<T, true, L, U><<<blocks, threads, 0, st>>>(out, a);
    } else {
      k_y_pass_a<T, false, L, U><<<blocks, threads, 0, st>>>(in, out, a);
      k_entries<T, 1, false><<<eblocks, threads, 0, st>>>(out, a);
      k_y_pass_d<T, false, L, U><<<blocks, threads, 0, st>>>(out, a);
    }
  } else {
    const int64_t blocks = (chains + threads - 1) / threads;
    const int smem = 4 * 2 * 32 * XP * static_cast<int>(sizeof(T));
    static bool attr = false;  // per T instantiation
    if (!attr) {
      cudaFuncSetAttribute(k_x_pass_a<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_x_pass_a<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_x_pass_d<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k_x_pass_d<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    if (a.transpose) {
      k_x_pass_a<T, true><<<blocks, threads, smem, st>>>(in, out, a);
      k_entries<T, 0, true><<<eblocks, threads, 0, st>>>(out, a);
      k_x_pass_d<T, true><<<blocks, threads, smem, st>>>(out, a);
    } else {
      k_x_pass_a<T, false><<<blocks, threads, smem, st>>>(in, out, a);
      k_entries<T, 0, false><<<eblocks, threads, 0, st>>>(out, a);
      k_x_pass_d<T, false><<<blocks, threads, smem, st>>>(out, a);
    }
  }
  return 3;
}

}  // namespace rgfb
