// TMA-fed producer/consumer sweeps for the 3rd-RF (forward G_dir and adjoint
// G_dir^T), used whenever rows are 16 B aligned.
//
// Pass A (ascending) and pass D (descending) are separate kernels; each has
// one producer warp that streams U-element stages of every chain of the CTA
// into an S-deep shared-memory ring with TMA tensor loads (one instruction
// per box; the TMA engine zero-fills out-of-range rows/planes), and consumer
// warps whose lanes each advance one chain.
//
// Segment ends are handled without a separate kernel: pass A writes the raw
// 3-value causal state of every chain at every segment end j (forward:
// p_j, p_{j-1}, p_{j-2}; adjoint: the pending causal-transpose contributions
// into the first three ghosts) to `state[var][segment]`. Pass D keeps the next
// segment's raw state, its right-ghost closure matrix (closures.cuh) and the
// descriptor after it in flight, so entering a segment is a 3x3 product on
// registers (covariance.cpp:271-273 + rf3.hpp:232-261 collapsed, see
// sweep_stream.cuh).
//
// y-sweep (lines = columns): a CTA owns a 32-column tile and NW planes; the
//   field box is [NW planes x U rows x 32 columns], coefficients one
//   [U rows x 32 columns] box shared by all NW planes; lanes = columns, so
//   smem reads are conflict-free and stores are coalesced 256 B st.global.
// x-sweep (lines = rows): a CTA owns one row and 32*NW planes; the field box
//   is [U x-positions x 32*NW planes] with 128 B swizzle (lanes = planes
//   read 16 B chunks without bank conflicts), coefficients a [U] row segment
//   broadcast to every lane; results are written back in place and returned
//   with one TMA tensor store per stage.
#pragma once
#include "async_copy.cuh"
#include "sweep_stream.cuh"
#include "tma.cuh"

namespace rgfb {

// ---------------------------------------------------------------- helpers
// Closure application between pass A and pass D. For every segment (one
// thread per segment, all variables) the right-ghost closure turns the raw
// causal state at the segment end j into the anti-causal entry
// e = (q_{j+1}, q_{j+2}, q_{j+3}), and the entry's contributions are folded
// into the stored pass-A terms at j, j-1, j-2 (inside the segment):
//   forward  (w = beta p):  w_j += a1_j e1 + a2_j e2 + a3_j e3,
//                           w_{j-1} += a2_{j-1} e1 + a3_{j-1} e2,
//                           w_{j-2} += a3_{j-2} e1          (rf3.hpp:255-261)
//   adjoint  (v = beta u):  same pattern with the ghost coefficients c_j
//                           (sources beyond j; rf3.hpp:264-274 gather form).
// Pass D then starts every segment from a zero state, exactly as the
// reference's startup rows do at an extended segment's far end.
template <typename T, int DIR, bool TR>
__global__ void __launch_bounds__(256) k_close(T* __restrict__ z, StreamArgs a) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= a.nsegs) return;
  const int64_t s = __ldg(a.close_order + t);
  const int64_t n = DIR == 0 ? a.nx : a.ny;
  const int64_t nlines = DIR == 0 ? a.ny : a.nx;
  const int64_t nh = a.nx * a.ny;
  const int64_t stride = DIR == 0 ? 1 : a.nx;
  const int64_t lg = __ldg(a.seg_line + s);
  const int64_t lev = lg / nlines, line = lg - lev * nlines;
  if (lev < a.lev0 || lev >= a.lev0 + a.nlev) return;  // level outside this launch
  const int2 sg = __ldg(a.segs + s);
  const int64_t j = sg.x + sg.y - 1;
  const int G = a.ghost[lev];
  if (!(j < n - 1 && G > 0)) return;  // no right ghosts: zero entry
  const int64_t h = DIR == 0 ? line * a.nx + j : j * a.nx + line;
  const double* Mp = a.clos + clos_off(a.cls[lev], DIR, TR ? 1 : 0, nh, h);
  double M[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) M[q] = __ldg(Mp + q);
  const Coef3 cj = ldc(a.c3 + h);
  Coef3 c1 = cj, c2 = cj;  // coefficients feeding w_{j-1}, w_{j-2}
  if (!TR) {
    if (sg.y >= 2) c1 = ldc(a.c3 + h - stride);
    if (sg.y >= 3) c2 = ldc(a.c3 + h - 2 * stride);
  }
  for (int64_t v = 0; v < a.nvar; ++v) {
    const double4 r = a.entry[v * a.nsegs + s];
    const double e1 = fma(M[0], r.x, fma(M[1], r.y, M[2] * r.z));
    const double e2 = fma(M[3], r.x, fma(M[4], r.y, M[5] * r.z));
    const double e3 = fma(M[6], r.x, fma(M[7], r.y, M[8] * r.z));
    T* zl = z + ((v * a.nlev + (lev - a.lev0)) * nh + h);
    *zl = static_cast<T>(static_cast<double>(*zl) +
                         fma(cj.a1, e1, fma(cj.a2, e2, cj.a3 * e3)));
    if (sg.y >= 2)
      zl[-stride] = static_cast<T>(static_cast<double>(zl[-stride]) + fma(c1.a2, e1, c1.a3 * e2));
    if (sg.y >= 3)
      zl[-2 * stride] = static_cast<T>(static_cast<double>(zl[-2 * stride]) + c2.a3 * e1);
  }
}

// Lean pass-D states: the entry is already folded into the stored terms, so
// a segment end is a plain reset.
struct FwdD2 {
  double q1 = 0.0, q2 = 0.0, q3 = 0.0;
  __device__ __forceinline__ void reset() { q1 = q2 = q3 = 0.0; }
  // w = beta p (+ folded entry)
  __device__ __forceinline__ double step(const Coef3& c, double w) {
    const double q = fma(c.a1, q1, fma(c.a2, q2, fma(c.a3, q3, w)));
    q3 = q2;
    q2 = q1;
    q1 = q;
    return q;
  }
};
struct AdjD2 {
  double U1 = 0.0, X1 = 0.0, Y21 = 0.0, Y22 = 0.0, Y31 = 0.0, Y32 = 0.0, Y33 = 0.0;
  __device__ __forceinline__ void reset() { U1 = Y21 = Y22 = Y31 = Y32 = Y33 = 0.0; }
  // v = beta u (+ folded entry); returns beta u'
  __device__ __forceinline__ double step(const Coef3& c, double v) {
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

// raw state written by pass A at a segment end
__device__ __forceinline__ double4 raw_state(const FwdA& s) {
  return make_double4(s.p1, s.p2, s.p3, 0.0);
}
__device__ __forceinline__ double4 raw_state(const AdjA& s) {
  return make_double4(fma(s.x1, s.u1, s.y33 + s.y22), s.y32 + s.y21, s.y31, 0.0);
}

// Lean pass-A states: no per-element land handling. The state is reset at
// each segment start (the reference's zero initial state); values computed on
// land are never stored as results (pass D masks land to exactly 0) and never
// reach a segment because the next segment starts with a reset.
struct FwdA2 {
  double p1 = 0.0, p2 = 0.0, p3 = 0.0;
  __device__ __forceinline__ void reset() { p1 = p2 = p3 = 0.0; }
  __device__ __forceinline__ double step(const Coef3& c, double s) {
    const double t = fma(c.a1, p1, fma(c.a2, p2, fma(c.a3, p3, c.b * s)));
    p3 = p2;
    p2 = p1;
    p1 = t;
    return t;
  }
  __device__ __forceinline__ double4 raw() const { return make_double4(p1, p2, p3, 0.0); }
};
struct AdjA2 {
  double u1 = 0.0, x1 = 0.0, y21 = 0.0, y22 = 0.0, y31 = 0.0, y32 = 0.0, y33 = 0.0;
  __device__ __forceinline__ void reset() { u1 = x1 = y21 = y22 = y31 = y32 = y33 = 0.0; }
  __device__ __forceinline__ double step(const Coef3& c, double w) {
    const double u = fma(x1, u1, (w + y33) + y22);
    y33 = y32;
    y32 = y31;
    y31 = c.a3 * u;
    y22 = y21;
    y21 = c.a2 * u;
    x1 = c.a1;
    u1 = u;
    return u;
  }
  // pending causal-transpose contributions into the first three ghosts
  __device__ __forceinline__ double4 raw() const {
    return make_double4(fma(x1, u1, y33 + y22), y32 + y21, y31, 0.0);
  }
};

// One-word-lookahead mask window, advanced once per stage. Stages never
// straddle a 64-bit word (U divides 64 and stages start at multiples of U).
// Two words of lookahead: `nxt` (the word after `cur` in pass order) arrived
// a word ago and `nn` (the one after it) is in flight, so neither the stage
// bits nor the after-stage bit ever wait on a load issued at this word
// change (a select on a fresh load stalled the 1st-RF passes ~25%).
struct StageBits {
  int64_t wi = -1;
  uint64_t cur = 0, nxt = 0, nn = 0;
  // word i of the line at W[i * stride]
  __device__ __forceinline__ void seek(const uint64_t* W, int64_t k, int64_t words, bool desc,
                                       int64_t stride = 1) {
    const int64_t w = k >> 6;
    if (w == wi) return;
    const int64_t step = desc ? -1 : 1;
    const int64_t w1 = w + step, w2 = w + 2 * step;
    if (wi >= 0 && w == wi + step) {
      cur = nxt;
      nxt = (w1 >= 0 && w1 < words) ? nn : 0ull;  // nn was loaded a word ago
    } else {  // first word of the pass
      cur = ldw(W, w * stride);
      nxt = (w1 >= 0 && w1 < words) ? ldw(W, w1 * stride) : 0ull;
    }
    nn = ldw(W, (w2 < 0 ? 0 : (w2 >= words ? words - 1 : w2)) * stride);  // masked at shift
    wi = w;
  }
  template <int U>
  __device__ __forceinline__ uint32_t stage(int64_t k0) const {
    return static_cast<uint32_t>((cur >> (k0 & 63)) & ((1ull << U) - 1ull));
  }
  // sea(k0 + U) for an ascending pass (first bit of the following stage)
  template <int U>
  __device__ __forceinline__ uint32_t after(int64_t k0) const {
    const int64_t kb = k0 + U;
    return (kb & 63) == 0 ? static_cast<uint32_t>(nxt & 1ull)
                          : static_cast<uint32_t>((cur >> (kb & 63)) & 1ull);
  }
};

// ================================================================ y-sweep
template <typename T, int NW, int U, bool FOLD>
struct YT {
  static constexpr size_t field = size_t(NW) * U * 32 * sizeof(T);
  static constexpr size_t coef = size_t(U) * 32 * sizeof(Coef3);
  static constexpr size_t idc = size_t(U) * 32 * sizeof(double);
  static constexpr size_t clos = FOLD ? size_t(U) * 32 * 10 * sizeof(double) : 0;
  static constexpr size_t bytes = field + coef + idc + clos;
};

// FOLD (pass A only, one closure class): the right-ghost closure rows are
// staged with the coefficients, and each segment end's entry is folded into
// the stored terms of rows j, j-1, j-2 on the fly (a 2-row store delay line
// keeps j-1 and j-2 in registers), so no raw-state buffer or closure pass.
template <typename T, bool TR, bool PD, bool IDC, bool VAR, bool FOLD, int NW, int U, int S>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    k_ytma(T* __restrict__ out, StreamArgs a, const __grid_constant__ CUtensorMap tm_field,
           const __grid_constant__ CUtensorMap tm_coef, const __grid_constant__ CUtensorMap tm_idc,
           const __grid_constant__ CUtensorMap tm_clos) {
  using L = YT<T, NW, U, FOLD>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 1024 B alignment by pointer arithmetic (keeps the shared address space)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * L::bytes);
  uint64_t* empty = full + S;

  const int64_t nx = a.nx, ny = a.ny, nh = nx * ny;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t PB = (planes + NW - 1) / NW;
  const int64_t tile = blockIdx.x / PB;
  const int64_t p0 = (blockIdx.x - tile * PB) * NW;
  const int64_t ix0 = tile * 32;
  const int ncol = static_cast<int>(nx - ix0 < 32 ? nx - ix0 : 32);
  const int nwp = static_cast<int>(planes - p0 < NW ? planes - p0 : NW);
  constexpr bool need_idc = IDC;  // inv_dc table staged (fwd pass D / adjoint pass A)
  const int64_t nst = (ny + U - 1) / U;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwp);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto lo_of = [&](int64_t i) -> int64_t { return (PD ? nst - 1 - i : i) * U; };

  if (warp == NW) {  // producer
    if (lane == 0) {
      const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
      tma_prefetch_desc(&tm_field);
      tma_prefetch_desc(&tm_coef);
      if (need_idc) tma_prefetch_desc(&tm_idc);
      const uint32_t total =
          static_cast<uint32_t>(L::field + L::coef + (need_idc ? L::idc : 0) + L::clos);
      for (int64_t i = 0; i < nst; ++i) {
        const int s = static_cast<int>(i % S);
        const int64_t m = i / S;
        if (m > 0) mbar_wait(&empty[s], static_cast<uint32_t>((m - 1) & 1));
        const int lo = static_cast<int>(lo_of(i));
        unsigned char* base = smem + s * L::bytes;
        mbar_arrive_expect_tx(&full[s], total);
        tma_load_3d(base, &tm_field, static_cast<int>(ix0), lo, static_cast<int>(p0), &full[s],
                    pol_stream);
        tma_load_2d(base + L::field, &tm_coef, static_cast<int>(4 * ix0), lo, &full[s], pol_keep);
        if (need_idc)
          tma_load_2d(base + L::field + L::coef, &tm_idc, static_cast<int>(ix0), lo, &full[s],
                      pol_keep);
        if constexpr (FOLD)
          tma_load_3d(base + L::field + L::coef + L::idc, &tm_clos, 0, static_cast<int>(ix0), lo,
                      &full[s], pol_keep);
      }
    }
    return;
  }
  if (warp >= nwp) return;

  // consumer: chain (plane p0+warp, column ix0+lane)
  const int64_t p = p0 + warp;
  const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
  const bool act = lane < ncol;
  const int64_t ix = ix0 + (act ? lane : 0);
  T* dst = out + p * nh + ix;
  const uint64_t* W = a.bits + (lev * nx + ix) * a.words;
  const double* PRE = (VAR && !PD && TR) ? a.pre_scale + lev * nh + ix : nullptr;
  const double* POST = (VAR && PD) ? a.post_scale + lev * nh + ix : nullptr;
  double4* RAW = a.entry + var * a.nsegs;
  const int64_t s0 = a.seg_off[lev * nx + ix], s1 = a.seg_off[lev * nx + ix + 1];
  StageBits sbw;
  typename std::conditional<PD, typename std::conditional<TR, AdjD2, FwdD2>::type,
                            typename std::conditional<TR, AdjA2, FwdA2>::type>::type st;
  int64_t sA = s0;      // pass A: next segment index to be closed
  uint32_t carry = 0;   // A: sea(lo-1); D: sea(lo+U)
  (void)s1;
  // FOLD: stored terms of rows k-1, k-2 (not yet written), the coefficients
  // feeding their corrections, and the current segment's length so far
  double d1 = 0.0, d2 = 0.0, pa2 = 0.0, pa3 = 0.0, ppa3 = 0.0;
  int seglen = 0;

  for (int64_t i = 0; i < nst; ++i) {
    const int s = static_cast<int>(i % S);
    const int64_t lo = lo_of(i);
    sbw.seek(W, lo, a.words, PD);
    const uint32_t sb = sbw.stage<U>(lo);
    mbar_wait(&full[s], static_cast<uint32_t>((i / S) & 1));
    const unsigned char* base = smem + s * L::bytes;
    const T* fld = reinterpret_cast<const T*>(base) + warp * U * 32 + lane;
    const Coef3* cf = reinterpret_cast<const Coef3*>(base + L::field) + lane;
    const double* id = reinterpret_cast<const double*>(base + L::field + L::coef) + lane;
    T* drow = dst + lo * nx;
    const int rvalid = act ? static_cast<int>(ny - lo < U ? ny - lo : U) : 0;
    if constexpr (!PD && FOLD) {
      const uint32_t starts = sb & ~((sb << 1) | carry);
      const uint32_t ends = sb & ~((sb >> 1) | (sbw.after<U>(lo) << (U - 1)));
      const double* cm = reinterpret_cast<const double*>(base + L::field + L::coef + L::idc) +
                         lane * 10;
#pragma unroll
      for (int r = 0; r < U; ++r) {
        const int64_t k = lo + r;
        if ((starts >> r) & 1u) {
          st.reset();
          seglen = 0;
        }
        ++seglen;
        double w = static_cast<double>(fld[r * 32]);
        if (TR) {
          if constexpr (VAR) w *= __ldg(PRE + k * nx);
          if constexpr (IDC) w *= id[r * 32];
        }
        const Coef3 c = cf[r * 32];
        double res = c.b * st.step(c, w);  // stored term beta*p / beta*u
        if (((ends >> r) & 1u) && k < ny - 1) {  // fold the right-ghost entry
          const double4 rw = st.raw();
          const double* M = cm + r * 320;
          const double e1 = fma(M[0], rw.x, fma(M[1], rw.y, M[2] * rw.z));
          const double e2 = fma(M[3], rw.x, fma(M[4], rw.y, M[5] * rw.z));
          const double e3 = fma(M[6], rw.x, fma(M[7], rw.y, M[8] * rw.z));
          res += fma(c.a1, e1, fma(c.a2, e2, c.a3 * e3));
          if (TR) {  // sources beyond j carry the ghost (= c_j) coefficients
            if (seglen >= 2) d1 += fma(c.a2, e1, c.a3 * e2);
            if (seglen >= 3) d2 += c.a3 * e1;
          } else {
            if (seglen >= 2) d1 += fma(pa2, e1, pa3 * e2);
            if (seglen >= 3) d2 += ppa3 * e1;
          }
        }
        if (act && k >= 2 && k - 2 < ny) __stcs(dst + (k - 2) * nx, static_cast<T>(d2));
        d2 = d1;
        d1 = res;
        ppa3 = pa3;
        pa2 = c.a2;
        pa3 = c.a3;
      }
      carry = (sb >> (U - 1)) & 1u;
    } else if constexpr (!PD) {
      const uint32_t starts = sb & ~((sb << 1) | carry);
      const uint32_t ends = sb & ~((sb >> 1) | (sbw.after<U>(lo) << (U - 1)));
#pragma unroll
      for (int r = 0; r < U; ++r) {
        if ((starts >> r) & 1u) st.reset();
        double w = static_cast<double>(fld[r * 32]);
        if (TR) {
          if constexpr (VAR) w *= __ldg(PRE + (lo + r) * nx);
          if constexpr (IDC) w *= id[r * 32];
        }
        const Coef3 c = cf[r * 32];
        const double res = c.b * st.step(c, w);  // stored term beta*p / beta*u
        if (r < rvalid) __stcs(drow + r * static_cast<int>(nx), static_cast<T>(res));
        if ((ends >> r) & 1u) {
          if (act) RAW[sA] = st.raw();
          ++sA;
        }
      }
      carry = (sb >> (U - 1)) & 1u;
    } else {
      const uint32_t events = sb & ~((sb >> 1) | (carry << (U - 1)));
#pragma unroll
      for (int r = U - 1; r >= 0; --r) {
        const Coef3 c = cf[r * 32];
        if ((events >> r) & 1u) st.reset();
        double o = st.step(c, static_cast<double>(fld[r * 32]));
        if constexpr (!TR && IDC) o *= id[r * 32];
        if constexpr (VAR) o *= __ldg(POST + (lo + r) * nx);
        if (r < rvalid)
          __stcs(drow + r * static_cast<int>(nx), static_cast<T>(((sb >> r) & 1u) ? o : 0.0));
      }
      carry = sb & 1u;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if constexpr (!PD && FOLD) {  // flush the delay line: rows kl-1, kl
    const int64_t kl = nst * U - 1;
    if (act && kl - 1 < ny) __stcs(dst + (kl - 1) * nx, static_cast<T>(d2));
    if (act && kl < ny) __stcs(dst + kl * nx, static_cast<T>(d1));
  }
}

constexpr int kYtNW = 16, kYtU = 8, kYtS = 4, kYtSFold = 3;

// ================================================================ x-sweep
// one row, up to 32*NW planes per CTA; U*sizeof(T) = 128 B (swizzle atom)
template <typename T, int NW, bool FOLD>
struct XT {
  static constexpr int U = 128 / int(sizeof(T));
  static constexpr size_t field = size_t(NW) * 32 * 128;
  static constexpr size_t coef = size_t(U) * sizeof(Coef3);
  static constexpr size_t idc = size_t(U) * sizeof(double);
  static constexpr size_t clos = FOLD ? size_t(U) * 10 * sizeof(double) : 0;
  static constexpr size_t bytes = (field + coef + idc + clos + 1023) / 1024 * 1024;
};

// byte offset of element u of plane-row r in a 128B-swizzled [rows][128 B] tile
__device__ __forceinline__ uint32_t swz128(int r, uint32_t byte_in_row) {
  return static_cast<uint32_t>(r) * 128u + ((((byte_in_row >> 4) ^ (r & 7)) << 4) | (byte_in_row & 15u));
}

template <typename T, bool TR, bool PD, bool IDC, bool VAR, bool FOLD, int NW, int S>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    k_xtma(T* __restrict__ out, StreamArgs a, const __grid_constant__ CUtensorMap tm_in,
           const __grid_constant__ CUtensorMap tm_out, const __grid_constant__ CUtensorMap tm_coef,
           const __grid_constant__ CUtensorMap tm_idc, const __grid_constant__ CUtensorMap tm_clos) {
  using L = XT<T, NW, FOLD>;
  constexpr int U = L::U;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 1024 B alignment by pointer arithmetic (keeps the shared address space)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * L::bytes);
  uint64_t* empty = full + S;

  const int64_t n = a.nx, ny = a.ny, nh = n * ny;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t PB = (planes + 32 * NW - 1) / (32 * NW);
  const int64_t iy = blockIdx.x / PB;
  const int64_t p0 = (blockIdx.x - iy * PB) * 32 * NW;
  const int npl = static_cast<int>(planes - p0 < 32 * NW ? planes - p0 : 32 * NW);
  constexpr bool need_idc = IDC;  // inv_dc table staged (fwd pass D / adjoint pass A)
  const int64_t nst = (n + U - 1) / U;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto k0_of = [&](int64_t i) -> int64_t { return (PD ? nst - 1 - i : i) * U; };

  if (warp == NW) {  // producer
    if (lane == 0) {
      const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
      tma_prefetch_desc(&tm_in);
      tma_prefetch_desc(&tm_coef);
      const uint32_t total =
          static_cast<uint32_t>(L::field + L::coef + (need_idc ? L::idc : 0) + L::clos);
      for (int64_t i = 0; i < nst; ++i) {
        const int s = static_cast<int>(i % S);
        const int64_t m = i / S;
        if (m > 0) mbar_wait(&empty[s], static_cast<uint32_t>((m - 1) & 1));
        const int k0 = static_cast<int>(k0_of(i));
        unsigned char* base = smem + s * L::bytes;
        mbar_arrive_expect_tx(&full[s], total);
        tma_load_3d(base, &tm_in, k0, static_cast<int>(iy), static_cast<int>(p0), &full[s],
                    pol_stream);
        tma_load_2d(base + L::field, &tm_coef, 4 * k0, static_cast<int>(iy), &full[s], pol_keep);
        if (need_idc)
          tma_load_2d(base + L::field + L::coef, &tm_idc, k0, static_cast<int>(iy), &full[s],
                      pol_keep);
        if constexpr (FOLD)
          tma_load_3d(base + L::field + L::coef + L::idc, &tm_clos, 0, k0, static_cast<int>(iy),
                      &full[s], pol_keep);
      }
    }
    return;
  }

  // consumers: lane = plane p0 + 32*warp + lane of row iy
  const int pr = warp * 32 + lane;  // row of the smem tile
  const bool act = pr < npl;
  const int64_t p = p0 + (act ? pr : 0);
  const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
  const uint64_t* W = a.bits + (lev * ny + iy) * a.words;
  const double* PRE = (VAR && !PD && TR) ? a.pre_scale + lev * nh + iy * n : nullptr;
  const double* POST = (VAR && PD) ? a.post_scale + lev * nh + iy * n : nullptr;
  double4* RAW = a.entry + var * a.nsegs;
  const int64_t s0 = a.seg_off[lev * ny + iy], s1 = a.seg_off[lev * ny + iy + 1];
  StageBits sbw;
  typename std::conditional<PD, typename std::conditional<TR, AdjD2, FwdD2>::type,
                            typename std::conditional<TR, AdjA2, FwdA2>::type>::type st;
  int64_t sA = s0;
  uint32_t carry = 0;  // A: sea(k0-1); D: sea(k0+U)
  (void)s1;
  // FOLD: stored terms of elements k-1, k-2 (not yet written back), the
  // coefficients feeding their corrections, current segment length
  double d1 = 0.0, d2 = 0.0, pa2 = 0.0, pa3 = 0.0, ppa3 = 0.0;
  int seglen = 0;
  constexpr int ESZ = static_cast<int>(sizeof(T));
  constexpr int EPCX = 16 / ESZ;
  auto elem = [&](unsigned char* tile_row, int u) -> T* {  // swizzled element address
    return reinterpret_cast<T*>(tile_row + (((u / EPCX) ^ (pr & 7)) << 4) + (u % EPCX) * ESZ);
  };

  for (int64_t i = 0; i < nst; ++i) {
    const int s = static_cast<int>(i % S);
    const int64_t k0 = k0_of(i);
    sbw.seek(W, k0, a.words, PD);
    const uint32_t sb = sbw.stage<U>(k0);
    mbar_wait(&full[s], static_cast<uint32_t>((i / S) & 1));
    unsigned char* base = smem + s * L::bytes;
    const Coef3* cf = reinterpret_cast<const Coef3*>(base + L::field);
    const double* id = reinterpret_cast<const double*>(base + L::field + L::coef);
    // this lane's U elements (128 B), 16 B chunk at a time through the swizzle
    constexpr int EPC = 16 / int(sizeof(T));  // elements per 16 B chunk
    unsigned char* rowp = base + pr * 128;
    const int sw = pr & 7;
    if constexpr (!PD && FOLD) {
      const uint32_t starts = sb & ~((sb << 1) | carry);
      const uint32_t ends = sb & ~((sb >> 1) | (sbw.after<U>(k0) << (U - 1)));
      const double* cm = reinterpret_cast<const double*>(base + L::field + L::coef + L::idc);
      unsigned char* prow = smem + ((i + S - 1) % S) * L::bytes + pr * 128;  // previous tile
#pragma unroll 4
      for (int u = 0; u < U; ++u) {
        const int64_t k = k0 + u;
        if ((starts >> u) & 1u) {
          st.reset();
          seglen = 0;
        }
        ++seglen;
        double w = static_cast<double>(*elem(rowp, u));
        if (TR) {
          if constexpr (VAR) w *= __ldg(PRE + k);
          if constexpr (IDC) w *= id[u];
        }
        const Coef3 c = cf[u];
        double res = c.b * st.step(c, w);
        if (((ends >> u) & 1u) && k < n - 1) {  // fold the right-ghost entry
          const double4 rw = st.raw();
          const double* M = cm + u * 10;
          const double e1 = fma(M[0], rw.x, fma(M[1], rw.y, M[2] * rw.z));
          const double e2 = fma(M[3], rw.x, fma(M[4], rw.y, M[5] * rw.z));
          const double e3 = fma(M[6], rw.x, fma(M[7], rw.y, M[8] * rw.z));
          res += fma(c.a1, e1, fma(c.a2, e2, c.a3 * e3));
          if (TR) {
            if (seglen >= 2) d1 += fma(c.a2, e1, c.a3 * e2);
            if (seglen >= 3) d2 += c.a3 * e1;
          } else {
            if (seglen >= 2) d1 += fma(pa2, e1, pa3 * e2);
            if (seglen >= 3) d2 += ppa3 * e1;
          }
        }
        if (k >= 2) *(u >= 2 ? elem(rowp, u - 2) : elem(prow, U + u - 2)) = static_cast<T>(d2);
        d2 = d1;
        d1 = res;
        ppa3 = pa3;
        pa2 = c.a2;
        pa3 = c.a3;
      }
      carry = (sb >> (U - 1)) & 1u;
    } else if constexpr (!PD) {
      const uint32_t starts = sb & ~((sb << 1) | carry);
      const uint32_t ends = sb & ~((sb >> 1) | (sbw.after<U>(k0) << (U - 1)));
#pragma unroll 1
      for (int q = 0; q < U / EPC; ++q) {
        void* cp = rowp + ((q ^ sw) << 4);
        double v[EPC];
        if constexpr (sizeof(T) == 8) {
          const double2 t = *reinterpret_cast<const double2*>(cp);
          v[0] = t.x;
          v[1] = t.y;
        } else {
          const float4 t = *reinterpret_cast<const float4*>(cp);
          v[0] = t.x;
          v[1] = t.y;
          v[2] = t.z;
          v[3] = t.w;
        }
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          const int u = q * EPC + e;
          if ((starts >> u) & 1u) st.reset();
          double w = v[e];
          if (TR) {
            if constexpr (VAR) w *= __ldg(PRE + k0 + u);
            if constexpr (IDC) w *= id[u];
          }
          const Coef3 c = cf[u];
          v[e] = c.b * st.step(c, w);  // stored term beta*p / beta*u
          if ((ends >> u) & 1u) {
            if (act) RAW[sA] = st.raw();
            ++sA;
          }
        }
        if constexpr (sizeof(T) == 8) {
          *reinterpret_cast<double2*>(cp) = make_double2(v[0], v[1]);
        } else {
          *reinterpret_cast<float4*>(cp) =
              make_float4(static_cast<float>(v[0]), static_cast<float>(v[1]),
                          static_cast<float>(v[2]), static_cast<float>(v[3]));
        }
      }
      carry = (sb >> (U - 1)) & 1u;
    } else {
      const uint32_t events = sb & ~((sb >> 1) | (carry << (U - 1)));
#pragma unroll 1
      for (int q = U / EPC - 1; q >= 0; --q) {
        void* cp = rowp + ((q ^ sw) << 4);
        double v[EPC];
        if constexpr (sizeof(T) == 8) {
          const double2 t = *reinterpret_cast<const double2*>(cp);
          v[0] = t.x;
          v[1] = t.y;
        } else {
          const float4 t = *reinterpret_cast<const float4*>(cp);
          v[0] = t.x;
          v[1] = t.y;
          v[2] = t.z;
          v[3] = t.w;
        }
#pragma unroll
        for (int e = EPC - 1; e >= 0; --e) {
          const int u = q * EPC + e;
          const Coef3 c = cf[u];
          if ((events >> u) & 1u) st.reset();
          double o = st.step(c, v[e]);
          if constexpr (!TR && IDC) o *= id[u];
          if constexpr (VAR) o *= __ldg(POST + k0 + u);
          v[e] = ((sb >> u) & 1u) ? o : 0.0;
        }
        if constexpr (sizeof(T) == 8) {
          *reinterpret_cast<double2*>(cp) = make_double2(v[0], v[1]);
        } else {
          *reinterpret_cast<float4*>(cp) =
              make_float4(static_cast<float>(v[0]), static_cast<float>(v[1]),
                          static_cast<float>(v[2]), static_cast<float>(v[3]));
        }
      }
      carry = sb & 1u;
    }
    // all consumers' results in smem -> one TMA store of the box
    fence_proxy_async_smem();
    asm volatile("bar.sync 1, %0;\n" ::"r"(32 * NW) : "memory");
    if constexpr (!PD && FOLD) {
      // the last two elements of a tile are final only after the next
      // stage's first two steps: store the previous stage's tile
      if (threadIdx.x == 0 && i > 0) {
        tma_store_3d(&tm_out, static_cast<int>(k0 - U), static_cast<int>(iy),
                     static_cast<int>(p0), smem + ((i - 1) % S) * L::bytes, l2_evict_first());
        bulk_commit();
        asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
        if (i > 1) mbar_arrive(&empty[(i - 2) % S]);
      }
    } else {
      if (threadIdx.x == 0) {
        tma_store_3d(&tm_out, static_cast<int>(k0), static_cast<int>(iy), static_cast<int>(p0),
                     base, l2_evict_first());
        bulk_commit();
        // the stage is free once the store has read it (the previous stage's
        // store is older; wait for it before releasing that stage)
        asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
        if (i > 0) mbar_arrive(&empty[(i - 1) % S]);
      }
    }
  }
  if constexpr (!PD && FOLD) {  // flush the delay line into the last tile and store it
    unsigned char* lrow = smem + ((nst - 1) % S) * L::bytes + pr * 128;
    *elem(lrow, U - 2) = static_cast<T>(d2);
    *elem(lrow, U - 1) = static_cast<T>(d1);
    fence_proxy_async_smem();
    asm volatile("bar.sync 1, %0;\n" ::"r"(32 * NW) : "memory");
    if (threadIdx.x == 0)
      tma_store_3d(&tm_out, static_cast<int>((nst - 1) * U), static_cast<int>(iy),
                   static_cast<int>(p0), smem + ((nst - 1) % S) * L::bytes, l2_evict_first());
    if (threadIdx.x == 0) bulk_commit();
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

constexpr int kXtNW = 4, kXtS = 4;

// ------------------------------------------------------------- launchers
template <typename T>
inline bool tma_supported(const T* in, const T* out, int64_t nx) {
  return (nx * static_cast<int64_t>(sizeof(T))) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(in) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0;
}

template <typename T, bool TR, bool PD, bool IDC, bool VAR, bool FOLD>
void launch_ytma_k(const T* in, T* out, const StreamArgs& a, cudaStream_t st) {
  constexpr int NW = kYtNW, U = kYtU, S = FOLD ? kYtSFold : kYtS;
  const size_t smem = S * YT<T, NW, U, FOLD>::bytes + 2 * S * sizeof(uint64_t) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ytma<T, TR, PD, IDC, VAR, FOLD, NW, U, S>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  const int64_t planes = a.nvar * a.nlev;
  const uint64_t sz = sizeof(T);
  const uint64_t fd[3] = {uint64_t(a.nx), uint64_t(a.ny), uint64_t(planes)};
  const uint64_t fs[2] = {uint64_t(a.nx) * sz, uint64_t(a.nx * a.ny) * sz};
  const uint32_t fb[3] = {32, U, NW};
  const CUtensorMap tf = make_tmap(PD ? static_cast<const void*>(out) : in, tma_dtype<T>(), 3, fd,
                                   fs, fb, CU_TENSOR_MAP_SWIZZLE_NONE);
  const uint64_t cd[2] = {uint64_t(4 * a.nx), uint64_t(a.ny)};
  const uint64_t cs[1] = {uint64_t(4 * a.nx) * 8};
  const uint32_t cb[2] = {128, U};
  const CUtensorMap tc = make_tmap(a.c3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, cd, cs, cb,
                                   CU_TENSOR_MAP_SWIZZLE_NONE);
  const uint64_t id[2] = {uint64_t(a.nx), uint64_t(a.ny)};
  const uint64_t is[1] = {uint64_t(a.nx) * 8};
  const uint32_t ib[2] = {32, U};
  const CUtensorMap ti = a.idc ? make_tmap(a.idc, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, id, is, ib,
                                           CU_TENSOR_MAP_SWIZZLE_NONE)
                               : tc;
  CUtensorMap tcl = tc;
  if (FOLD) {  // closure rows of class 0, this direction/part: [ny][nx][10]
    const uint64_t md[3] = {10, uint64_t(a.nx), uint64_t(a.ny)};
    const uint64_t ms[2] = {80, uint64_t(a.nx) * 80};
    const uint32_t mb[3] = {10, 32, U};
    tcl = make_tmap(a.clos + clos_off(0, 1, TR ? 1 : 0, a.nx * a.ny, 0),
                    CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, md, ms, mb, CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  const int64_t blocks = ((a.nx + 31) / 32) * ((planes + NW - 1) / NW);
  k_ytma<T, TR, PD, IDC, VAR, FOLD, NW, U, S><<<blocks, 32 * (NW + 1), smem, st>>>(out, a, tf, tc,
                                                                                  ti, tcl);
}

template <typename T, bool TR, bool PD, bool IDC, bool VAR, bool FOLD>
void launch_xtma_k(const T* in, T* out, const StreamArgs& a, cudaStream_t st) {
  constexpr int NW = kXtNW, S = kXtS;
  using L = XT<T, NW, FOLD>;
  const size_t smem = S * L::bytes + 2 * S * sizeof(uint64_t) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_xtma<T, TR, PD, IDC, VAR, FOLD, NW, S>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  const int64_t planes = a.nvar * a.nlev;
  const uint64_t sz = sizeof(T);
  const uint64_t fd[3] = {uint64_t(a.nx), uint64_t(a.ny), uint64_t(planes)};
  const uint64_t fs[2] = {uint64_t(a.nx) * sz, uint64_t(a.nx * a.ny) * sz};
  const uint32_t fb[3] = {uint32_t(L::U), 1, uint32_t(32 * NW)};
  // box rows are exactly one 128 B line: no L2 over-fetch
  const CUtensorMap tin = make_tmap(PD ? static_cast<const void*>(out) : in, tma_dtype<T>(), 3,
                                    fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
  const CUtensorMap tout = make_tmap(out, tma_dtype<T>(), 3, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_128B,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
  const uint64_t cd[2] = {uint64_t(4 * a.nx), uint64_t(a.ny)};
  const uint64_t cs[1] = {uint64_t(4 * a.nx) * 8};
  const uint32_t cb[2] = {uint32_t(4 * L::U), 1};
  const CUtensorMap tc = make_tmap(a.c3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, cd, cs, cb,
                                   CU_TENSOR_MAP_SWIZZLE_NONE);
  const uint64_t id[2] = {uint64_t(a.nx), uint64_t(a.ny)};
  const uint64_t is[1] = {uint64_t(a.nx) * 8};
  const uint32_t ib[2] = {uint32_t(L::U), 1};
  const CUtensorMap ti = a.idc ? make_tmap(a.idc, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, id, is, ib,
                                           CU_TENSOR_MAP_SWIZZLE_NONE)
                               : tc;
  CUtensorMap tcl = tc;
  if (FOLD) {
    const uint64_t md[3] = {10, uint64_t(a.nx), uint64_t(a.ny)};
    const uint64_t ms[2] = {80, uint64_t(a.nx) * 80};
    const uint32_t mb[3] = {10, uint32_t(L::U), 1};
    tcl = make_tmap(a.clos + clos_off(0, 0, TR ? 1 : 0, a.nx * a.ny, 0),
                    CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, md, ms, mb, CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  const int64_t PB = (planes + 32 * NW - 1) / (32 * NW);
  const int64_t blocks = a.ny * PB;
  k_xtma<T, TR, PD, IDC, VAR, FOLD, NW, S><<<blocks, 32 * (NW + 1), smem, st>>>(out, a, tin, tout,
                                                                                tc, ti, tcl);
}

// runtime flags -> template flags
template <typename T, bool TR, bool PD, bool FOLD>
void launch_ytma(const T* in, T* out, const StreamArgs& a, cudaStream_t st) {
  const bool idc = a.idc != nullptr && (PD ? !TR : TR);
  const bool var = PD ? a.post_scale != nullptr : (TR && a.pre_scale != nullptr);
  if (idc) {
    if (var) launch_ytma_k<T, TR, PD, true, true, FOLD>(in, out, a, st);
    else launch_ytma_k<T, TR, PD, true, false, FOLD>(in, out, a, st);
  } else {
    if (var) launch_ytma_k<T, TR, PD, false, true, FOLD>(in, out, a, st);
    else launch_ytma_k<T, TR, PD, false, false, FOLD>(in, out, a, st);
  }
}
template <typename T, bool TR, bool PD, bool FOLD>
void launch_xtma(const T* in, T* out, const StreamArgs& a, cudaStream_t st) {
  const bool idc = a.idc != nullptr && (PD ? !TR : TR);
  const bool var = PD ? a.post_scale != nullptr : (TR && a.pre_scale != nullptr);
  if (idc) {
    if (var) launch_xtma_k<T, TR, PD, true, true, FOLD>(in, out, a, st);
    else launch_xtma_k<T, TR, PD, true, false, FOLD>(in, out, a, st);
  } else {
    if (var) launch_xtma_k<T, TR, PD, false, true, FOLD>(in, out, a, st);
    else launch_xtma_k<T, TR, PD, false, false, FOLD>(in, out, a, st);
  }
}

template <typename T>
int launch_tma_sweep(const T* in, T* out, const StreamArgs& a, cudaStream_t st) {
  const int64_t cblocks = (a.nsegs + 255) / 256;
  if (a.nclass == 1) {  // fused closure (single ghost-width class)
    if (a.dir == 1) {
      if (a.transpose) {
        launch_ytma<T, true, false, true>(in, out, a, st);
        launch_ytma<T, true, true, false>(out, out, a, st);
      } else {
        launch_ytma<T, false, false, true>(in, out, a, st);
        launch_ytma<T, false, true, false>(out, out, a, st);
      }
    } else {
      if (a.transpose) {
        launch_xtma<T, true, false, true>(in, out, a, st);
        launch_xtma<T, true, true, false>(out, out, a, st);
      } else {
        launch_xtma<T, false, false, true>(in, out, a, st);
        launch_xtma<T, false, true, false>(out, out, a, st);
      }
    }
    return 2;
  }
  if (a.dir == 1) {
    if (a.transpose) {
      launch_ytma<T, true, false, false>(in, out, a, st);
      k_close<T, 1, true><<<cblocks, 256, 0, st>>>(out, a);
      launch_ytma<T, true, true, false>(out, out, a, st);
    } else {
      launch_ytma<T, false, false, false>(in, out, a, st);
      k_close<T, 1, false><<<cblocks, 256, 0, st>>>(out, a);
      launch_ytma<T, false, true, false>(out, out, a, st);
    }
  } else {
    if (a.transpose) {
      launch_xtma<T, true, false, false>(in, out, a, st);
      k_close<T, 0, true><<<cblocks, 256, 0, st>>>(out, a);
      launch_xtma<T, true, true, false>(out, out, a, st);
    } else {
      launch_xtma<T, false, false, false>(in, out, a, st);
      k_close<T, 0, false><<<cblocks, 256, 0, st>>>(out, a);
      launch_xtma<T, false, true, false>(out, out, a, st);
    }
  }
  return 3;
}

}  // namespace rgfb
