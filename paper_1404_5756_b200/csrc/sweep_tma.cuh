// Shared pieces of the TMA-fed 3rd-RF sweeps: chain states (causal pass A,
// anti-causal pass D, forward and adjoint), mask-bit windows and tile
// layouts. The two-pass kernels that first used them were retired in round 2
// (the checkpointed and single-pass sweeps supersede them); the notes below
// describe the layouts the current kernels still use.
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


// ------------------------------------------------------------- launchers
template <typename T>
inline bool tma_supported(const T* in, const T* out, int64_t nx) {
  return (nx * static_cast<int64_t>(sizeof(T))) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(in) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0;
}

}  // namespace rgfb
