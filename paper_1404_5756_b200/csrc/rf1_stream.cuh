// Streaming 1st-RF (K iterations, live ghosts on both sides).
//
// Reference (rf1.hpp:20-63, 113-137; covariance.cpp:283-286, 319-322,
// 334-339): each sea segment is extended by G imaginary points on each side
// that meets land (zero input, coefficients replicated from the segment's end
// points), then K times {forward, backward} run in place over the extended
// segment (the adjoint: K times {backward-transpose, forward-transpose}). The
// ghost values persist across iterations, so unlike the 3rd-RF both ghost
// zones matter.
//
// A ghost zone has constant coefficients and zero input, so across the K
// iterations it is a linear time-invariant system with one input and one
// output on its segment boundary:
//   left zone:  entry state of the ascending pass of iteration k
//               E_L(k) = sum_{j<k}  hL[k-j] x_j,
//               x_j = the segment-start state the descending pass of
//               iteration j hands to the zone;
//   right zone: entry state of the descending pass of iteration k
//               E_R(k) = sum_{j<=k} cR[k-j] y_j,
//               y_j = the segment-end state the ascending pass of
//               iteration j hands to the zone.
// hL (K-1 scalars) and cR (K scalars) depend only on the end point's alpha and
// on G; `k_rf1_zones` computes them per segment by running the reference's
// own zone updates on unit impulses. Each iteration is then one ascending and
// one descending streaming pass over the sea points only; the x_j, y_j of
// every segment are kept in a small history buffer. This removes the 2G ghost
// steps per segment per pass (SURVEY §7 hard part 3: 3.5-9.9x the serial
// work at the configs' masks).
#pragma once
#include "sweep_stream.cuh"
#include "sweep_tma.cuh"

namespace rgfb {

struct Rf1Args {
  int dir, transpose;
  int k;                      // iterations
  int64_t nx, ny, nlev, nvar, lev0;
  int64_t nlev_all;           // levels of the operator (bitsT stride)
  const double2* c1;          // (alpha, beta) per point of this direction
  const uint64_t* bits;       // bit-packed masks (level-major)
  const uint64_t* bitsT;      // chain-minor copy: x [iy][word][lev] (TMA kernels)
  const int64_t* seg_off;     // per (lev, line) segment prefix offsets
  const int2* segs;           // (start, len) per segment (line-resident kernel)
  const int32_t* lpt_ord;     // segments of each line, longest first (k_rf1_sort)
  int64_t nsegs;
  int64_t seg_begin, seg_end;  // segments of this launch's levels
  const double* zone;         // [2K][seg]: hL[0..K) (hL[0] = 0), cR[0..K)
  double* hist;               // [2K][var][seg]: x_1..x_K, y_1..y_K (iteration-major:
                              // an entry-state launch reads only the slices it needs)
  double* ent;                // [var][seg]: entry state of the current pass
  const double* pre_scale;    // first pass only
  const double* post_scale;   // last pass only
};

// ------------------------------------------------------------ zone setup
// One thread per segment: hL / cR of its two zones, forward or adjoint
// dynamics, from unit impulses (scratch: 2 slabs of G per thread).
__global__ void k_rf1_zones(const int2* __restrict__ segs, const int32_t* __restrict__ seg_line,
                            int64_t nsegs, int dir, int64_t nx, int64_t ny,
                            const double2* __restrict__ c1, const int* __restrict__ ghost, int K,
                            bool transpose, double* __restrict__ zone, double* __restrict__ scratch,
                            int64_t slab) {
  const int64_t nlines = dir == 0 ? ny : nx;
  const int64_t n = dir == 0 ? nx : ny;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double* g = scratch + tid * 2 * slab;
  double* p = g + slab;
  for (int64_t s = tid; s < nsegs; s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t lg = seg_line[s];
    const int64_t lev = lg / nlines, line = lg - lev * nlines;
    const int2 sg = segs[s];
    const int64_t i = sg.x, j = sg.x + sg.y - 1;
    const int G = ghost[lev];
    const int gl = i > 0 ? G : 0, gr = j < n - 1 ? G : 0;
    auto pt = [&](int64_t k) { return dir == 0 ? line * nx + k : k * nx + line; };
    const double2 cl = c1[pt(i)], cr = c1[pt(j)];
    double* z = zone + s;  // z[d * nsegs]
    // ---- left zone (alpha, beta of the segment's first point)
    {
      const double a = cl.x, b = cl.y;
      for (int q = 0; q < gl; ++q) g[q] = 0.0;
      z[0] = 0.0;  // hL[0] unused
      for (int k = 1; k <= K; ++k) {
        const double x = k == 1 ? 1.0 : 0.0;  // the impulse enters after iteration 1
        double e = 0.0;
        if (!transpose) {
          // rf1_forward over the ghosts from a zero state; its last value enters
          double prev = 0.0;
          for (int q = 0; q < gl; ++q) {
            prev = b * g[q] + a * prev;
            p[q] = prev;
          }
          e = gl > 0 ? prev : 0.0;
          // rf1_backward into the ghosts, entering state = segment start value
          prev = x;
          for (int q = gl - 1; q >= 0; --q) {
            prev = b * p[q] + a * prev;
            g[q] = prev;
          }
        } else {
          // rf1_backward_transpose (ascending) over the ghosts; its state enters
          double cur = 0.0;
          for (int q = 0; q < gl; ++q) {
            cur = q == 0 ? g[0] : g[q] + a * cur;
            p[q] = b * cur;
          }
          e = gl > 0 ? cur : 0.0;
          // rf1_forward_transpose (descending) into the ghosts, entering state x
          double prev = x;
          for (int q = gl - 1; q >= 0; --q) {
            const double c = p[q] + a * prev;
            g[q] = b * c;
            prev = c;
          }
        }
        if (k >= 2) z[(k - 1) * nsegs] = e;  // hL[k-1]: response at iteration k to x_1
      }
    }
    // ---- right zone (alpha, beta of the segment's last point)
    {
      const double a = cr.x, b = cr.y;
      for (int q = 0; q < gr; ++q) g[q] = 0.0;
      for (int k = 1; k <= K; ++k) {
        const double y = k == 1 ? 1.0 : 0.0;
        double e = 0.0;
        if (!transpose) {
          // rf1_forward continues into the ghosts from the segment end value
          double prev = y;
          for (int q = 0; q < gr; ++q) {
            prev = b * g[q] + a * prev;
            p[q] = prev;
          }
          // rf1_backward from the far end (zero state); its value at the
          // first ghost enters the segment
          prev = 0.0;
          for (int q = gr - 1; q >= 0; --q) {
            prev = b * p[q] + a * prev;
            g[q] = prev;
          }
          e = gr > 0 ? g[0] : 0.0;
        } else {
          // rf1_backward_transpose continues (state y from the segment end)
          double cur = y;
          for (int q = 0; q < gr; ++q) {
            cur = g[q] + a * cur;
            p[q] = b * cur;
          }
          // rf1_forward_transpose from the far end; its state at the first
          // ghost enters the segment
          double prev = 0.0;
          for (int q = gr - 1; q >= 0; --q) {
            const double c = q == gr - 1 ? p[q] : p[q] + a * prev;
            g[q] = b * c;
            prev = c;
          }
          e = gr > 0 ? prev : 0.0;
        }
        z[(K + k - 1) * nsegs] = e;  // cR[k-1]
      }
    }
  }
}

// ------------------------------------------------------------ pass kernels
// Ascending pass (forward: rf1_forward; adjoint: rf1_backward_transpose) and
// descending pass (rf1_backward / rf1_forward_transpose) of iteration `it`.
struct Rf1Asc {
  // non-transposed: state = previous output; transposed: state = internal cur
  // with the previous point's alpha
  double st = 0.0, ap = 0.0;
  template <bool TR>
  __device__ __forceinline__ double step(double a, double b, double w) {
    if (!TR) {
      st = fma(a, st, b * w);  // b_i s_i + a_i prev (covariance.cpp order: mul, mul, add)
      return st;
    }
    st = fma(ap, st, w);  // cur_i = w_i + a_{i-1} cur_{i-1}
    ap = a;
    return b * st;
  }
};

// z = zone + seg (stride zs = nsegs), h = hist + var*nsegs + seg (stride hs =
// nvar*nsegs)
__device__ __forceinline__ double rf1_entry_left(const double* z, int64_t zs, const double* h,
                                                 int64_t hs, int it) {
  double e = 0.0;
  for (int j = 1; j < it; ++j) e = fma(z[(it - j) * zs], h[(j - 1) * hs], e);
  return e;
}
__device__ __forceinline__ double rf1_entry_right(const double* z, int64_t zs, const double* h,
                                                  int64_t hs, int it, int K) {
  double e = 0.0;
  for (int j = 1; j <= it; ++j) e = fma(z[(K + it - j) * zs], h[(K + j - 1) * hs], e);
  return e;
}
// slot of x_it (descending exit) / y_it (ascending exit) in the history
__device__ __forceinline__ int64_t rf1_hist_slot(bool asc, int it, int K, int64_t hs) {
  return (asc ? K + it - 1 : it - 1) * hs;
}

// Entry states of every segment for the coming pass, from the histories
// (one thread per (var, segment), coalesced), so a pass only loads one value
// per segment entry -- prefetched a segment ahead -- instead of a dependent
// K-term sum on scattered memory.
// Only the segments of this launch's levels [s0, s1) (segments are stored
// level-major, so a level chunk's segments are contiguous).
template <bool ASC>
__global__ void k_rf1_entries(Rf1Args a, int it, int64_t s0, int64_t s1) {
  const int K = a.k;
  const int64_t total = a.nvar * a.nsegs;  // history stride
  const int64_t span = s1 - s0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < a.nvar * span;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = q / span, s = s0 + (q - v * span);
    const int64_t t = v * a.nsegs + s;
    const double* z = a.zone + s;
    const double* h = a.hist + t;
    a.ent[t] = ASC ? rf1_entry_left(z, a.nsegs, h, total, it)
                   : rf1_entry_right(z, a.nsegs, h, total, it, K);
  }
}

// y-direction (lines = columns): L planes per thread, U rows per batch,
// lanes = adjacent columns (coalesced row accesses)
template <typename T, bool TR, bool ASC, bool FIRST, bool LAST, int L, int U>
__global__ void __launch_bounds__(128) k_rf1_y(const T* __restrict__ in, T* __restrict__ out,
                                               Rf1Args a, int it) {
  const int64_t nx = a.nx, n = a.ny, nh = nx * n;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t groups = (planes + L - 1) / L;
  // CTA order: plane groups of one column block are adjacent, so they share
  // the column's coefficients and mask words through L2
  const int64_t cb = blockIdx.x / groups, g = blockIdx.x - cb * groups;
  const int64_t ix = cb * blockDim.x + threadIdx.x;
  if (ix >= nx) return;
  const int K = a.k;
  const double2* C = a.c1 + ix;
  const T* src[L];
  T* dst[L];
  const uint64_t* W[L];
  const double* SC[L];
  double* H[L];
  const double* E[L];
  int64_t sidx[L], slo[L], shi[L];
  bool on[L];
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const int64_t p = g * L + l;
    on[l] = p < planes;
    const int64_t pp = on[l] ? p : planes - 1;
    const int64_t var = pp / a.nlev, lev = a.lev0 + (pp - var * a.nlev);
    src[l] = in + pp * nh + ix;
    dst[l] = out + pp * nh + ix;
    W[l] = a.bits + (lev * nx + ix) * ((n + 63) / 64);
    SC[l] = nullptr;
    if (FIRST && TR && a.pre_scale) SC[l] = a.pre_scale + lev * nh + ix;
    if (LAST && a.post_scale) SC[l] = a.post_scale + lev * nh + ix;
    H[l] = a.hist + var * a.nsegs;
    sidx[l] = ASC ? a.seg_off[lev * nx + ix] - 1 : a.seg_off[lev * nx + ix + 1];
    slo[l] = a.seg_off[lev * nx + ix];
    shi[l] = a.seg_off[lev * nx + ix + 1];
    E[l] = a.ent + var * a.nsegs;
  }
  // entry state of each chain's next segment in pass order (prefetched)
  double en[L];
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const int64_t sn = ASC ? sidx[l] + 1 : sidx[l] - 1;
    en[l] = (sn >= slo[l] && sn < shi[l]) ? E[l][sn] : 0.0;
  }
  Rf1Asc st[L];
  uint64_t wc[L], wn[L];
  int prev_sea[L];
#pragma unroll
  for (int l = 0; l < L; ++l) prev_sea[l] = 0;
  const int64_t words = (n + 63) / 64;
  int64_t widx = -1;
  for (int64_t b0 = 0; b0 < n; b0 += U) {
    double2 c[U];
    double s[L][U];
    double sc[L][U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = ASC ? b0 + u : n - 1 - b0 - u;
      if (k >= 0 && k < n) {
        c[u] = __ldg(C + k * nx);
#pragma unroll
        for (int l = 0; l < L; ++l) {
          s[l][u] = on[l] ? static_cast<double>(src[l][k * nx]) : 0.0;
          sc[l][u] = SC[l] ? __ldg(SC[l] + k * nx) : 1.0;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t k = ASC ? b0 + u : n - 1 - b0 - u;
      if (k < 0 || k >= n) continue;
      if ((k >> 6) != widx) {
        widx = k >> 6;
        const int64_t wq = ASC ? widx + 1 : widx - 1;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          wc[l] = ldw(W[l], widx);
          wn[l] = (wq >= 0 && wq < words) ? ldw(W[l], wq) : 0ull;
        }
      }
#pragma unroll
      for (int l = 0; l < L; ++l) {
        const int sea = static_cast<int>((wc[l] >> (k & 63)) & 1ull);
        const int64_t kn = ASC ? k + 1 : k - 1;  // next point in pass order
        int nsea = 0;
        if (kn >= 0 && kn < n)
          nsea = static_cast<int>((((kn >> 6) == widx ? wc[l] : wn[l]) >> (kn & 63)) & 1ull);
        double w = s[l][u];
        if (FIRST && TR) w *= sc[l][u];
        if (sea && !prev_sea[l]) {  // segment entry in pass order
          if (ASC) ++sidx[l]; else --sidx[l];
          st[l].st = en[l];
          st[l].ap = c[u].x;  // the ghost carries this end point's alpha
          const int64_t sn = ASC ? sidx[l] + 1 : sidx[l] - 1;
          en[l] = (sn >= slo[l] && sn < shi[l]) ? E[l][sn] : 0.0;
        }
        double o = st[l].template step<TR>(c[u].x, c[u].y, w);
        if (sea && !nsea && on[l]) {  // segment exit in pass order: record the handed-over state
          // ascending: y_it at the segment end; descending: x_it at its start
          H[l][sidx[l] + rf1_hist_slot(ASC, it, K, a.nvar * a.nsegs)] = st[l].st;
        }
        if (LAST && a.post_scale) o *= sc[l][u];
        if (on[l]) dst[l][k * nx] = static_cast<T>(sea ? o : 0.0);
        prev_sea[l] = sea;
      }
    }
  }
}

// x-direction (lines = rows): thread = chain (plane, row), lanes = planes of
// one row (coefficient loads are broadcasts); each warp stages
// [32 chains x 32 points] tiles with cp.async (one coalesced 256 B row
// segment per instruction) and stores them back cooperatively.
template <typename T, bool TR, bool ASC, bool FIRST, bool LAST>
__global__ void __launch_bounds__(128) k_rf1_x(const T* __restrict__ in, T* __restrict__ out,
                                               Rf1Args a, int it) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* const sm = reinterpret_cast<T*>(smraw);
  const int64_t n = a.nx, ny = a.ny, nh = n * ny;
  const int64_t planes = a.nvar * a.nlev;
  const int K = a.k;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool on = tid < planes * ny;
  const int64_t t = on ? tid : planes * ny - 1;
  const int64_t iy = t / planes, p = t - iy * planes;
  const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
  const int64_t hb = iy * n;
  const T* src = on ? in + p * nh + hb : nullptr;
  T* dst = on ? out + p * nh + hb : nullptr;
  const double2* C = a.c1 + hb;
  const double* SC = nullptr;
  if (FIRST && TR && a.pre_scale) SC = a.pre_scale + lev * nh + hb;
  if (LAST && a.post_scale) SC = a.post_scale + lev * nh + hb;
  const int64_t words = (n + 63) / 64;
  const uint64_t* W = a.bits + (lev * ny + iy) * words;
  double* H = a.hist + var * a.nsegs;
  const double* E = a.ent + var * a.nsegs;
  int64_t sidx = ASC ? a.seg_off[lev * ny + iy] - 1 : a.seg_off[lev * ny + iy + 1];
  const int64_t slo = a.seg_off[lev * ny + iy], shi = a.seg_off[lev * ny + iy + 1];
  auto ent_of = [&](int64_t sn) { return (sn >= slo && sn < shi) ? E[sn] : 0.0; };
  double en = ent_of(ASC ? sidx + 1 : sidx - 1);
  T* const tiles = sm + wid * 2 * 32 * XP;
  const int64_t nb = (n + XB - 1) / XB;

  Rf1Asc st;
  int prev_sea = 0;
  auto bidx = [&](int64_t i) { return ASC ? i : nb - 1 - i; };
  x_stage<T>(tiles + (bidx(0) & 1) * 32 * XP, src, in, bidx(0) * XB, n, lane);
  cp_async_commit();
  for (int64_t i = 0; i < nb; ++i) {
    const int64_t b = bidx(i);
    const int64_t k0 = b * XB;
    T* cur = tiles + (b & 1) * 32 * XP;
    if (i + 1 < nb) {
      const int64_t bn = bidx(i + 1);
      x_stage<T>(tiles + (bn & 1) * 32 * XP, src, in, bn * XB, n, lane);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    // this batch's mask bits plus the neighbours in pass order
    const uint64_t w0 = ldw(W, k0 >> 6);
    const uint64_t wprev = (k0 >> 6) > 0 ? ldw(W, (k0 >> 6) - 1) : 0ull;
    const uint64_t wnext = (k0 >> 6) + 1 < words ? ldw(W, (k0 >> 6) + 1) : 0ull;
    auto sea_at = [&](int64_t k) -> int {
      if (k < 0 || k >= n) return 0;
      const int64_t wi = k >> 6;
      const uint64_t w = wi == (k0 >> 6) ? w0 : (wi < (k0 >> 6) ? wprev : wnext);
      return static_cast<int>((w >> (k & 63)) & 1ull);
    };
    T* row = cur + lane * XP;
#pragma unroll 4
    for (int uu = 0; uu < XB; ++uu) {
      const int u = ASC ? uu : XB - 1 - uu;
      const int64_t k = k0 + u;
      if (k >= n) continue;
      const double2 c = __ldg(C + k);
      const int sea = sea_at(k);
      const int nsea = sea_at(ASC ? k + 1 : k - 1);
      double w = static_cast<double>(row[u]);
      if (FIRST && TR && SC) w *= __ldg(SC + k);
      if (sea && !prev_sea) {  // segment entry in pass order
        if (ASC) ++sidx; else --sidx;
        st.st = en;
        st.ap = c.x;
        en = ent_of(ASC ? sidx + 1 : sidx - 1);
      }
      double o = st.template step<TR>(c.x, c.y, w);
      if (sea && !nsea && on) {
        H[sidx + rf1_hist_slot(ASC, it, K, a.nvar * a.nsegs)] = st.st;
      }
      if (LAST && SC) o *= __ldg(SC + k);
      row[u] = static_cast<T>(sea ? o : 0.0);
      prev_sea = sea;
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

// ------------------------------------------------------------ TMA passes
// Rows 16 B aligned: TMA-fed producer/consumer passes (the structure of the
// 3rd-RF two-pass kernels, sweep_tma.cuh), one producer warp streaming
// field and (alpha, beta) stages into an S-deep ring.

// mask bit of the point after this stage in pass order
template <int U, bool ASC>
__device__ __forceinline__ uint32_t next_after_stage(const StageBits& b, int64_t lo) {
  if (ASC) return b.after<U>(lo);
  return (lo & 63) == 0 ? static_cast<uint32_t>(b.nxt >> 63)
                        : static_cast<uint32_t>((b.cur >> ((lo - 1) & 63)) & 1ull);
}

template <typename T, int NW, int U>
struct R1Y {
  static constexpr size_t field = size_t(NW) * U * 32 * sizeof(T);
  static constexpr size_t coef = size_t(U) * 64 * sizeof(double);
  static constexpr size_t bytes = field + coef;
};

// y: 32 columns x NW planes per CTA, stages of U rows; lanes = columns,
// warps = planes; results stored straight to global (coalesced rows)
template <typename T, bool TR, bool ASC, bool FIRST, bool LAST, int NW, int U, int S>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    k_rf1_ytma(T* __restrict__ out, Rf1Args a, int it, const __grid_constant__ CUtensorMap tm_field,
               const __grid_constant__ CUtensorMap tm_coef) {
  using L = R1Y<T, NW, U>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
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
  const int64_t nst = (ny + U - 1) / U;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = a.k;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwp);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto lo_of = [&](int64_t i) -> int64_t { return (ASC ? i : nst - 1 - i) * U; };
  if (warp == NW) {  // producer
    if (lane == 0) {
      const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
      tma_prefetch_desc(&tm_field);
      tma_prefetch_desc(&tm_coef);
      for (int64_t i = 0; i < nst; ++i) {
        const int s = static_cast<int>(i % S);
        if (i >= S) mbar_wait(&empty[s], static_cast<uint32_t>((i / S - 1) & 1));
        const int lo = static_cast<int>(lo_of(i));
        unsigned char* base = smem + s * L::bytes;
        mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(L::bytes));
        tma_load_3d(base, &tm_field, static_cast<int>(ix0), lo, static_cast<int>(p0), &full[s],
                    pol_stream);
        tma_load_2d(base + L::field, &tm_coef, static_cast<int>(2 * ix0), lo, &full[s], pol_keep);
      }
    }
    return;
  }
  if (warp >= nwp) return;
  const int64_t p = p0 + warp;
  const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
  const bool act = lane < ncol;
  const int64_t ix = ix0 + (act ? lane : 0);
  T* dst = out + p * nh + ix;
  const uint64_t* W = a.bits + (lev * nx + ix) * ((ny + 63) / 64);
  const int64_t words = (ny + 63) / 64;
  const double* SC = nullptr;
  if (FIRST && TR && a.pre_scale) SC = a.pre_scale + lev * nh + ix;
  if (LAST && a.post_scale) SC = a.post_scale + lev * nh + ix;
  double* H = a.hist + var * a.nsegs;
  const double* E = a.ent + var * a.nsegs;
  const int64_t slo = a.seg_off[lev * nx + ix], shi = a.seg_off[lev * nx + ix + 1];
  int64_t sidx = ASC ? slo - 1 : shi;
  auto ent_of = [&](int64_t sn) { return (sn >= slo && sn < shi) ? E[sn] : 0.0; };
  double en = ent_of(ASC ? sidx + 1 : sidx - 1);
  StageBits sbw;
  Rf1Asc st;
  uint32_t prevb = 0;  // sea bit of the previous point in pass order
  for (int64_t i = 0; i < nst; ++i) {
    const int s = static_cast<int>(i % S);
    const int64_t lo = lo_of(i);
    sbw.seek(W, lo, words, !ASC);
    const uint32_t sb = sbw.stage<U>(lo);
    const uint32_t nb = next_after_stage<U, ASC>(sbw, lo);
    mbar_wait(&full[s], static_cast<uint32_t>((i / S) & 1));
    const unsigned char* base = smem + s * L::bytes;
    const T* fld = reinterpret_cast<const T*>(base) + warp * U * 32 + lane;
    const double2* cf = reinterpret_cast<const double2*>(base + L::field) + lane;
    const int rvalid = static_cast<int>(ny - lo < U ? ny - lo : U);
#pragma unroll
    for (int uu = 0; uu < U; ++uu) {
      const int r = ASC ? uu : U - 1 - uu;
      const int64_t k = lo + r;
      const uint32_t sea = (sb >> r) & 1u;
      const uint32_t nsea = ASC ? (r + 1 < U ? (sb >> (r + 1)) & 1u : nb)
                                : (r > 0 ? (sb >> (r - 1)) & 1u : nb);
      const double2 c = cf[r * 32];
      double w = static_cast<double>(fld[r * 32]);
      if (FIRST && TR && SC && r < rvalid) w *= __ldg(SC + k * nx);
      if (sea && !prevb) {  // segment entry in pass order
        if (ASC) ++sidx; else --sidx;
        st.st = en;
        st.ap = c.x;
        en = ent_of(ASC ? sidx + 1 : sidx - 1);
      }
      double o = st.template step<TR>(c.x, c.y, w);
      if (sea && !nsea && act) {
        H[sidx + rf1_hist_slot(ASC, it, K, a.nvar * a.nsegs)] = st.st;
      }
      if (LAST && SC && r < rvalid) o *= __ldg(SC + k * nx);
      if (act && r < rvalid) __stcs(dst + k * nx, static_cast<T>(sea ? o : 0.0));
      prevb = sea;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// x: one row x 32*NW planes per CTA; U-point stages of [U x 128 planes],
// 128 B swizzled; results written back in place and returned by TMA stores
template <typename T, bool TR, bool ASC, bool FIRST, bool LAST, int NW, int S>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    k_rf1_xtma(Rf1Args a, int it, const __grid_constant__ CUtensorMap tm_in,
               const __grid_constant__ CUtensorMap tm_out, const __grid_constant__ CUtensorMap tm_coef) {
  constexpr int U = 128 / int(sizeof(T));
  constexpr size_t FIELD = size_t(NW) * 32 * 128;
  constexpr size_t COEF = size_t(U) * 16;
  constexpr size_t BYTES = (FIELD + COEF + 1023) / 1024 * 1024;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * BYTES);
  uint64_t* empty = full + S;
  const int64_t n = a.nx, ny = a.ny, nh = n * ny;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t PB = (planes + 32 * NW - 1) / (32 * NW);
  const int64_t iy = blockIdx.x / PB;
  const int64_t p0 = (blockIdx.x - iy * PB) * 32 * NW;
  const int npl = static_cast<int>(planes - p0 < 32 * NW ? planes - p0 : 32 * NW);
  const int64_t nst = (n + U - 1) / U;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = a.k;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  auto k0_of = [&](int64_t i) -> int64_t { return (ASC ? i : nst - 1 - i) * U; };
  if (warp == NW) {  // producer
    if (lane == 0) {
      const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
      tma_prefetch_desc(&tm_in);
      tma_prefetch_desc(&tm_coef);
      for (int64_t i = 0; i < nst; ++i) {
        const int s = static_cast<int>(i % S);
        if (i >= S) mbar_wait(&empty[s], static_cast<uint32_t>((i / S - 1) & 1));
        const int k0 = static_cast<int>(k0_of(i));
        unsigned char* base = smem + s * BYTES;
        mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(FIELD + COEF));
        tma_load_3d(base, &tm_in, k0, static_cast<int>(iy), static_cast<int>(p0), &full[s],
                    pol_stream);
        tma_load_2d(base + FIELD, &tm_coef, 2 * k0, static_cast<int>(iy), &full[s], pol_keep);
      }
    }
    return;
  }
  const int pr = warp * 32 + lane;
  const bool act = pr < npl;
  const int64_t p = p0 + (act ? pr : 0);
  const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
  const int64_t words = (n + 63) / 64;
  const uint64_t* W = a.bitsT + iy * words * a.nlev_all + lev;  // lanes: consecutive words
  const int64_t ws = a.nlev_all;
  const double* SC = nullptr;
  if (FIRST && TR && a.pre_scale) SC = a.pre_scale + lev * nh + iy * n;
  if (LAST && a.post_scale) SC = a.post_scale + lev * nh + iy * n;
  double* H = a.hist + var * a.nsegs;
  const double* E = a.ent + var * a.nsegs;
  const int64_t slo = a.seg_off[lev * ny + iy], shi = a.seg_off[lev * ny + iy + 1];
  int64_t sidx = ASC ? slo - 1 : shi;
  auto ent_of = [&](int64_t sn) { return (sn >= slo && sn < shi) ? E[sn] : 0.0; };
  double en = ent_of(ASC ? sidx + 1 : sidx - 1);
  StageBits sbw;
  Rf1Asc st;
  uint32_t prevb = 0;
  constexpr int ESZ = static_cast<int>(sizeof(T));
  constexpr int EPC = 16 / ESZ;
  const int sw = pr & 7;
  for (int64_t i = 0; i < nst; ++i) {
    const int s = static_cast<int>(i % S);
    const int64_t k0 = k0_of(i);
    sbw.seek(W, k0, words, !ASC, ws);
    const uint32_t sb = sbw.stage<U>(k0);
    const uint32_t nb = next_after_stage<U, ASC>(sbw, k0);
    mbar_wait(&full[s], static_cast<uint32_t>((i / S) & 1));
    unsigned char* base = smem + s * BYTES;
    const double2* cf = reinterpret_cast<const double2*>(base + FIELD);
    unsigned char* rowp = base + pr * 128;
#pragma unroll
    for (int qq = 0; qq < U / EPC; ++qq) {
      const int q = ASC ? qq : U / EPC - 1 - qq;
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
      for (int ee = 0; ee < EPC; ++ee) {
        const int e = ASC ? ee : EPC - 1 - ee;
        const int u = q * EPC + e;
        const int64_t k = k0 + u;
        const uint32_t sea = (sb >> u) & 1u;
        const uint32_t nsea = ASC ? (u + 1 < U ? (sb >> (u + 1)) & 1u : nb)
                                  : (u > 0 ? (sb >> (u - 1)) & 1u : nb);
        const double2 c = cf[u];
        double w = v[e];
        if (FIRST && TR && SC && k < n) w *= __ldg(SC + k);
        if (sea && !prevb) {
          if (ASC) ++sidx; else --sidx;
          st.st = en;
          st.ap = c.x;
          en = ent_of(ASC ? sidx + 1 : sidx - 1);
        }
        double o = st.template step<TR>(c.x, c.y, w);
        if (sea && !nsea && act) {
          H[sidx + rf1_hist_slot(ASC, it, K, a.nvar * a.nsegs)] = st.st;
        }
        if (LAST && SC && k < n) o *= __ldg(SC + k);
        v[e] = sea ? o : 0.0;
        prevb = sea;
      }
      if constexpr (sizeof(T) == 8) {
        *reinterpret_cast<double2*>(cp) = make_double2(v[0], v[1]);
      } else {
        *reinterpret_cast<float4*>(cp) =
            make_float4(static_cast<float>(v[0]), static_cast<float>(v[1]),
                        static_cast<float>(v[2]), static_cast<float>(v[3]));
      }
    }
    fence_proxy_async_smem();
    asm volatile("bar.sync 1, %0;\n" ::"r"(32 * NW) : "memory");
    if (threadIdx.x == 0) {
      tma_store_3d(&tm_out, static_cast<int>(k0), static_cast<int>(iy), static_cast<int>(p0), base,
                   l2_evict_first());
      bulk_commit();
      asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
      if (i > 0) mbar_arrive(&empty[(i - 1) % S]);
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

template <typename T, bool TR, bool ASC, bool F, bool LST>
void launch_rf1_tma(const T* src, T* dst, const Rf1Args& a, int it, cudaStream_t st) {
  const int64_t planes = a.nvar * a.nlev;
  const uint64_t sz = sizeof(T);
  const uint64_t fd[3] = {uint64_t(a.nx), uint64_t(a.ny), uint64_t(planes)};
  const uint64_t fs[2] = {uint64_t(a.nx) * sz, uint64_t(a.nx * a.ny) * sz};
  const uint64_t cd[2] = {uint64_t(2 * a.nx), uint64_t(a.ny)};
  const uint64_t cs[1] = {uint64_t(2 * a.nx) * 8};
  if (a.dir == 1) {
    constexpr int NW = 16, U = 8, S = 4;
    using L = R1Y<T, NW, U>;
    const size_t smem = S * L::bytes + 2 * S * sizeof(uint64_t) + 1024;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_rf1_ytma<T, TR, ASC, F, LST, NW, U, S>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      attr = true;
    }
    const uint32_t fb[3] = {32, U, NW};
    const CUtensorMap tf = make_tmap(src, tma_dtype<T>(), 3, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_NONE);
    const uint32_t cb[2] = {64, U};
    const CUtensorMap tc =
        make_tmap(a.c1, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, cd, cs, cb, CU_TENSOR_MAP_SWIZZLE_NONE);
    const int64_t blocks = ((a.nx + 31) / 32) * ((planes + NW - 1) / NW);
    k_rf1_ytma<T, TR, ASC, F, LST, NW, U, S><<<blocks, 32 * (NW + 1), smem, st>>>(dst, a, it, tf, tc);
  } else {
    constexpr int NW = 4, S = 4;
    constexpr int U = 128 / int(sizeof(T));
    constexpr size_t BYTES = (size_t(NW) * 32 * 128 + size_t(U) * 16 + 1023) / 1024 * 1024;
    const size_t smem = S * BYTES + 2 * S * sizeof(uint64_t) + 1024;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_rf1_xtma<T, TR, ASC, F, LST, NW, S>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      attr = true;
    }
    const uint32_t fb[3] = {uint32_t(U), 1, uint32_t(32 * NW)};
    const CUtensorMap tin = make_tmap(src, tma_dtype<T>(), 3, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
    const CUtensorMap tout = make_tmap(dst, tma_dtype<T>(), 3, fd, fs, fb,
                                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
    const uint32_t cb[2] = {uint32_t(2 * U), 1};
    const CUtensorMap tc =
        make_tmap(a.c1, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, cd, cs, cb, CU_TENSOR_MAP_SWIZZLE_NONE);
    const int64_t PB = (planes + 32 * NW - 1) / (32 * NW);
    k_rf1_xtma<T, TR, ASC, F, LST, NW, S><<<a.ny * PB, 32 * (NW + 1), smem, st>>>(a, it, tin, tout,
                                                                               tc);
  }
}

// K iterations of one directional sweep (2K passes + entry-state kernels)
template <typename T>
int launch_rf1_sweep(const T* in, T* out, const Rf1Args& a, cudaStream_t st) {
  const int threads = 128;
  const int64_t planes = a.nvar * a.nlev;
  int launches = 0;
  const bool tma = a.bitsT != nullptr && tma_supported(in, out, a.nx);
  auto pass = [&](bool asc, bool first, bool last, const T* src, T* dst, int it) {
    if (tma) {
#define RGFB_RF1T(TR, ASC, F, L) launch_rf1_tma<T, TR, ASC, F, L>(src, dst, a, it, st);
      if (a.transpose) {
        if (asc) {
          if (first) { RGFB_RF1T(true, true, true, false) } else { RGFB_RF1T(true, true, false, false) }
        } else {
          if (last) { RGFB_RF1T(true, false, false, true) } else { RGFB_RF1T(true, false, false, false) }
        }
      } else {
        if (asc) {
          if (first) { RGFB_RF1T(false, true, true, false) } else { RGFB_RF1T(false, true, false, false) }
        } else {
          if (last) { RGFB_RF1T(false, false, false, true) } else { RGFB_RF1T(false, false, false, false) }
        }
      }
#undef RGFB_RF1T
      ++launches;
      return;
    }
#define RGFB_RF1(TR, ASC, F, L)                                                                  \
  if (a.dir == 1) {                                                                              \
    constexpr int LL = 4, UU = 4;                                                                \
    const int64_t blocks = ((planes + LL - 1) / LL) * ((a.nx + threads - 1) / threads);        \
    k_rf1_y<T, TR, ASC, F, L, LL, UU><<<blocks, threads, 0, st>>>(src, dst, a, it);            \
  } else {                                                                                       \
    const int smem = 4 * 2 * 32 * XP * static_cast<int>(sizeof(T));                            \
    static bool attr = false;                                                                    \
    if (!attr) {                                                                                 \
      cudaFuncSetAttribute(k_rf1_x<T, TR, ASC, F, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           smem);                                                                \
      attr = true;                                                                               \
    }                                                                                            \
    const int64_t chains = planes * a.ny;                                                        \
    k_rf1_x<T, TR, ASC, F, L><<<(chains + threads - 1) / threads, threads, smem, st>>>(src, dst, \
                                                                                     a, it);     \
  }
    if (a.transpose) {
      if (asc) {
        if (first) { RGFB_RF1(true, true, true, false) } else { RGFB_RF1(true, true, false, false) }
      } else {
        if (last) { RGFB_RF1(true, false, false, true) } else { RGFB_RF1(true, false, false, false) }
      }
    } else {
      if (asc) {
        if (first) { RGFB_RF1(false, true, true, false) } else { RGFB_RF1(false, true, false, false) }
      } else {
        if (last) { RGFB_RF1(false, false, false, true) } else { RGFB_RF1(false, false, false, false) }
      }
    }
#undef RGFB_RF1
    ++launches;
  };
  // this launch's segments: levels [lev0, lev0 + nlev) of every line
  const int64_t nlines = a.dir == 0 ? a.ny : a.nx;
  const int64_t s0 = a.seg_begin, s1 = a.seg_end;
  (void)nlines;
  const int64_t ne = a.nvar * (s1 - s0);
  const int eblocks = static_cast<int>(std::min<int64_t>((ne + 255) / 256, 148 * 16));
  for (int it = 1; it <= a.k; ++it) {
    if (it > 1 && ne > 0) {  // iteration 1 enters every segment from zero
      k_rf1_entries<true><<<eblocks, 256, 0, st>>>(a, it, s0, s1);
      ++launches;
    } else if (ne > 0) {
      for (int64_t v = 0; v < a.nvar; ++v)
        cudaMemsetAsync(a.ent + v * a.nsegs + s0, 0, static_cast<size_t>(s1 - s0) * sizeof(double),
                        st);
    }
    pass(true, it == 1, false, it == 1 ? in : out, out, it);
    if (ne > 0) {
      k_rf1_entries<false><<<eblocks, 256, 0, st>>>(a, it, s0, s1);
      ++launches;
    }
    pass(false, false, it == a.k, out, out, it);
  }
  return launches;
}

}  // namespace rgfb
