// Line-resident 1st-RF: all K iterations of one sweep in ONE field pass.
//
// Reference (rf1.hpp:20-63, 113-137; covariance.cpp:283-286, 319-322,
// 334-339): K x {forward, backward} (adjoint: K x {backward-transpose,
// forward-transpose}) over every sea segment extended by G ghosts per side.
// The streaming form (rf1_stream.cuh) runs each of the 2K passes as its own
// kernel: 4K field moves per sweep. Here a whole line (x: one row of one
// plane; y: C adjacent columns of one plane) stays in shared memory for all
// 2K passes, and each pass is a PARALLEL SCAN along the line instead of a
// serial walk, so the line needs no other chains to hide the recursion
// latency: one read and one write of the field per sweep.
//
//   * A first-order pass r_i = l_i r_{i-1} + t_i composes as affine maps
//     (A, B) -> (A' A, A' B + B'). Thread (q, c) owns V consecutive points of
//     line c: it runs the recursion over its chunk from a zero state (B) with
//     the chunk's link product A = prod l_i fixed per line, one warp per line
//     scans the NQ chunk aggregates (lane-serial + shuffle scan), and the
//     thread re-runs its chunk from the true carry, writing in place.
//   * Links l_i are alpha_i at sea points and 0 on land, so land cuts the
//     chain and a land point keeps its stored value. That makes land points
//     free storage: the ghost-zone entry state of the coming pass (E_L before
//     a segment start for ascending passes, E_R after a segment end for
//     descending ones; rf1_stream.cuh explains the zone algebra) is PLACED in
//     the adjacent land slot, and the uniform recursion picks it up as the
//     previous state. No per-point segment logic in the passes.
//   * Between passes one thread per segment records the handed-over state
//     (x_it at the start, y_it at the end), evaluates the zone convolution
//     from the histories kept in shared memory, and places the next entry.
//   * The adjoint passes cur_i = w_i + a_{i-1} cur_{i-1}, out = b_i cur_i
//     run on z_i = a_i cur_i (z_i = a_i z_{i-1} + a_i w_i: the same links),
//     with cur_i = w_i + z_{i-1} stored and the b_i factor applied to the
//     next pass's input (and to the final output).
//
// Arithmetic differs from the serial passes by FMA association only
// (~1e-15 relative; parity tests require 1e-12 fp64 / 1e-5 fp32).
#pragma once
#include "rf1_stream.cuh"

namespace rgfb {

struct Rf1LineArgs {
  int dir, transpose, k;
  int64_t nx, ny, nlev, nvar, lev0;
  const double2* c1;        // (alpha, beta) per point of this direction
  const uint64_t* bits;     // level-major bit-packed masks along dir
  int64_t words;            // 64-bit words per line
  const int64_t* seg_off;   // per (lev, line) segment prefix offsets
  const int2* segs;         // (start, len) per segment
  int64_t nsegs;            // zone stride
  const double* zone;       // [2K][nsegs]: hL[0..K), cR[0..K)
  const int* ghost;         // per level
  const uint8_t* same;      // per level: mask and ghost width equal the previous level's
  const double* pre_scale;  // adjoint: input multiplier (nlev*nh) or null
  const double* post_scale; // output multiplier or null
  int segcap;               // max segments per line of this direction
  int planes_per_cta;       // planes a CTA walks through
};

// 64 mask bits of a line starting at bit `start` (>= 0); bits past the packed
// words read as 0 (bits past the line end are 0 in the packed mask)
__device__ __forceinline__ uint64_t rf1l_window(const uint64_t* W, int64_t words, int64_t start) {
  const int64_t wi = start >> 6;
  const int sh = static_cast<int>(start & 63);
  const uint64_t lo = wi < words ? ldw(W, wi) : 0ull;
  const uint64_t hi = wi + 1 < words ? ldw(W, wi + 1) : 0ull;
  return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
}

template <typename S, int NT, int V, int C>
struct Rf1LineSmem {
  static constexpr int NQ = NT / C;    // chunks per line
  static constexpr int CAP = NQ * V;   // points per line held
  static size_t bytes(int K, int segcap) {
    size_t b = size_t(CAP) * C * sizeof(S);
    b = (b + 15) / 16 * 16;
    b += size_t(3) * NT * sizeof(double);                 // aggA, aggB, cin
    b += size_t(2) * K * C * segcap * sizeof(double);     // zone cache
    b += size_t(2) * K * C * segcap * sizeof(double);     // histories x_j, y_j
    b += size_t(C) * segcap * sizeof(int2);               // (start, len)
    b += size_t(2) * C * sizeof(int64_t);                 // segment base / count per line
    b += size_t(C) * (CAP / 64 + 2) * sizeof(uint64_t);   // mask words of the C lines
    return b;
  }
};

// One CTA: C adjacent lines (x: C = 1 row; y: C columns) of `planes_per_cta`
// planes, one plane at a time. Thread t = q*C + c owns points [q*V, q*V+V) of
// line c. S is the shared-memory storage type of the resident line.
template <typename T, typename S, bool TR, int NT, int V, int C, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_rf1_line(const T* __restrict__ in, T* __restrict__ out,
                                                       Rf1LineArgs a) {
  using L = Rf1LineSmem<S, NT, V, C>;
  constexpr int NQ = L::NQ, CAP = L::CAP;
  constexpr int SS = NQ / 32;  // chunk aggregates per scanning lane
  static_assert(NQ % 32 == 0, "one warp scans a line's chunk aggregates");
  static_assert(V + 2 <= 64, "chunk mask window");
  extern __shared__ __align__(16) unsigned char smraw[];
  const int K = a.k, segcap = a.segcap;
  S* const sd = reinterpret_cast<S*>(smraw);
  double* const aggA =
      reinterpret_cast<double*>(smraw + (size_t(CAP) * C * sizeof(S) + 15) / 16 * 16);
  double* const aggB = aggA + NT;
  double* const cinv = aggB + NT;
  double* const zc = cinv + NT;                       // [2K][C*segcap]
  double* const hist = zc + size_t(2) * K * C * segcap;  // [2K][C*segcap]: x_1..x_K, y_1..y_K
  int2* const sseg = reinterpret_cast<int2*>(hist + size_t(2) * K * C * segcap);
  int64_t* const sbase = reinterpret_cast<int64_t*>(sseg + size_t(C) * segcap);
  int64_t* const scnt = sbase + C;
  uint64_t* const mw = reinterpret_cast<uint64_t*>(scnt + C);  // [C][MWW]
  constexpr int MWW = CAP / 64 + 2;
  constexpr bool XD = C == 1;       // x sweeps hold one row, y sweeps C columns
  constexpr int U = V == 35 ? 7 : V;  // loads in flight per thread (V = U * batches)

  const int64_t nx = a.nx, ny = a.ny, nh = nx * ny;
  const bool xdir = a.dir == 0;
  const int64_t n = xdir ? nx : ny;            // points per line
  const int64_t nl = xdir ? ny : nx;           // lines per level
  const int64_t planes = a.nvar * a.nlev;
  const int64_t ntile = (nl + C - 1) / C;
  const int64_t groups = (planes + a.planes_per_cta - 1) / a.planes_per_cta;
  const int64_t tile = blockIdx.x / groups, grp = blockIdx.x - tile * groups;
  const int64_t line0 = tile * C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = tid % C, q = tid / C;
  const int64_t line = line0 + c;
  const bool lineok = line < nl;
  const int64_t p0 = int64_t(q) * V;           // first point of this thread's chunk
  // strides of (point, line) in a plane
  const int64_t sp = XD ? 1 : nx, sl = XD ? nx : 1;
  (void)ntile;
  (void)xdir;

  const int64_t pl_begin = grp * a.planes_per_cta;
  const int64_t pl_end = pl_begin + a.planes_per_cta < planes ? pl_begin + a.planes_per_cta : planes;
  for (int64_t pl = pl_begin; pl < pl_end; ++pl) {
    const int64_t var = pl / a.nlev, lev = a.lev0 + (pl - var * a.nlev);
    (void)var;
    const uint64_t* Wl = a.bits + (lev * nl + (lineok ? line : 0)) * a.words;
    const int G = a.ghost[lev];

    // ---- chunk masks and links (registers)
    uint64_t win = 0;
    if (lineok) win = p0 > 0 ? rf1l_window(Wl, a.words, p0 - 1) : (rf1l_window(Wl, a.words, 0) << 1);
    constexpr uint64_t VM = (1ull << V) - 1ull;
    const uint64_t sea = (win >> 1) & VM, prv = win & VM, nxt = (win >> 2) & VM;
    const uint64_t frozen = G == 0 ? (sea & ~prv & ~nxt) : 0ull;  // covariance.cpp:260-269
    const uint64_t live = sea & ~frozen;
    double la[V];
    {
      const double* cp = reinterpret_cast<const double*>(a.c1 + (lineok ? line * sl + p0 * sp : 0));
      const int64_t cst = 2 * sp;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        double al = 0.0;
        if ((live >> i) & 1ull) al = __ldg(cp + i * cst);
        la[i] = al;
      }
    }
    double A = 1.0;
#pragma unroll
    for (int i = 0; i < V; ++i) A *= la[i];
    aggA[c * NQ + q] = A;
    for (int w = tid; w < C * MWW; w += NT) {
      const int cc = w / MWW, ww = w - cc * MWW;
      mw[w] = (line0 + cc < nl && ww < a.words) ? ldw(a.bits + (lev * nl + line0 + cc) * a.words, ww)
                                                : 0ull;
    }

    // ---- segments of the C lines, zone responses, histories
    if (tid < C) {
      const int64_t ln = line0 + tid;
      const int64_t b0 = ln < nl ? a.seg_off[lev * nl + ln] : 0;
      const int64_t b1 = ln < nl ? a.seg_off[lev * nl + ln + 1] : 0;
      sbase[tid] = b0;
      scnt[tid] = b1 - b0;
    }
    __syncthreads();
    for (int w = tid; w < C * segcap; w += NT) {
      const int cc = w % C, s = w / C;
      if (s < scnt[cc]) {
        const int64_t g = sbase[cc] + s;
        sseg[w] = a.segs[g];
        for (int d = 0; d < 2 * K; ++d) zc[d * C * segcap + w] = __ldg(a.zone + d * a.nsegs + g);
      }
    }

    // ---- load the lines (coalesced, U loads in flight per thread), land = 0,
    // adjoint input scaling
    {
      const T* src = in + pl * nh + line0 * sl;
      const double* pre = (TR && a.pre_scale) ? a.pre_scale + lev * nh + line0 * sl : nullptr;
#pragma unroll 1
      for (int k0 = 0; k0 < V; k0 += U) {
        T buf[U];
        double pb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = tid + (k0 + u) * NT;
          const int i = e / C, cc = e % C;
          const bool ok = i < n && line0 + cc < nl;
          buf[u] = ok ? src[i * sp + cc * sl] : T(0);
          pb[u] = 1.0;
          if (TR) pb[u] = (pre && ok) ? __ldg(pre + i * sp + cc * sl) : 1.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = tid + (k0 + u) * NT;
          const int i = e / C, cc = e % C;
          const bool on = (mw[cc * MWW + (i >> 6)] >> (i & 63)) & 1ull;
          double v = on ? static_cast<double>(buf[u]) : 0.0;
          if (TR) v *= pb[u];
          sd[e] = static_cast<S>(v);
        }
      }
    }
    __syncthreads();

    // ---- one pass: chunk recursion from zero, scan, re-run from the carry
    auto pass = [&](auto asc_c, auto first_c, auto last_c) {
      constexpr bool ASC = decltype(asc_c)::value;
      constexpr bool FIRST = decltype(first_c)::value;  // adjoint: raw input
      constexpr bool LAST = decltype(last_c)::value;    // adjoint: b_i on the output
      double r = 0.0;
#pragma unroll
      for (int ii = 0; ii < V; ++ii) {
        const int i = ASC ? ii : V - 1 - ii;
        const double v = static_cast<double>(sd[(p0 + i) * C + c]);
        double t;
        if constexpr (!TR) {
          t = fma(-la[i], v, v);  // b_i s_i, b = 1 - a; a land slot keeps its value
        } else {
          const double w = FIRST ? v : fma(-la[i], v, v);
          t = ((live >> i) & 1ull) ? la[i] * w : v;
        }
        r = fma(la[i], r, t);
      }
      aggB[c * NQ + (ASC ? q : NQ - 1 - q)] = r;
      __syncthreads();
      if (warp < C) {  // warp `warp` scans line `warp`
        double ea[SS], eb[SS];
        double ar = 1.0, br = 0.0;
#pragma unroll
        for (int kk = 0; kk < SS; ++kk) {
          const int pos = lane * SS + kk;
          const double aj = aggA[warp * NQ + (ASC ? pos : NQ - 1 - pos)];
          const double bj = aggB[warp * NQ + pos];
          ea[kk] = ar;
          eb[kk] = br;
          br = fma(aj, br, bj);
          ar *= aj;
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const double ua = __shfl_up_sync(0xffffffffu, ar, d);
          const double ub = __shfl_up_sync(0xffffffffu, br, d);
          if (lane >= d) {
            br = fma(ar, ub, br);
            ar *= ua;
          }
        }
        double X = __shfl_up_sync(0xffffffffu, br, 1);
        if (lane == 0) X = 0.0;
#pragma unroll
        for (int kk = 0; kk < SS; ++kk) cinv[warp * NQ + lane * SS + kk] = fma(ea[kk], X, eb[kk]);
      }
      __syncthreads();
      r = cinv[c * NQ + (ASC ? q : NQ - 1 - q)];
#pragma unroll
      for (int ii = 0; ii < V; ++ii) {
        const int i = ASC ? ii : V - 1 - ii;
        S* const ptr = &sd[(p0 + i) * C + c];
        const double v = static_cast<double>(*ptr);
        if constexpr (!TR) {
          r = fma(la[i], r, fma(-la[i], v, v));
          *ptr = static_cast<S>(r);
        } else {
          const bool on = (live >> i) & 1ull;
          const double w = FIRST ? v : fma(-la[i], v, v);
          const double cur = w + r;  // cur_i = w_i + a_{i-1} cur_{i-1}
          r = fma(la[i], r, on ? la[i] * w : v);
          if (on) *ptr = static_cast<S>(LAST ? fma(-la[i], cur, cur) : cur);
        }
      }
      __syncthreads();
    };

    // ---- between passes: record exits, place the next entries
    // after the ascending pass of iteration it: y_it at segment ends, E_R(it)
    // after the descending pass (it < K): x_it at segment starts, E_L(it+1)
    auto boundary = [&](bool after_asc, int it) {
      const int SC = C * segcap;
      for (int w = tid; w < SC; w += NT) {
        const int cc = w % C, s = w / C;
        if (s >= scnt[cc]) continue;
        const int2 sg = sseg[w];
        const int64_t i0 = sg.x, j0 = int64_t(sg.x) + sg.y - 1;
        if (after_asc) {
          hist[(K + it - 1) * SC + w] = static_cast<double>(sd[j0 * C + cc]);
          if (j0 < n - 1) {
            double e = 0.0;
            for (int j = 1; j <= it; ++j)
              e = fma(zc[(K + it - j) * SC + w], hist[(K + j - 1) * SC + w], e);
            if (TR) e *= __ldg(&a.c1[(line0 + cc) * sl + j0 * sp].x);
            sd[(j0 + 1) * C + cc] = static_cast<S>(e);
          }
        } else {
          hist[(it - 1) * SC + w] = static_cast<double>(sd[i0 * C + cc]);
          if (i0 > 0) {
            double e = 0.0;
            for (int j = 1; j <= it; ++j) e = fma(zc[(it + 1 - j) * SC + w], hist[(j - 1) * SC + w], e);
            if (TR) e *= __ldg(&a.c1[(line0 + cc) * sl + i0 * sp].x);
            sd[(i0 - 1) * C + cc] = static_cast<S>(e);
          }
        }
      }
      __syncthreads();
    };

    using Tt = std::true_type;
    using Ft = std::false_type;
    for (int it = 1; it <= K; ++it) {
      if (TR && it == 1) pass(Tt{}, Tt{}, Ft{}); else pass(Tt{}, Ft{}, Ft{});
      boundary(true, it);
      if (TR && it == K) pass(Ft{}, Ft{}, Tt{}); else pass(Ft{}, Ft{}, Ft{});
      if (it < K) boundary(false, it);
    }

    // ---- store (coalesced), land exactly 0, output scaling
    {
      T* dst = out + pl * nh + line0 * sl;
      const double* post = a.post_scale ? a.post_scale + lev * nh + line0 * sl : nullptr;
#pragma unroll 1
      for (int k0 = 0; k0 < V; k0 += U) {
        double pb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = tid + (k0 + u) * NT;
          const int i = e / C, cc = e % C;
          pb[u] = (post && i < n && line0 + cc < nl) ? __ldg(post + i * sp + cc * sl) : 1.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = tid + (k0 + u) * NT;
          const int i = e / C, cc = e % C;
          if (i < n && line0 + cc < nl) {
            const bool on = (mw[cc * MWW + (i >> 6)] >> (i & 63)) & 1ull;
            const double v = on ? static_cast<double>(sd[e]) * pb[u] : 0.0;
            dst[i * sp + cc * sl] = static_cast<T>(v);
          }
        }
      }
    }
    __syncthreads();  // the next plane rewrites the mask words and the line
  }
}

// ------------------------------------------------------------ row kernel
// Register-resident form for lines that are rows of the field (x sweeps, and y
// sweeps on a transposed field): thread t keeps its V points AND their links in
// registers for all 2K passes, so a pass touches shared memory only where a
// value changes hands: a land slot next to a segment is re-read (its entry
// was placed by the boundary phase) and a segment's exit point is published.
// The chunk aggregates are scanned by every warp with shuffles (no idle
// warps) and the warp totals folded through shared memory.
struct Rf1RowArgs {
  int transpose, k;
  int n, nl;                // points per line, lines per level
  int64_t nlev, nvar, lev0;
  const double2* c1;        // (alpha, beta): point (line, i) at c1[line*csl + i*csp]
  int64_t csp, csl;
  const uint64_t* bits;     // [(lev*nl + line)*words + w]
  int64_t words;
  const int64_t* seg_off;
  const int2* segs;
  int64_t nsegs;
  const double* zone;
  const int* ghost;
  const uint8_t* same;      // per level: mask and ghost width equal the previous level's
  const double* pre_scale;  // [lev][line][i] (dense rows) or null
  const double* post_scale;
  int segcap;
  int planes_per_cta;
};

// predicated shared-memory exchange on a precomputed 32-bit shared address (the
// compiler otherwise rebuilds the base address for every predicated access)
__device__ __forceinline__ void rf1l_lds_if(double& v, uint32_t addr, uint32_t on) {
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p ld.shared.f64 %0, [%1];\n}\n"
               : "+d"(v)
               : "r"(addr), "r"(on)
               : "memory");
}
__device__ __forceinline__ void rf1l_sts_if(uint32_t addr, double v, uint32_t on) {
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.shared.f64 [%0], %1;\n}\n" ::"r"(addr),
               "d"(v), "r"(on)
               : "memory");
}

template <int NT, int V>
struct Rf1RowSmem {
  static constexpr int CAP = NT * V;
  static constexpr int MWW = CAP / 64 + 2;
  static constexpr int NW = NT / 32;
  static size_t bytes(int K, int segcap) {
    size_t b = size_t(2) * CAP * sizeof(double);        // exchange line + input staging
    b += size_t(2) * NW * sizeof(double);               // warp totals
    b += size_t(4) * K * segcap * sizeof(double);       // zone cache + histories
    b += size_t(segcap) * sizeof(int2);
    b += size_t(MWW + 1) * sizeof(uint64_t);            // mask words, mbarrier
    return b;
  }
};

// same[lev] = 1 when level lev has the mask of level lev-1 (caller presets 1)
__global__ void k_mask_same(const uint8_t* __restrict__ mask, int64_t nh, int64_t nlev,
                            uint8_t* __restrict__ same) {
  const int64_t total = nh * (nlev - 1);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lev = 1 + q / nh;
    if ((mask[q + nh] != 0) != (mask[q] != 0)) same[lev] = 0;
  }
}

__device__ __forceinline__ void rf1l_cp_async(void* dst, const void* src, int bytes) {
  if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

template <typename T, bool TR, int NT, int V, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_rf1_row(const T* __restrict__ in, T* __restrict__ out,
                                                      Rf1RowArgs a) {
  using L = Rf1RowSmem<NT, V>;
  constexpr int CAP = L::CAP, MWW = L::MWW, NW = L::NW;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int K = a.k, segcap = a.segcap;
  double* const sd = reinterpret_cast<double*>(smraw);  // exchange line; output staging
  T* const stg = reinterpret_cast<T*>(sd + CAP);        // input staging (next plane's row)
  double* const wtA = sd + 2 * CAP;
  double* const wtB = wtA + NW;
  double* const zc = wtB + NW;                         // [2K][segcap]
  double* const hist = zc + size_t(2) * K * segcap;    // [2K][segcap]
  int2* const sseg = reinterpret_cast<int2*>(hist + size_t(2) * K * segcap);
  uint64_t* const mw = reinterpret_cast<uint64_t*>(sseg + segcap);
  uint64_t* const bar = mw + MWW;

  const int n = a.n, nl = a.nl;
  const int64_t nh = int64_t(n) * nl;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t groups = (planes + a.planes_per_cta - 1) / a.planes_per_cta;
  const int64_t line = blockIdx.x / groups, grp = blockIdx.x - line * groups;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p0 = tid * V;
  const uint32_t sdb = smem_u32(sd + p0);  // this thread's chunk in the exchange line
  constexpr uint64_t VM = (1ull << V) - 1ull;
  const uint32_t rowbytes = static_cast<uint32_t>(n) * sizeof(T);
  // bulk (TMA) row copies need 16 B aligned rows
  const bool bulk = (rowbytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(in) |
                                               reinterpret_cast<uintptr_t>(out)) % 16 == 0);

  const int64_t pl_begin = grp * a.planes_per_cta;
  const int64_t pl_end = pl_begin + a.planes_per_cta < planes ? pl_begin + a.planes_per_cta : planes;

  auto fetch = [&](int64_t pl) {  // start the row of plane pl towards the staging buffer
    const T* src = in + pl * nh + line * n;
    if (bulk) {
      if (tid == 0) {
        mbar_arrive_expect_tx(bar, rowbytes);
        bulk_g2s(stg, src, rowbytes, bar);
      }
    } else {
#pragma unroll
      for (int u = 0; u < V; ++u) {
        const int i = tid + u * NT;
        if (i < n) rf1l_cp_async(stg + i, src + i, sizeof(T));
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
  };
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  fetch(pl_begin);

  uint32_t live = 0, starts = 0, ends = 0, slotL = 0, slotR = 0, seab = 0;
  double la[V];
  double A = 1.0;
  int nseg = 0;
  uint32_t phase = 0;
  for (int64_t pl = pl_begin; pl < pl_end; ++pl) {
    const int64_t var = pl / a.nlev, lev = a.lev0 + (pl - var * a.nlev);
    const bool reuse = pl > pl_begin && pl - var * a.nlev > 0 && a.same[lev];
    if (!reuse) {
      // ---- chunk masks and links, mask words, segments and zone responses
      const uint64_t* Wl = a.bits + (lev * nl + line) * a.words;
      const int G = a.ghost[lev];
      const uint64_t win =
          p0 > 0 ? rf1l_window(Wl, a.words, p0 - 1) : (rf1l_window(Wl, a.words, 0) << 1);
      const uint64_t sea = (win >> 1) & VM, prv = win & VM, nxt = (win >> 2) & VM;
      const uint64_t frozen = G == 0 ? (sea & ~prv & ~nxt) : 0ull;  // covariance.cpp:260-269
      seab = static_cast<uint32_t>(sea);
      live = static_cast<uint32_t>(sea & ~frozen);
      starts = static_cast<uint32_t>(sea & ~prv);
      ends = static_cast<uint32_t>(sea & ~nxt);
      slotL = static_cast<uint32_t>(~sea & nxt & VM);  // land before a segment start
      // land after a segment end; none past the line (a segment ending at the
      // last point has no right ghosts, and nothing places a value there)
      const int inl = n - p0;
      const uint64_t inm = inl >= V ? VM : (inl > 0 ? (1ull << inl) - 1ull : 0ull);
      slotR = static_cast<uint32_t>(~sea & prv & inm);
      {
        const double* cp = reinterpret_cast<const double*>(a.c1 + line * a.csl + p0 * a.csp);
        const int64_t cst = 2 * a.csp;
#pragma unroll
        for (int i = 0; i < V; ++i) {
          double al = 0.0;
          if ((live >> i) & 1u) al = __ldg(cp + i * cst);
          la[i] = al;
        }
      }
      A = 1.0;
#pragma unroll
      for (int i = 0; i < V; ++i) A *= la[i];
      for (int w = tid; w < MWW; w += NT) mw[w] = w < a.words ? ldw(Wl, w) : 0ull;
      const int64_t sb0 = a.seg_off[lev * nl + line];
      nseg = static_cast<int>(a.seg_off[lev * nl + line + 1] - sb0);
      for (int s = tid; s < nseg; s += NT) {
        sseg[s] = a.segs[sb0 + s];
        for (int d = 0; d < 2 * K; ++d) zc[d * segcap + s] = __ldg(a.zone + d * a.nsegs + sb0 + s);
      }
    }

    // ---- this plane's row: staging -> registers (land = 0, adjoint input scaling)
    if (bulk) {
      mbar_wait(bar, phase);
      phase ^= 1u;
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    double v[V];
    {
      const double* pre = (TR && a.pre_scale) ? a.pre_scale + lev * nh + line * n + p0 : nullptr;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        double x = static_cast<double>(stg[p0 + i]);
        if (TR) {
          if (pre && ((seab >> i) & 1u)) x *= __ldg(pre + i);
        }
        v[i] = ((seab >> i) & 1u) ? x : 0.0;
      }
    }
    __syncthreads();  // the staging buffer is free
    if (pl + 1 < pl_end) fetch(pl + 1);
    // the previous plane's bulk store must have read the exchange line before
    // this plane's first exit is published (after the first pass's barrier)
    if (bulk && tid == 0) bulk_wait_read_all();

    // ---- one pass
    auto pass = [&](auto asc_c, auto first_c, auto last_c, auto pull_c) {
      constexpr bool ASC = decltype(asc_c)::value;
      constexpr bool FIRST = decltype(first_c)::value;  // adjoint: raw input
      constexpr bool LAST = decltype(last_c)::value;    // adjoint: b_i on the output
      constexpr bool PULL = decltype(pull_c)::value;    // entries were placed for this pass
      const uint32_t slots = ASC ? slotL : slotR;       // land slots holding this pass's entries
      const uint32_t exits = ASC ? ends : starts;       // states handed to the zones
      double r = 0.0;
#pragma unroll
      for (int ii = 0; ii < V; ++ii) {
        const int i = ASC ? ii : V - 1 - ii;
        if constexpr (PULL) rf1l_lds_if(v[i], sdb + 8u * i, slots & (1u << i));
        double t;
        if constexpr (!TR) {
          t = fma(-la[i], v[i], v[i]);  // b_i s_i with b = 1 - a; a land slot keeps its value
        } else {
          const double w = FIRST ? v[i] : fma(-la[i], v[i], v[i]);
          t = ((live >> i) & 1u) ? la[i] * w : v[i];
        }
        r = fma(la[i], r, t);
      }
      // inclusive scan of (A, r) over the warp's lanes in pass order
      const int pos = ASC ? lane : 31 - lane;
      double ar = A, br = r;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double ua = ASC ? __shfl_up_sync(0xffffffffu, ar, d) : __shfl_down_sync(0xffffffffu, ar, d);
        const double ub = ASC ? __shfl_up_sync(0xffffffffu, br, d) : __shfl_down_sync(0xffffffffu, br, d);
        if (pos >= d) {
          br = fma(ar, ub, br);
          ar *= ua;
        }
      }
      double ae = ASC ? __shfl_up_sync(0xffffffffu, ar, 1) : __shfl_down_sync(0xffffffffu, ar, 1);
      double be = ASC ? __shfl_up_sync(0xffffffffu, br, 1) : __shfl_down_sync(0xffffffffu, br, 1);
      if (pos == 0) {
        ae = 1.0;
        be = 0.0;
      }
      if (pos == 31) {
        wtA[warp] = ar;
        wtB[warp] = br;
      }
      __syncthreads();
      double cw = 0.0;  // state entering this warp: fold the totals of the warps before it
#pragma unroll
      for (int k2 = 0; k2 < NW; ++k2) {
        const int w2 = ASC ? k2 : NW - 1 - k2;
        const double ta = wtA[w2], tb = wtB[w2];
        if (ASC ? w2 < warp : w2 > warp) cw = fma(ta, cw, tb);
      }
      r = fma(ae, cw, be);
#pragma unroll
      for (int ii = 0; ii < V; ++ii) {
        const int i = ASC ? ii : V - 1 - ii;
        if constexpr (!TR) {
          r = fma(la[i], r, fma(-la[i], v[i], v[i]));
          v[i] = r;
          rf1l_sts_if(sdb + 8u * i, r, exits & (1u << i));
        } else {
          const bool on = (live >> i) & 1u;
          const double w = FIRST ? v[i] : fma(-la[i], v[i], v[i]);
          const double cur = w + r;  // cur_i = w_i + a_{i-1} cur_{i-1}
          r = fma(la[i], r, on ? la[i] * w : v[i]);
          if (on) v[i] = LAST ? fma(-la[i], cur, cur) : cur;
          rf1l_sts_if(sdb + 8u * i, cur, exits & (1u << i));
        }
      }
      __syncthreads();
    };

    // ---- between passes: record exits, place the next entries
    auto boundary = [&](bool after_asc, int it) {
      for (int s = tid; s < nseg; s += NT) {
        const int2 sg = sseg[s];
        const int i0 = sg.x, j0 = sg.x + sg.y - 1;
        if (after_asc) {
          hist[(K + it - 1) * segcap + s] = sd[j0];
          if (j0 < n - 1) {
            double e = 0.0;
            for (int j = 1; j <= it; ++j)
              e = fma(zc[(K + it - j) * segcap + s], hist[(K + j - 1) * segcap + s], e);
            if (TR) e *= __ldg(&a.c1[line * a.csl + j0 * a.csp].x);
            sd[j0 + 1] = e;
          }
        } else {
          hist[(it - 1) * segcap + s] = sd[i0];
          if (i0 > 0) {
            double e = 0.0;
            for (int j = 1; j <= it; ++j) e = fma(zc[(it + 1 - j) * segcap + s], hist[(j - 1) * segcap + s], e);
            if (TR) e *= __ldg(&a.c1[line * a.csl + i0 * a.csp].x);
            sd[i0 - 1] = e;
          }
        }
      }
      __syncthreads();
    };

    using Tt = std::true_type;
    using Ft = std::false_type;
    for (int it = 1; it <= K; ++it) {
      // iteration 1 enters every segment from zero: no entries to pull
      if (it == 1) pass(Tt{}, std::integral_constant<bool, TR>{}, Ft{}, Ft{});
      else pass(Tt{}, Ft{}, Ft{}, Tt{});
      boundary(true, it);
      if (TR && it == K) pass(Ft{}, Ft{}, Tt{}, Tt{}); else pass(Ft{}, Ft{}, Ft{}, Tt{});
      if (it < K) boundary(false, it);
    }

    // ---- publish the chunks (land exactly 0, output scaling) and store the row
    {
      T* const ost = reinterpret_cast<T*>(sd);
      const double* post = a.post_scale ? a.post_scale + lev * nh + line * n + p0 : nullptr;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        double o = ((seab >> i) & 1u) ? v[i] : 0.0;
        if (post && ((seab >> i) & 1u)) o *= __ldg(post + i);
        ost[p0 + i] = static_cast<T>(o);
      }
      T* dst = out + pl * nh + line * n;
      if (bulk) {
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
          bulk_s2g(dst, ost, rowbytes);
          bulk_commit();
        }
      } else {
        __syncthreads();
#pragma unroll
        for (int u = 0; u < V; ++u) {
          const int i = tid + u * NT;
          if (i < n) dst[i] = ost[i];
        }
        __syncthreads();  // the next plane's passes write the exchange line
      }
    }
  }
  if (bulk && tid == 0) bulk_wait_all();
}

template <typename T, bool TR, int NT, int V, int MINB>
bool rf1_row_launch_shape(const T* in, T* out, const Rf1RowArgs& a, cudaStream_t st) {
  using L = Rf1RowSmem<NT, V>;
  const size_t smem = L::bytes(a.k, a.segcap);
  if (smem > 227 * 1024 / MINB) return false;
  auto kern = k_rf1_row<T, TR, NT, V, MINB>;
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess)
      return false;
    attr = smem;
  }
  const int64_t planes = a.nvar * a.nlev;
  const int64_t groups = (planes + a.planes_per_cta - 1) / a.planes_per_cta;
  kern<<<static_cast<unsigned>(int64_t(a.nl) * groups), NT, smem, st>>>(in, out, a);
  return true;
}

// rows of up to 8704 points; false: the caller falls back
template <typename T, bool TR>
bool launch_rf1_row_tr(const T* in, T* out, Rf1RowArgs a, cudaStream_t st) {
  const int64_t planes = a.nvar * a.nlev;
  int ppc = static_cast<int>(std::max<int64_t>(1, int64_t(a.nl) * planes / (148 * 4 * 4)));
  a.planes_per_cta = static_cast<int>(std::min<int64_t>(std::min<int64_t>(ppc, 16), planes));
  if (a.n <= 128 * 9) return rf1_row_launch_shape<T, TR, 128, 9, 4>(in, out, a, st);
  if (a.n <= 128 * 17) return rf1_row_launch_shape<T, TR, 128, 17, 4>(in, out, a, st);
  if (a.n <= 256 * 17) return rf1_row_launch_shape<T, TR, 256, 17, 2>(in, out, a, st);
  if (a.n <= 512 * 17) return rf1_row_launch_shape<T, TR, 512, 17, 1>(in, out, a, st);
  return false;
}
template <typename T>
bool launch_rf1_row(const T* in, T* out, const Rf1RowArgs& a, cudaStream_t st) {
  return a.transpose ? launch_rf1_row_tr<T, true>(in, out, a, st)
                     : launch_rf1_row_tr<T, false>(in, out, a, st);
}

// ------------------------------------------------------------- launcher
// shapes: x lines NT=128 (4 CTAs/SM), y tiles of 64 B rows NT=512 (1 CTA/SM)
template <typename T, typename S, bool TR, int NT, int V, int C, int MINB>
bool rf1_line_launch_shape(const T* in, T* out, const Rf1LineArgs& a, cudaStream_t st) {
  using L = Rf1LineSmem<S, NT, V, C>;
  const size_t smem = L::bytes(a.k, a.segcap);
  if (smem > 227 * 1024) return false;
  auto kern = k_rf1_line<T, S, TR, NT, V, C, MINB>;
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess)
      return false;
    attr = smem;
  }
  const int64_t nl = a.dir == 0 ? a.ny : a.nx;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t tiles = (nl + C - 1) / C;
  const int64_t groups = (planes + a.planes_per_cta - 1) / a.planes_per_cta;
  kern<<<static_cast<unsigned>(tiles * groups), NT, smem, st>>>(in, out, a);
  return true;
}

template <typename T, typename S, bool TR, int NT, int C, int MINB>
bool rf1_line_launch_v(const T* in, T* out, const Rf1LineArgs& a, cudaStream_t st) {
  const int64_t n = a.dir == 0 ? a.nx : a.ny;
  constexpr int NQ = NT / C;
  if (n <= int64_t(NQ) * 7) return rf1_line_launch_shape<T, S, TR, NT, 7, C, MINB>(in, out, a, st);
  if (n <= int64_t(NQ) * 9) return rf1_line_launch_shape<T, S, TR, NT, 9, C, MINB>(in, out, a, st);
  if (n <= int64_t(NQ) * 17) return rf1_line_launch_shape<T, S, TR, NT, 17, C, MINB>(in, out, a, st);
  if (n <= int64_t(NQ) * 35) return rf1_line_launch_shape<T, S, TR, NT, 35, C, MINB>(in, out, a, st);
  return false;
}

// One sweep (all K iterations) of direction a.dir; false when the line does
// not fit the resident shapes (the caller falls back to the streaming passes).
template <typename T>
bool launch_rf1_line(const T* in, T* out, Rf1LineArgs a, cudaStream_t st) {
  const int64_t planes = a.nvar * a.nlev;
  if (a.dir == 0 && a.nx <= 512 * 17) {
    Rf1RowArgs r{};
    r.transpose = a.transpose;
    r.k = a.k;
    r.n = static_cast<int>(a.nx);
    r.nl = static_cast<int>(a.ny);
    r.nlev = a.nlev;
    r.nvar = a.nvar;
    r.lev0 = a.lev0;
    r.c1 = a.c1;
    r.csp = 1;
    r.csl = a.nx;
    r.bits = a.bits;
    r.words = a.words;
    r.seg_off = a.seg_off;
    r.segs = a.segs;
    r.nsegs = a.nsegs;
    r.zone = a.zone;
    r.ghost = a.ghost;
    r.same = a.same;
    r.pre_scale = a.pre_scale;
    r.post_scale = a.post_scale;
    r.segcap = a.segcap;
    if (launch_rf1_row<T>(in, out, r, st)) return true;
  }
  if (a.dir == 0) {
    const int64_t nl = a.ny;
    // enough CTAs for ~4 waves of 148 x 4
    int ppc = static_cast<int>(std::max<int64_t>(1, nl * planes / (148 * 4 * 4)));
    a.planes_per_cta = static_cast<int>(std::min<int64_t>(std::min<int64_t>(ppc, 16), planes));
    if (a.transpose) return rf1_line_launch_v<T, double, true, 128, 1, 4>(in, out, a, st);
    return rf1_line_launch_v<T, double, false, 128, 1, 4>(in, out, a, st);
  }
  constexpr int CY = 8;  // columns per tile: 64 B (fp64) / 32 B (fp32) row pieces
  const int64_t tiles = (a.nx + CY - 1) / CY;
  int ppc = static_cast<int>(std::max<int64_t>(1, tiles * planes / (148 * 4)));
  a.planes_per_cta = static_cast<int>(std::min<int64_t>(std::min<int64_t>(ppc, 8), planes));
  if (a.transpose) return rf1_line_launch_v<T, T, true, 512, CY, 1>(in, out, a, st);
  return rf1_line_launch_v<T, T, false, 512, CY, 1>(in, out, a, st);
}

}  // namespace rgfb
