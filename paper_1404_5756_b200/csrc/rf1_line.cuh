// Line-resident 1st-RF: all K iterations of one sweep in ONE field pass.
//
// Reference (rf1.hpp:20-63, 113-137; covariance.cpp:283-286, 319-322,
// 334-339): K x {forward, backward} (adjoint: K x {backward-transpose,
// forward-transpose}) over every sea segment extended by G ghosts per side.
// The streaming form (rf1_stream.cuh) runs each of the 2K passes as its own
// kernel: 4K field moves per sweep. Here a CTA keeps whole lines (x: one row
// of a plane; y: C adjacent columns of a plane) on chip for all 2K passes,
// and each pass is a PARALLEL SCAN along the line instead of a serial walk,
// so a line needs no other chains to hide the recursion latency: one read
// and one write of the field per sweep.
//
//   * A first-order pass r_i = l_i r_{i-1} + t_i composes as affine maps
//     (A, B) -> (A' A, A' B + B'). Thread (q, c) keeps V consecutive points of
//     line c and their links in REGISTERS: it runs the recursion over its
//     chunk from a zero state (B; the chunk's link product A = prod l_i is
//     fixed per line), the chunk aggregates are scanned with warp shuffles and
//     the warp totals folded through shared memory, and the thread re-runs
//     its chunk from the true carry.
//   * Links l_i are alpha_i at sea points and 0 on land, so land cuts the
//     chain and a land point keeps its stored value. That makes land points
//     free storage: the ghost-zone entry state of the coming pass (E_L before
//     a segment start for ascending passes, E_R after a segment end for
//     descending ones; rf1_stream.cuh explains the zone algebra) is PLACED in
//     the adjacent land slot, and the uniform recursion picks it up as the
//     previous state. No per-point segment logic in the passes.
//   * Shared memory holds an exchange copy of the line that is touched only
//     where a value changes hands: a segment's exit point is published
//     (predicated store), one thread per segment takes it (x_it at the start,
//     y_it at the end), adds its zone response to the pending entries of the
//     coming iterations and places the next entry, and the owner of that land
//     slot pulls it (predicated load) at the start of the next pass.
//   * The adjoint passes cur_i = w_i + a_{i-1} cur_{i-1}, out = b_i cur_i
//     run on z_i = a_i cur_i (z_i = a_i z_{i-1} + a_i w_i: the same links),
//     with cur_i = w_i + z_{i-1} stored and the b_i factor applied to the
//     next pass's input (and to the final output).
//   * Rows move by bulk async copies (TMA, x sweeps with 16 B aligned rows)
//     or cp.async pieces; the next plane's lines are in flight during the
//     passes, and masks/links/zone tables are reused across consecutive
//     levels that share a mask.
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
  int tma;                  // y tiles move by tensor copies (maps valid)
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


template <int NT, int V, int C>
struct Rf1ResSmem {
  static constexpr int NQ = NT / C;     // chunks per line
  static constexpr int CAP = NQ * V;    // points per line held
  static constexpr int NW = NT / 32;
  static size_t bytes(int K, int segcap) {
    size_t b = size_t(2) * CAP * C * sizeof(double);    // exchange lines + input staging
    b += size_t(2) * NW * C * sizeof(double);           // warp totals
    b += size_t(4) * K * C * segcap * sizeof(double);   // zone cache + pending entries
    b += size_t(2) * C * segcap * sizeof(double);       // alpha at segment starts / ends
    b += size_t(C) * segcap * sizeof(int2);
    b += size_t(C) * sizeof(int) + 16;                  // segments per line, mbarrier
    return b;
  }
};

// One CTA: C adjacent lines (x sweeps: C = 1 row; y sweeps: C columns) of
// `planes_per_cta` planes, one plane at a time. Thread t = q*C + c keeps
// points [q*V, q*V + V) of line c in registers.
template <typename T, bool TR, int NT, int V, int C, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_rf1_res(const T* __restrict__ in, T* __restrict__ out,
                                                      Rf1LineArgs a,
                                                      const __grid_constant__ CUtensorMap tm_in,
                                                      const __grid_constant__ CUtensorMap tm_out) {
  using L = Rf1ResSmem<NT, V, C>;
  constexpr int CAP = L::CAP, NW = L::NW;
  constexpr int QW = 32 / C;          // chunks of one line per warp
  constexpr bool XD = C == 1;         // lines are rows of the field
  static_assert(32 % C == 0 && V <= 30, "shape");
  extern __shared__ __align__(128) unsigned char smraw[];
  const int K = a.k, segcap = a.segcap;
  double* const sd = reinterpret_cast<double*>(smraw);  // exchange lines [p][C]; output staging
  T* const stg = reinterpret_cast<T*>(sd + CAP * C);    // input staging [p][C] (next plane)
  double* const wtA = sd + 2 * CAP * C;                 // [NW][C]
  double* const wtB = wtA + NW * C;
  double* const zc = wtB + NW * C;                          // [2K][C*segcap]
  double* const acc = zc + size_t(2) * K * C * segcap;      // [2K][C*segcap]: pending entries
  double* const salpha = acc + size_t(2) * K * C * segcap;  // [2][C*segcap]: alpha at start / end
  int2* const sseg = reinterpret_cast<int2*>(salpha + size_t(2) * C * segcap);  // [C][segcap]
  int* const scnt = reinterpret_cast<int*>(sseg + size_t(C) * segcap);
  uint64_t* const bar = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(scnt + C) + 7) & ~uintptr_t(7));

  const int n = static_cast<int>(XD ? a.nx : a.ny);    // points per line
  const int nl = static_cast<int>(XD ? a.ny : a.nx);   // lines per level
  const int64_t nh = int64_t(n) * nl;
  const int64_t gsp = XD ? 1 : nl, gsl = XD ? n : 1;   // field/coefficient strides (point, line)
  const int64_t planes = a.nvar * a.nlev;
  const int64_t groups = (planes + a.planes_per_cta - 1) / a.planes_per_cta;
  // y tiles come in cluster pairs: the two CTAs of a cluster own neighbouring
  // tiles (in fp64 the two halves of each 32 B sector) and keep step plane by
  // plane, so their loads and stores of a sector meet in L2. (fp32: clusters
  // of four covering a sector measured slower, 16.4 vs 15.7 ms per C5 y sweep.)
  constexpr int CL = C > 1 ? 2 : 1;
  const int64_t unit = blockIdx.x / CL;
  const int64_t upos = unit / groups, grp = unit - upos * groups;
  const int64_t tile = CL * upos + (blockIdx.x % CL);
  const int line0 = static_cast<int>(tile) * C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = tid % C, q = tid / C;
  const int line = line0 + c;
  const bool lineok = line < nl;
  const int p0 = q * V;
  const uint32_t sdb = smem_u32(sd + p0 * C + c);  // this thread's chunk in the exchange lines
  constexpr uint32_t SST = 8u * C;                 // byte stride between its points
  constexpr uint64_t VM = (1ull << V) - 1ull;
  const uint32_t rowbytes = static_cast<uint32_t>(n) * sizeof(T);
  // x sweeps: bulk (TMA) row copies need 16 B aligned rows. y sweeps: 16 B
  // cp.async pieces / vector stores need aligned full tiles.
  const bool al16 = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) % 16 == 0);
  const bool bulk = XD && al16 && rowbytes % 16 == 0;
  constexpr int EPP = 16 / int(sizeof(T));  // elements per 16 B piece
  const bool vec = !XD && al16 && (C % EPP == 0) && (int64_t(nl) * sizeof(T)) % 16 == 0 &&
                   line0 + C <= nl;
  // fp32 tiles of two columns: one 8 B piece per row
  const bool vec8 = !XD && sizeof(T) == 4 && C == 2 && nl % 2 == 0 && line0 + C <= nl &&
                    ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) % 8 == 0);

  // y tiles as tensor copies: boxes of NQ rows x C columns (one thread issues them)
  const bool tma = !XD && a.tma != 0;
  constexpr int BR = L::NQ;
  const int nbox = (n + BR - 1) / BR;
  const bool abar = bulk || tma;  // arrivals counted on the mbarrier

  const int64_t pl_begin = grp * a.planes_per_cta;
  const int64_t pl_end = pl_begin + a.planes_per_cta < planes ? pl_begin + a.planes_per_cta : planes;

  auto fetch = [&](int64_t pl) {  // start the lines of plane pl towards the staging buffer
    const T* src = in + pl * nh + line0 * gsl;
    if (bulk) {
      if (tid == 0) {
        mbar_arrive_expect_tx(bar, rowbytes);
        bulk_g2s(stg, src, rowbytes, bar);
      }
      return;
    }
    if (tma) {
      if (tid == 0) {
        const uint64_t pol = l2_evict_normal();
        mbar_arrive_expect_tx(bar, static_cast<uint32_t>(nbox) * BR * C * sizeof(T));
        for (int b = 0; b < nbox; ++b)
          tma_load_3d(stg + b * BR * C, &tm_in, line0, b * BR, static_cast<int>(pl), bar, pol);
      }
      return;
    }
    if (vec) {
      constexpr int PPR = (C + EPP - 1) / EPP;  // 16 B pieces per staged row
      for (int e = tid; e < n * PPR; e += NT) {
        const int p = e / PPR, k = e - p * PPR;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(stg + p * C + k * EPP)),
                     "l"(src + p * gsp + k * EPP)
                     : "memory");
      }
    } else if (vec8) {
      for (int p = tid; p < n; p += NT) rf1l_cp_async(stg + p * C, src + p * gsp, 8);
    } else {
      for (int e = tid; e < n * C; e += NT) {
        const int p = e / C, cc = e - p * C;
        if (line0 + cc < nl) rf1l_cp_async(stg + e, src + p * gsp + cc * gsl, sizeof(T));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  fetch(pl_begin);

  uint32_t live = 0, starts = 0, ends = 0, slotL = 0, slotR = 0, seab = 0;
  double la[V];
  double A = 1.0;  // the chunk's link product
  int my_i0 = 0, my_j0 = -1;
  uint32_t phase = 0;
  for (int64_t pl = pl_begin; pl < pl_end; ++pl) {
    const int64_t var = pl / a.nlev, lev = a.lev0 + (pl - var * a.nlev);
    const bool reuse = pl > pl_begin && pl - var * a.nlev > 0 && a.same[lev];
    if (!reuse) {
      // ---- chunk masks and links, segments and zone responses
      uint64_t win = 0;
      if (lineok) {
        const uint64_t* Wl = a.bits + (lev * nl + line) * a.words;
        win = p0 > 0 ? rf1l_window(Wl, a.words, p0 - 1) : (rf1l_window(Wl, a.words, 0) << 1);
      }
      const int G = a.ghost[lev];
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
        const double* cp =
            reinterpret_cast<const double*>(a.c1 + (lineok ? line * gsl + p0 * gsp : 0));
        const int64_t cst = 2 * gsp;
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
      for (int cc = 0; cc < C; ++cc) {
        if (line0 + cc >= nl) {
          if (tid == 0) scnt[cc] = 0;
          continue;
        }
        const int64_t sb0 = a.seg_off[lev * nl + line0 + cc];
        const int ns = static_cast<int>(a.seg_off[lev * nl + line0 + cc + 1] - sb0);
        if (tid == 0) scnt[cc] = ns;
        for (int s = tid; s < ns; s += NT) {
          const int2 sg = a.segs[sb0 + s];
          sseg[cc * segcap + s] = sg;
          for (int d = 0; d < 2 * K; ++d)
            zc[(d * C + cc) * segcap + s] = __ldg(a.zone + d * a.nsegs + sb0 + s);
          if (TR) {  // the adjoint's entries are scaled by the end point's alpha
            const double2* cl = a.c1 + (line0 + cc) * gsl;
            salpha[cc * segcap + s] = __ldg(&cl[sg.x * gsp].x);
            salpha[C * segcap + cc * segcap + s] = __ldg(&cl[(sg.x + sg.y - 1) * gsp].x);
          }
        }
      }
    }

    // ---- this plane's lines: staging -> registers (land = 0, adjoint input scaling)
    if (abar) {
      mbar_wait(bar, phase);
      phase ^= 1u;
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    if (!reuse) {  // this thread's first segment of the between-pass phase
      my_j0 = -1;
      if (tid < C * segcap) {
        const int cc = tid / segcap, sgi = tid - cc * segcap;
        if (sgi < scnt[cc]) {
          const int2 sg = sseg[tid];
          my_i0 = sg.x;
          my_j0 = sg.x + sg.y - 1;
        }
      }
    }
    double v[V];
    {
      const double* pre =
          (TR && a.pre_scale && lineok) ? a.pre_scale + lev * nh + line * gsl + p0 * gsp : nullptr;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        double x = static_cast<double>(stg[(p0 + i) * C + c]);
        if (TR) {
          if (pre && ((seab >> i) & 1u)) x *= __ldg(pre + i * gsp);
        }
        v[i] = ((seab >> i) & 1u) ? x : 0.0;
      }
    }
    __syncthreads();  // the staging buffer is free
    if constexpr (C > 1) {  // re-align the pair every 8th plane (every plane: +5 % time, same traffic)
      if (((pl - pl_begin) & 7) == 0)
        asm volatile(
            "barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;\n" ::
                : "memory");
    }
    if (pl + 1 < pl_end) fetch(pl + 1);
    // the previous plane's bulk store must have read the exchange line before
    // this plane's first exit is published (after the first pass's barrier)
    if (abar && tid == 0) bulk_wait_read_all();

    // ---- one pass
    auto pass = [&](auto asc_c, auto first_c, auto last_c, auto pull_c) {
      constexpr bool ASC = decltype(asc_c)::value;
      constexpr bool FIRST = decltype(first_c)::value;  // adjoint: raw input
      constexpr bool LAST = decltype(last_c)::value;    // adjoint: b_i on the output
      constexpr bool PULL = decltype(pull_c)::value;    // entries were placed for this pass
      const uint32_t slots = ASC ? slotL : slotR;       // land slots holding this pass's entries
      const uint32_t exits = ASC ? ends : starts;       // states handed to the zones
      // input term of point i (and, adjoint, its input w_i). `again`: second
      // walk of the pass (a forward value pulled in the first walk is kept)
      auto term = [&](int i, double& w, bool again) -> double {
        if constexpr (!TR) {
          if (PULL && !again) rf1l_lds_if(v[i], sdb + SST * i, slots & (1u << i));
          w = 0.0;
          return fma(-la[i], v[i], v[i]);  // b_i s_i with b = 1 - a; a land slot keeps its value
        } else {
          double e = 0.0;  // entry placed in this land slot (z-type: a_s E)
          if constexpr (PULL) rf1l_lds_if(e, sdb + SST * i, slots & (1u << i));
          w = FIRST ? v[i] : fma(-la[i], v[i], v[i]);
          return fma(la[i], w, e);
        }
      };
      double r = 0.0, wdummy;
#pragma unroll
      for (int ii = 0; ii < V; ++ii) {
        const int i = ASC ? ii : V - 1 - ii;
        r = fma(la[i], r, term(i, wdummy, false));
      }
      // inclusive scan of (A, r) over the line's chunks in this warp, in pass order
      const int pos = ASC ? lane / C : QW - 1 - lane / C;
      double ar = A, br = r;
#pragma unroll
      for (int d = 1; d < QW; d <<= 1) {
        const double ua = ASC ? __shfl_up_sync(0xffffffffu, ar, d * C) : __shfl_down_sync(0xffffffffu, ar, d * C);
        const double ub = ASC ? __shfl_up_sync(0xffffffffu, br, d * C) : __shfl_down_sync(0xffffffffu, br, d * C);
        if (pos >= d) {
          br = fma(ar, ub, br);
          ar *= ua;
        }
      }
      double ae = ASC ? __shfl_up_sync(0xffffffffu, ar, C) : __shfl_down_sync(0xffffffffu, ar, C);
      double be = ASC ? __shfl_up_sync(0xffffffffu, br, C) : __shfl_down_sync(0xffffffffu, br, C);
      if (pos == 0) {
        ae = 1.0;
        be = 0.0;
      }
      if (pos == QW - 1) {
        wtA[warp * C + c] = ar;
        wtB[warp * C + c] = br;
      }
      __syncthreads();
      double cw = 0.0;  // state entering this warp: fold the totals of the warps before it
#pragma unroll
      for (int k2 = 0; k2 < NW; ++k2) {
        const int w2 = ASC ? k2 : NW - 1 - k2;
        const double ta = wtA[w2 * C + c], tb = wtB[w2 * C + c];
        if (ASC ? w2 < warp : w2 > warp) cw = fma(ta, cw, tb);
      }
      r = fma(ae, cw, be);  // state entering the chunk
#pragma unroll
      for (int ii = 0; ii < V; ++ii) {
        const int i = ASC ? ii : V - 1 - ii;
        double w;
        const double t = term(i, w, true);
        if constexpr (!TR) {
          r = fma(la[i], r, t);
          v[i] = r;
          rf1l_sts_if(sdb + SST * i, r, exits & (1u << i));
        } else {
          const double cur = w + r;  // cur_i = w_i + a_{i-1} cur_{i-1}
          r = fma(la[i], r, t);
          // land values are never read back into sea points (their link is 0)
          v[i] = LAST ? fma(-la[i], cur, cur) : cur;
          rf1l_sts_if(sdb + SST * i, cur, exits & (1u << i));
        }
      }
      __syncthreads();
    };

    // ---- between passes: one thread per segment takes the state handed to
    // the zone (y_it at the end after an ascending pass, x_it at the start
    // after a descending one), adds its response to the entries of the coming
    // iterations (independent FMAs; each entry sums its terms in iteration
    // order, as rf1_entry_left/right do), and places the entry of the next
    // pass in the land slot. (Doing this in the thread that owns the exit
    // point saves the barrier before it but costs 15 % more instructions in
    // divergent warps: measured equal, 2.06 / 3.06 ms per 20-level x / y sweep.)
    auto boundary = [&](bool after_asc, int it) {
      const int SC = C * segcap;
      auto serve = [&](int w, int cc, int i0, int j0) {
        if (after_asc) {  // entries E_R(k), k = it..K, live in acc[K + k - 1]
          const double y = sd[j0 * C + cc];
          double e = 0.0;
          for (int k = it; k <= K; ++k) {
            const double prev = it == 1 ? 0.0 : acc[(K + k - 1) * SC + w];
            const double nv = fma(zc[(K + k - it) * SC + w], y, prev);
            if (k == it) e = nv; else acc[(K + k - 1) * SC + w] = nv;
          }
          if (j0 < n - 1) sd[(j0 + 1) * C + cc] = TR ? e * salpha[SC + w] : e;
        } else {          // entries E_L(k), k = it+1..K, live in acc[k - 1]
          const double x = sd[i0 * C + cc];
          double e = 0.0;
          for (int k = it + 1; k <= K; ++k) {
            const double prev = it == 1 ? 0.0 : acc[(k - 1) * SC + w];
            const double nv = fma(zc[(k - it) * SC + w], x, prev);
            if (k == it + 1) e = nv; else acc[(k - 1) * SC + w] = nv;
          }
          if (i0 > 0) sd[(i0 - 1) * C + cc] = TR ? e * salpha[w] : e;
        }
      };
      // the thread's first segment sits in registers (no lookups on the
      // latency path between the two barriers); further ones come from the list
      if (my_j0 >= 0) serve(tid, tid / segcap, my_i0, my_j0);
      for (int w = tid + NT; w < SC; w += NT) {
        const int cc = w / segcap, s = w - cc * segcap;
        if (s >= scnt[cc]) continue;
        const int2 sg = sseg[w];
        serve(w, cc, sg.x, sg.x + sg.y - 1);
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

    // ---- publish the chunks (land exactly 0, output scaling) and store the lines
    {
      T* const ost = reinterpret_cast<T*>(sd);
      const double* post =
          (a.post_scale && lineok) ? a.post_scale + lev * nh + line * gsl + p0 * gsp : nullptr;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        double o = ((seab >> i) & 1u) ? v[i] : 0.0;
        if (post && ((seab >> i) & 1u)) o *= __ldg(post + i * gsp);
        ost[(p0 + i) * C + c] = static_cast<T>(o);
      }
      T* dst = out + pl * nh + line0 * gsl;
      if (bulk) {
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
          bulk_s2g(dst, ost, rowbytes);
          bulk_commit();
        }
      } else if (tma) {
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
          const uint64_t pol = l2_evict_normal();
          for (int b = 0; b < nbox; ++b)
            tma_store_3d(&tm_out, line0, b * BR, static_cast<int>(pl), ost + b * BR * C, pol);
          bulk_commit();
        }
      } else {
        __syncthreads();
        if (vec) {
          constexpr int PPR = (C + EPP - 1) / EPP;
          for (int e = tid; e < n * PPR; e += NT) {
            const int p = e / PPR, k = e - p * PPR;
            *reinterpret_cast<int4*>(dst + p * gsp + k * EPP) =
                *reinterpret_cast<const int4*>(ost + p * C + k * EPP);
          }
        } else if (vec8) {
          for (int p = tid; p < n; p += NT)
            *reinterpret_cast<float2*>(dst + p * gsp) = *reinterpret_cast<const float2*>(ost + p * C);
        } else {
          for (int e = tid; e < n * C; e += NT) {
            const int p = e / C, cc = e - p * C;
            if (line0 + cc < nl) dst[p * gsp + cc * gsl] = ost[e];
          }
        }
        __syncthreads();  // the next plane's passes write the exchange lines
      }
    }
  }
  if (abar && tid == 0) bulk_wait_all();
}

// ------------------------------------------------------------- launcher
template <typename T, bool TR, int NT, int V, int C, int MINB>
bool rf1_res_launch_shape(const T* in, T* out, const Rf1LineArgs& a, cudaStream_t st) {
  using L = Rf1ResSmem<NT, V, C>;
  const size_t smem = L::bytes(a.k, a.segcap);
  if (smem > size_t(227) * 1024) return false;  // MINB is a register hint; more smem only lowers occupancy
  auto kern = k_rf1_res<T, TR, NT, V, C, MINB>;
  static size_t attr = 0;
  if (smem > attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem)) != cudaSuccess) {
      (void)cudaGetLastError();
      return false;
    }
    attr = smem;
  }
  const int64_t nl = C == 1 ? a.ny : a.nx;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t tiles = (nl + C - 1) / C;
  const int64_t groups = (planes + a.planes_per_cta - 1) / a.planes_per_cta;
  CUtensorMap tmi{}, tmo{};
  if (C == 1) {
    kern<<<static_cast<unsigned>(tiles * groups), NT, smem, st>>>(in, out, a, tmi, tmo);
    return true;
  }
  Rf1LineArgs b = a;
  b.tma = 0;
  if (C * sizeof(T) >= 16 && (a.nx * sizeof(T)) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) % 16 == 0) {
    // field as a [planes][ny][nx] tensor; a tile's boxes are NQ rows x C columns
    const uint64_t dims[3] = {static_cast<uint64_t>(a.nx), static_cast<uint64_t>(a.ny),
                              static_cast<uint64_t>(planes)};
    const uint64_t strides[2] = {static_cast<uint64_t>(a.nx) * sizeof(T),
                                 static_cast<uint64_t>(a.nx) * a.ny * sizeof(T)};
    const uint32_t box[3] = {static_cast<uint32_t>(C), static_cast<uint32_t>(NT / C), 1u};
    tmi = make_tmap(in, tma_dtype<T>(), 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE);
    tmo = make_tmap(out, tma_dtype<T>(), 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE);
    b.tma = 1;
  }
  // clusters of CL CTAs = CL neighbouring tiles (a short last cluster gets idle partners)
  constexpr int CL = 2;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>((tiles + CL - 1) / CL * groups * CL));
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, in, out, b, tmi, tmo) != cudaSuccess) {
    (void)cudaGetLastError();  // the caller falls back to the streaming passes
    return false;
  }
  return true;
}

// y sweeps: tiles of CY adjacent columns, up to 2176 rows
template <typename T, bool TR, int CY>
bool launch_rf1_cols(const T* in, T* out, Rf1LineArgs a, cudaStream_t st) {
  constexpr int W = CY / 2;  // thread-count factor of the 4-column shapes
  const int64_t planes = a.nvar * a.nlev;
  const int64_t n = a.ny, tiles = (a.nx + CY - 1) / CY;
  int ppc = static_cast<int>(std::max<int64_t>(1, tiles * planes / (148 * 4 * 2)));
  a.planes_per_cta = static_cast<int>(std::min<int64_t>(std::min<int64_t>(ppc, 16), planes));
  if (n <= 32 * 9) return rf1_res_launch_shape<T, TR, 64 * W, 9, CY, 4>(in, out, a, st);
  if (n <= 64 * 9) return rf1_res_launch_shape<T, TR, 128 * W, 9, CY, 4 / W>(in, out, a, st);
  if (n <= 64 * 17) return rf1_res_launch_shape<T, TR, 128 * W, 17, CY, 4 / W>(in, out, a, st);
  if (n <= 128 * 17) return rf1_res_launch_shape<T, TR, 256 * W, 17, CY, 2 / W>(in, out, a, st);
  return false;
}

template <typename T, bool TR>
bool launch_rf1_line_tr(const T* in, T* out, Rf1LineArgs a, cudaStream_t st) {
  const int64_t planes = a.nvar * a.nlev;
  if (a.dir == 0) {  // rows: one line per CTA, up to 8704 points
    const int64_t n = a.nx;
    int ppc = static_cast<int>(std::max<int64_t>(1, a.ny * planes / (148 * 4 * 4)));
    a.planes_per_cta = static_cast<int>(std::min<int64_t>(std::min<int64_t>(ppc, 16), planes));
    if (n <= 128 * 9) return rf1_res_launch_shape<T, TR, 128, 9, 1, 4>(in, out, a, st);
    if (n <= 128 * 17) return rf1_res_launch_shape<T, TR, 128, 17, 1, 4>(in, out, a, st);
    if (n <= 256 * 17) return rf1_res_launch_shape<T, TR, 256, 17, 1, 2>(in, out, a, st);
    if (n <= 512 * 17) return rf1_res_launch_shape<T, TR, 512, 17, 1, 1>(in, out, a, st);
    return false;
  }
  // columns: tiles of 2 adjacent columns (16 B row pieces in fp64; the other
  // half of each 32 B sector belongs to the neighbouring tile of the cluster).
  // Measured on C5 (20 levels, fp64 y sweep, cp.async pieces): 2 columns x 256
  // threads, two CTAs per SM 2.93 ms; 4 columns x 512 threads, one CTA per SM
  // 3.20 ms. fp32 fields whose rows allow tensor copies take 4-column tiles
  // (16 B pieces; C5 fp32 y sweep 15.7 -> 14.3 ms), others 2-column tiles
  // with 8 B cp.async pieces.
  if (sizeof(T) == 4 && (a.nx * sizeof(T)) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) % 16 == 0)
    return launch_rf1_cols<T, TR, 4>(in, out, a, st);
  return launch_rf1_cols<T, TR, 2>(in, out, a, st);
}

// One sweep (all K iterations) of direction a.dir; false when the line does
// not fit the resident shapes (the caller falls back to the streaming passes).
template <typename T>
bool launch_rf1_line(const T* in, T* out, const Rf1LineArgs& a, cudaStream_t st) {
  return a.transpose ? launch_rf1_line_tr<T, true>(in, out, a, st)
                     : launch_rf1_line_tr<T, false>(in, out, a, st);
}

}  // namespace rgfb
