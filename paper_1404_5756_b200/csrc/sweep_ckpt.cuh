// Checkpointed 3rd-RF sweeps: three field passes per direction instead of four.
//
// The two-pass sweep (sweep_tma.cuh) moves every element four times: pass A
// reads the input and writes the causal terms, pass D reads them back and
// writes the result. Here a line is cut into blocks of X points and swept by
// two kernels:
//
//   C1 (ascending, read-only): the causal recursion over the whole line;
//      its only output is the raw 3-value causal state entering every block
//      (`ck`, 24 B per chain and block).
//   C2 (descending over blocks): one block at a time is staged in shared
//      memory by TMA. Each thread re-runs the causal recursion of its chain
//      over the block from the checkpoint, keeping the block's causal values
//      in registers (the loop is fully unrolled), then runs the anti-causal
//      recursion down the block — its state carried in registers from the
//      block on the right — and writes the result. At a segment end j the
//      anti-causal state is entered from the right-ghost closure,
//      e = M_j raw_j (closures.cuh; rf3.hpp:241-274 with the G ghost steps
//      collapsed), raw_j being rebuilt from the registers (or the checkpoint
//      for the block's first two points). M_j is read from global memory only
//      at segment ends.
//
// Field traffic per direction: read, read, write (plus checkpoints), against
// read, write, read, write for the two-pass form. The arithmetic is the
// two-pass kernels' step for step (FMA order included); the causal state is
// resumed from its raw form at block starts.
#pragma once
#include <cstdlib>

#include "sweep_tma.cuh"

namespace rgfb {

// block length: x one 128 B subtile (16 doubles / 32 floats), y 16 rows
template <typename T>
constexpr int ck_x() {
  return 128 / int(sizeof(T));
}
// y: 16 rows (16 warps x 32-register value arrays). 8-warp shapes with
// 32-row blocks (half the checkpoint traffic) measured slower for fp32 too.
template <typename T>
constexpr int ck_y() {
  return 16;
}

// Mask words of an ascending pass, one word of lookahead: on entering word w
// the current word is the one loaded 64 points ago (no load on the critical
// path, no branch around a load). Word i of the line is W[i * stride].
struct WordStream {
  uint64_t cur = 0, nxt = 0;
  int64_t wi = -1;
  __device__ __forceinline__ void start(const uint64_t* W, int64_t stride, int64_t words) {
    cur = ldw(W, 0);
    nxt = words > 1 ? ldw(W, stride) : 0ull;
    wi = 0;
  }
  // call with k0 ascending in steps that divide 64
  __device__ __forceinline__ void advance(const uint64_t* W, int64_t stride, int64_t words,
                                          int64_t k0) {
    if ((k0 >> 6) != wi) {
      wi = k0 >> 6;
      cur = nxt;
      const int64_t w2 = wi + 1 < words ? wi + 1 : wi;  // clamped, value unused past the end
      nxt = ldw(W, w2 * stride);
    }
  }
  template <int U>
  __device__ __forceinline__ uint32_t stage(int64_t k0) const {
    return static_cast<uint32_t>((cur >> (k0 & 63)) & ((1ull << U) - 1ull));
  }
};

// resume a pass-A state from its raw form (raw())
__device__ __forceinline__ void restore(FwdA2& s, double r1, double r2, double r3) {
  s.p1 = r1;
  s.p2 = r2;
  s.p3 = r3;
}
__device__ __forceinline__ void restore(AdjA2& s, double r1, double r2, double r3) {
  // pending contributions into k, k+1, k+2: canonical gather form
  s.u1 = 0.0;
  s.x1 = 0.0;
  s.y22 = 0.0;
  s.y21 = 0.0;
  s.y33 = r1;
  s.y32 = r2;
  s.y31 = r3;
}
// Segment-start reset as predicated zero moves (the compiler's selects cost
// two FSEL per double on every step).
__device__ __forceinline__ void zero_if(double& v, uint32_t on) {
  asm("{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n @p mov.f64 %0, 0d0000000000000000;\n}\n"
      : "+d"(v)
      : "r"(on));
}
__device__ __forceinline__ void reset_if(FwdA2& s, uint32_t on) {
  zero_if(s.p1, on);
  zero_if(s.p2, on);
  zero_if(s.p3, on);
}
__device__ __forceinline__ void reset_if(AdjA2& s, uint32_t on) {
  zero_if(s.u1, on);
  zero_if(s.x1, on);
  zero_if(s.y21, on);
  zero_if(s.y22, on);
  zero_if(s.y31, on);
  zero_if(s.y32, on);
  zero_if(s.y33, on);
}
// predicated streaming store (no branch around it)
__device__ __forceinline__ void st_cs_if(double* p, double v, bool on) {
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.global.cs.f64 [%0], %1;\n}\n"
               ::"l"(p), "d"(v), "r"(static_cast<uint32_t>(on))
               : "memory");
}
__device__ __forceinline__ void st_cs_if(float* p, double v, bool on) {
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p st.global.cs.f32 [%0], %1;\n}\n"
               ::"l"(p), "f"(static_cast<float>(v)), "r"(static_cast<uint32_t>(on))
               : "memory");
}

// anti-causal entry states (as FwdD::enter / AdjD::enter)
__device__ __forceinline__ void enter(FwdD2& s, const double3& e, const Coef3&) {
  s.q1 = e.x;
  s.q2 = e.y;
  s.q3 = e.z;
}
__device__ __forceinline__ void enter(AdjD2& s, const double3& e, const Coef3& c) {
  s.U1 = e.x;
  s.X1 = c.a1;
  s.Y21 = c.a2 * e.x;
  s.Y22 = c.a2 * e.y;
  s.Y31 = c.a3 * e.x;
  s.Y32 = c.a3 * e.y;
  s.Y33 = c.a3 * e.z;
}


// Per-block metadata of one chain, loaded a block ahead (prefetch): the
// checkpoint and the two mask words the block's bits come from.
struct BlockMeta {
  double r1, r2, r3;
  uint64_t w0, wp, wn;  // mask words of kb, the one before and the one after
};
// Issued one block ahead and consumed a block later, so everything here is
// branch-free (a branch around the loads would make the compiler wait for
// them): the checkpoint loads are predicated, the neighbour words clamped.
// ck: this chain's checkpoint of block b (3 values `cs` apart), valid if `has`.
template <int X>
__device__ __forceinline__ BlockMeta load_meta(const double* ck, bool has, int64_t cs,
                                               const uint64_t* W, int64_t ws, int64_t kb,
                                               int64_t words) {
  BlockMeta m;
  m.r1 = m.r2 = m.r3 = 0.0;
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " @p ld.global.cs.f64 %0, [%3];\n"
      " @p ld.global.cs.f64 %1, [%5];\n"
      " @p ld.global.cs.f64 %2, [%6];\n}\n"
      : "+d"(m.r1), "+d"(m.r2), "+d"(m.r3)
      : "l"(ck), "r"(static_cast<int>(has)), "l"(ck + cs), "l"(ck + 2 * cs));
  const int64_t wi = kb >> 6;
  m.w0 = ldw(W, wi * ws);
  m.wp = ldw(W, (wi > 0 ? wi - 1 : 0) * ws);
  m.wn = ldw(W, (wi + 1 < words ? wi + 1 : wi) * ws);
  return m;
}
struct BlockBits {
  uint32_t sb, sm1, sm2, after;
};
// bits of an X-point block at kb, X in {16, 32} (bits past the line are 0
// in the packed mask; neighbour words outside the line count as 0)
template <int X>
__device__ __forceinline__ BlockBits decode_bits(const BlockMeta& m, int64_t kb, int64_t words) {
  BlockBits b;
  const int off = static_cast<int>(kb & 63);
  const uint64_t wp = kb >= 64 ? m.wp : 0ull;
  const uint64_t wn = (kb >> 6) + 1 < words ? m.wn : 0ull;
  b.sb = static_cast<uint32_t>(m.w0 >> off) & static_cast<uint32_t>((1ull << X) - 1ull);
  if (off == 0) {
    b.sm1 = static_cast<uint32_t>(wp >> 63) & 1u;
    b.sm2 = static_cast<uint32_t>(wp >> 62) & 1u;
  } else {
    b.sm1 = static_cast<uint32_t>(m.w0 >> (off - 1)) & 1u;
    b.sm2 = static_cast<uint32_t>(m.w0 >> (off - 2)) & 1u;
  }
  b.after = off + X < 64 ? static_cast<uint32_t>(m.w0 >> (off + X)) & 1u
                         : static_cast<uint32_t>(wn) & 1u;
  return b;
}

// closure matrix of one segment end. `ldg_early` is emitted where it is
// written (volatile), so a prefetch is not sunk next to its use.
struct Closure {
  double m[9];
};
// rows are 10 doubles (80 B, 16 B aligned): five 16 B loads
__device__ __forceinline__ double2 ldg_early(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ Closure load_closure(const double* M) {
  Closure c;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(M) + q);
    c.m[2 * q] = v.x;
    c.m[2 * q + 1] = v.y;
  }
  c.m[8] = __ldg(M + 8);
  return c;
}
// predicated (no branch: see load_meta); values undefined when !on
__device__ __forceinline__ Closure prefetch_closure(const double* M, bool on) {
  Closure c;
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    double x = 0.0, y = 0.0;
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n"
        " @p ld.global.nc.v2.f64 {%0, %1}, [%2];\n}\n"
        : "+d"(x), "+d"(y)
        : "l"(M + 2 * q), "r"(static_cast<int>(on)));
    c.m[2 * q] = x;
    if (q < 4) c.m[2 * q + 1] = y;
  }
  return c;
}
// first segment end met by the descending pass (highest end bit); its
// closure is fetched at block start, hidden behind the causal pass
__device__ __forceinline__ int first_end(uint32_t ends) { return ends ? 31 - __clz(ends) : -1; }

__device__ __forceinline__ double3 apply_m(const Closure& C, double x0, double x1, double x2) {
  const double* m = C.m;
  return make_double3(fma(m[0], x0, fma(m[1], x1, m[2] * x2)),
                      fma(m[3], x0, fma(m[4], x1, m[5] * x2)),
                      fma(m[6], x0, fma(m[7], x1, m[8] * x2)));
}

// Right-ghost entry at a segment end at block offset u (compile-time after
// unrolling). pv: the block's causal values (p forward, u adjoint); r: the
// block's checkpoint; s1/s2: the segment reaches back to j-1 / j-2.
template <bool TR, int X, class CF>
__device__ __forceinline__ double3 segment_entry(const double (&pv)[X], int u, double r1,
                                                 double r2, double r3, bool s1, bool s2,
                                                 const Coef3& c, CF cf, const Closure& M) {
  double x0, x1, x2;
  if constexpr (!TR) {  // raw = (p_j, p_{j-1}, p_{j-2})
    x0 = pv[u];
    x1 = s1 ? (u >= 1 ? pv[u >= 1 ? u - 1 : 0] : r1) : 0.0;
    x2 = s2 ? (u >= 2 ? pv[u >= 2 ? u - 2 : 0] : (u == 1 ? r1 : r2)) : 0.0;
  } else {  // raw = pending sums into j+1, j+2, j+3 (AdjA2::raw)
    const double uj = pv[u];
    double t1, t2, t3;  // a2_{j-1} u_{j-1}, a3_{j-1} u_{j-1}, a3_{j-2} u_{j-2}
    if (u >= 2) {
      const Coef3 c1 = cf(u - 1), c2 = cf(u - 2);
      const double um1 = pv[u >= 2 ? u - 1 : 0], um2 = pv[u >= 2 ? u - 2 : 0];
      t1 = c1.a2 * um1;
      t2 = c1.a3 * um1;
      t3 = c2.a3 * um2;
    } else if (u == 1) {
      const Coef3 c1 = cf(0);
      t1 = c1.a2 * pv[0];
      t2 = c1.a3 * pv[0];
      t3 = r3;
    } else {
      t1 = r2;  // checkpoint pending sums already combine j-1 and j-2
      t2 = r3;
      t3 = 0.0;
    }
    if (!s1) t1 = t2 = t3 = 0.0;
    if (!s2) t3 = 0.0;
    x0 = fma(c.a1, uj, t3 + t1);
    x1 = t2 + c.a2 * uj;
    x2 = c.a3 * uj;
  }
  return apply_m(M, x0, x1, x2);
}

// Loaded with volatile ld.shared so the compiler re-reads them in the
// anti-causal pass instead of keeping 128 values live (spills).
__device__ __forceinline__ double2 lds_f64x2(const double* p) {
  double2 v;
  asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];\n"
               : "=d"(v.x), "=d"(v.y)
               : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ Coef3 lds_coef(const Coef3* c) {
  const double2 lo = lds_f64x2(reinterpret_cast<const double*>(c));
  const double2 hi = lds_f64x2(reinterpret_cast<const double*>(c) + 2);
  return Coef3{lo.x, lo.y, hi.x, hi.y};
}

// ============================================================ x-sweep
// C1, x: one row x 32*NW planes per CTA, TMA stages of U points (as k_xtma)
template <typename T, bool TR, bool IDC, bool VAR, int NW, int S>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    k_xck1(StreamArgs a, double* __restrict__ ck, const __grid_constant__ CUtensorMap tm_in,
           const __grid_constant__ CUtensorMap tm_coef, const __grid_constant__ CUtensorMap tm_idc) {
  using L = XT<T, NW, false>;
  constexpr int U = L::U, X = ck_x<T>(), SPB = X / U;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * L::bytes);
  uint64_t* empty = full + S;

  const int64_t n = a.nx, ny = a.ny;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t PB = (planes + 32 * NW - 1) / (32 * NW);
  const int64_t iy = blockIdx.x / PB;
  const int64_t p0 = (blockIdx.x - iy * PB) * 32 * NW;
  const int npl = static_cast<int>(planes - p0 < 32 * NW ? planes - p0 : 32 * NW);
  const int nwp = (npl + 31) / 32;
  const int64_t NB = (n + X - 1) / X;
  const int64_t nst = (NB - 1) * SPB;  // stages up to the last checkpoint
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwp);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == NW) {  // producer
    if (lane == 0) {
      const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
      tma_prefetch_desc(&tm_in);
      tma_prefetch_desc(&tm_coef);
      const uint32_t total = static_cast<uint32_t>(L::field + L::coef + (IDC ? L::idc : 0));
      for (int64_t i = 0; i < nst; ++i) {
        const int s = static_cast<int>(i % S);
        const int64_t m = i / S;
        if (m > 0) mbar_wait(&empty[s], static_cast<uint32_t>((m - 1) & 1));
        const int k0 = static_cast<int>(i * U);
        unsigned char* base = smem + s * L::bytes;
        mbar_arrive_expect_tx(&full[s], total);
        tma_load_3d(base, &tm_in, k0, static_cast<int>(iy), static_cast<int>(p0), &full[s],
                    pol_stream);
        tma_load_2d(base + L::field, &tm_coef, 4 * k0, static_cast<int>(iy), &full[s], pol_keep);
        if constexpr (IDC)
          tma_load_2d(base + L::field + L::coef, &tm_idc, k0, static_cast<int>(iy), &full[s],
                      pol_keep);
      }
    }
    return;
  }
  if (warp >= nwp) return;

  const int pr = warp * 32 + lane;
  const bool act = pr < npl;
  const int64_t p = p0 + (act ? pr : 0);
  const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
  // transposed mask words: lanes (consecutive levels) read consecutive words
  const uint64_t* W = a.bitsT + iy * a.words * a.nlev_all + lev;
  const int64_t ws = a.nlev_all;
  const double* PRE = VAR ? a.pre_scale + lev * n * ny + iy * n : nullptr;
  WordStream sbw;
  sbw.start(W, ws, a.words);
  typename std::conditional<TR, AdjA2, FwdA2>::type st;
  uint32_t carry = 0;
  constexpr int EPC = 16 / int(sizeof(T));
  const int sw = pr & 7;

  for (int64_t i = 0; i < nst; ++i) {
    const int s = static_cast<int>(i % S);
    const int64_t k0 = i * U;
    sbw.advance(W, ws, a.words, k0);
    const uint32_t sb = sbw.stage<U>(k0);
    const uint32_t starts = sb & ~((sb << 1) | carry);
    mbar_wait(&full[s], static_cast<uint32_t>((i / S) & 1));
    const unsigned char* base = smem + s * L::bytes;
    const Coef3* cf = reinterpret_cast<const Coef3*>(base + L::field);
    const double* id = reinterpret_cast<const double*>(base + L::field + L::coef);
    const unsigned char* rowp = base + pr * 128;
#pragma unroll 1
    for (int q = 0; q < U / EPC; ++q) {
      const void* cp = rowp + ((q ^ sw) << 4);
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
        if constexpr (TR && VAR) w *= __ldg(PRE + (k0 + u < n ? k0 + u : n - 1));
        if constexpr (TR && IDC) w *= id[u];
        st.step(cf[u], w);
      }
    }
    carry = (sb >> (U - 1)) & 1u;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if ((i + 1) % SPB == 0 && act) {  // raw state entering block b
      const int64_t b = (i + 1) / SPB;
      const double4 r = st.raw();
      double* o = ck + ((iy * NB + b) * 3) * planes + p;
      __stcg(o, r.x);
      __stcg(o + planes, r.y);
      __stcg(o + 2 * planes, r.z);
    }
  }
}

// Paired-stage C1, x (see k_xck1): a stage is two U-point halves fetched as
// one [32*NW planes][2][U] box, so every (plane, row) is a 256 B run
template <typename T, bool TR, bool IDC, bool VAR, int NW, int S>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    k_xck1p(StreamArgs a, double* __restrict__ ck, const __grid_constant__ CUtensorMap tm_in,
           const __grid_constant__ CUtensorMap tm_coef, const __grid_constant__ CUtensorMap tm_idc) {
  using L = XT<T, NW, false>;
  constexpr int U = L::U, X = ck_x<T>();
  static_assert(X == U, "one checkpoint per half stage");
  constexpr size_t PF = 2 * L::field, PC = 2 * L::coef, PI = 2 * L::idc;
  constexpr size_t PBYTES = (PF + PC + PI + 1023) / 1024 * 1024;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * PBYTES);
  uint64_t* empty = full + S;

  const int64_t n = a.nx, ny = a.ny;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t PB = (planes + 32 * NW - 1) / (32 * NW);
  const int64_t iy = blockIdx.x / PB;
  const int64_t p0 = (blockIdx.x - iy * PB) * 32 * NW;
  const int npl = static_cast<int>(planes - p0 < 32 * NW ? planes - p0 : 32 * NW);
  const int nwp = (npl + 31) / 32;
  const int64_t NB = (n + X - 1) / X;
  const int64_t nst = NB / 2;  // paired stages covering blocks 0..NB-2 (checkpoints 1..NB-1)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwp);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == NW) {  // producer
    if (lane == 0) {
      const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
      tma_prefetch_desc(&tm_in);
      tma_prefetch_desc(&tm_coef);
      const uint32_t total = static_cast<uint32_t>(PF + PC + (IDC ? PI : 0));
      for (int64_t i = 0; i < nst; ++i) {
        const int s = static_cast<int>(i % S);
        const int64_t m = i / S;
        if (m > 0) mbar_wait(&empty[s], static_cast<uint32_t>((m - 1) & 1));
        const int k0 = static_cast<int>(i * 2 * U);
        unsigned char* base = smem + s * PBYTES;
        mbar_arrive_expect_tx(&full[s], total);
        tma_load_4d(base, &tm_in, 0, static_cast<int>(2 * i), static_cast<int>(iy),
                    static_cast<int>(p0), &full[s], pol_stream);
        tma_load_2d(base + PF, &tm_coef, 4 * k0, static_cast<int>(iy), &full[s], pol_keep);
        if constexpr (IDC)
          tma_load_2d(base + PF + PC, &tm_idc, k0, static_cast<int>(iy), &full[s], pol_keep);
      }
    }
    return;
  }
  if (warp >= nwp) return;

  const int pr = warp * 32 + lane;
  const bool act = pr < npl;
  const int64_t p = p0 + (act ? pr : 0);
  const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
  // transposed mask words: lanes (consecutive levels) read consecutive words
  const uint64_t* W = a.bitsT + iy * a.words * a.nlev_all + lev;
  const int64_t ws = a.nlev_all;
  const double* PRE = VAR ? a.pre_scale + lev * n * ny + iy * n : nullptr;
  WordStream sbw;
  sbw.start(W, ws, a.words);
  typename std::conditional<TR, AdjA2, FwdA2>::type st;
  uint32_t carry = 0;
  constexpr int EPC = 16 / int(sizeof(T));
  const int sw = pr & 7;

  for (int64_t i = 0; i < nst; ++i) {
    const int s = static_cast<int>(i % S);
    mbar_wait(&full[s], static_cast<uint32_t>((i / S) & 1));
    const unsigned char* base = smem + s * PBYTES;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t k0 = (2 * i + h) * U;
      sbw.advance(W, ws, a.words, k0);
      const uint32_t sb = sbw.stage<U>(k0);
      const uint32_t starts = sb & ~((sb << 1) | carry);
      const Coef3* cf = reinterpret_cast<const Coef3*>(base + PF) + h * U;
      const double* id = reinterpret_cast<const double*>(base + PF + PC) + h * U;
      const int rr = pr * 2 + h;
      const unsigned char* rowp = base + rr * 128;
      const int sw = rr & 7;
#pragma unroll 1
      for (int q = 0; q < U / EPC; ++q) {
        const void* cp = rowp + ((q ^ sw) << 4);
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
          if constexpr (TR && VAR) w *= __ldg(PRE + (k0 + u < n ? k0 + u : n - 1));
          if constexpr (TR && IDC) w *= id[u];
          st.step(cf[u], w);
        }
      }
      carry = (sb >> (U - 1)) & 1u;
      const int64_t b = 2 * i + h + 1;  // raw state entering block b
      if (act && b < NB) {
        const double4 r = st.raw();
        double* o = ck + ((iy * NB + b) * 3) * planes + p;
        __stcg(o, r.x);
        __stcg(o + planes, r.y);
        __stcg(o + 2 * planes, r.z);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}


// C2, x layout: R rows x 32*NWR planes per CTA; a block is NS subtiles of
// [R rows][32*NWR planes][128 B], 128 B swizzled (the tensor map lists the
// plane dimension before the row dimension, so a warp's 32 planes are 32
// consecutive 128 B rows: conflict-free 16 B accesses).
template <typename T, int R, int NWR>
struct XC2 {
  static constexpr int U = 128 / int(sizeof(T));
  static constexpr int X = ck_x<T>();
  static constexpr int NS = X / U;
  static constexpr size_t sub = size_t(R) * NWR * 32 * 128;
  static constexpr size_t field = NS * sub;
  static constexpr size_t coef = size_t(R) * X * sizeof(Coef3);
  static constexpr size_t idc = size_t(R) * X * sizeof(double);
  static constexpr size_t bytes = (field + coef + idc + 1023) / 1024 * 1024;
};

template <typename T, bool TR, bool IDC, bool PRE, bool POST, int R, int NWR, int S>
__global__ void __launch_bounds__(32 * R * NWR, 1)
    k_xck2(StreamArgs a, const double* __restrict__ ck, const __grid_constant__ CUtensorMap tm_in,
           const __grid_constant__ CUtensorMap tm_out, const __grid_constant__ CUtensorMap tm_coef,
           const __grid_constant__ CUtensorMap tm_idc) {
  using L = XC2<T, R, NWR>;
  constexpr int U = L::U, X = L::X, NS = L::NS, NWC = R * NWR;
  constexpr int ESZ = static_cast<int>(sizeof(T));
  constexpr int EPC = 16 / ESZ;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * L::bytes);
  int* released = reinterpret_cast<int*>(full + S);  // warps done with a buffer

  const int64_t n = a.nx, ny = a.ny, nh = n * ny;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t PB = (planes + 32 * NWR - 1) / (32 * NWR);
  const int64_t iyb = blockIdx.x / PB;
  const int64_t p0 = (blockIdx.x - iyb * PB) * 32 * NWR;
  const int64_t iy0 = iyb * R;
  const int npl = static_cast<int>(planes - p0 < 32 * NWR ? planes - p0 : 32 * NWR);
  const int64_t NB = (n + X - 1) / X;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // No producer warp and no CTA-wide barrier: each warp returns its own
  // [32 planes x 1 row] part of a block with a TMA store, and the last warp
  // to release a buffer (its store read out) issues the buffer's next load.
  auto load_block = [&](int64_t bi) {
    const int s = static_cast<int>(bi % S);
    const int64_t kb = (NB - 1 - bi) * X;
    const int nsub = static_cast<int>((n - kb + U - 1) / U < NS ? (n - kb + U - 1) / U : NS);
    unsigned char* base = smem + s * L::bytes;
    const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(nsub * L::sub + L::coef +
                                                           (IDC ? L::idc : 0)));
    for (int t = 0; t < nsub; ++t)
      tma_load_3d(base + t * L::sub, &tm_in, static_cast<int>(kb + t * U), static_cast<int>(p0),
                  static_cast<int>(iy0), &full[s], pol_stream);
    tma_load_2d(base + L::field, &tm_coef, static_cast<int>(4 * kb), static_cast<int>(iy0),
                &full[s], pol_keep);
    if constexpr (IDC)
      tma_load_2d(base + L::field + L::coef, &tm_idc, static_cast<int>(kb), static_cast<int>(iy0),
                  &full[s], pol_keep);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0;
    }
    mbar_fence_init();
    tma_prefetch_desc(&tm_in);
    tma_prefetch_desc(&tm_coef);
    for (int64_t bi = 0; bi < S && bi < NB; ++bi) load_block(bi);
  }
  __syncthreads();
  // lane 0 of each warp: once this warp's store of block `bi` has read its
  // buffer, count the warp out; the last one refills the buffer
  auto release = [&](int64_t bi) {
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    const int s = static_cast<int>(bi % S);
    if (atomicAdd(&released[s], 1) == NWC - 1) {
      released[s] = 0;
      if (bi + S < NB) load_block(bi + S);
    }
  };

  // consumers: warp -> (row r, 32 planes)
  const int r = warp / NWR;
  const int pg = warp - r * NWR;
  const int pl = pg * 32 + lane;
  const int64_t iy = iy0 + r;
  const bool act = pl < npl && iy < ny;
  const int64_t p = p0 + (pl < npl ? pl : 0);
  const int64_t iyc = iy < ny ? iy : iy0;
  const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
  (void)var;
  const uint64_t* W = a.bitsT + iyc * a.words * a.nlev_all + lev;
  const int64_t ws = a.nlev_all;
  const double* PREp = PRE ? a.pre_scale + lev * nh + iyc * n : nullptr;
  const double* POSTp = POST ? a.post_scale + lev * nh + iyc * n : nullptr;
  const double* Mrow = a.clos + clos_off(a.cls[lev], 0, TR ? 1 : 0, nh, iyc * n);
  const bool ghosts = a.ghost[lev] > 0;
  const int rs = r * 32 * NWR + pl;  // 128 B row of this chain in a subtile
  const int sw = rs & 7;
  typename std::conditional<TR, AdjA2, FwdA2>::type sa;
  typename std::conditional<TR, AdjD2, FwdD2>::type sd;
  auto meta = [&](int64_t b) {
    return load_meta<X>(ck + ((iy * NB + b) * 3) * planes + p, b > 0 && act, planes, W, ws,
                        b * X, a.words);
  };
  BlockMeta next = meta(NB - 1);

  for (int64_t bi = 0; bi < NB; ++bi) {
    const int s = static_cast<int>(bi % S);
    const int64_t b = NB - 1 - bi;
    const int64_t kb = b * X;
    const BlockMeta cur = next;
    if (b > 0) next = meta(b - 1);  // consumed one block from now
    const double r1 = cur.r1, r2 = cur.r2, r3 = cur.r3;
    const BlockBits bb = decode_bits<X>(cur, kb, a.words);
    const uint32_t sb = bb.sb, sm1 = bb.sm1, sm2 = bb.sm2, after = bb.after;
    const uint32_t starts = sb & ~((sb << 1) | sm1);
    const uint32_t ends = sb & ~((sb >> 1) | (after << (X - 1)));
    const int jl = first_end(ends);
    const Closure mpre = prefetch_closure(Mrow + (kb + (jl > 0 ? jl : 0)) * 10,
                                          jl >= 0 && kb + jl < n - 1 && ghosts);
    mbar_wait(&full[s], static_cast<uint32_t>((bi / S) & 1));
    unsigned char* base = smem + s * L::bytes;
    const Coef3* cf = reinterpret_cast<const Coef3*>(base + L::field) + r * X;
    const double* id = reinterpret_cast<const double*>(base + L::field + L::coef) + r * X;
    auto cfu = [&](int uu) -> Coef3 { return lds_coef(cf + uu); };

    // ---- causal recursion over the block from its checkpoint (registers)
    restore(sa, r1, r2, r3);
    double pv[X];
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      const unsigned char* rowp = base + t * L::sub + rs * 128;
#pragma unroll
      for (int q = 0; q < U / EPC; ++q) {
        const void* cp = rowp + ((q ^ sw) << 4);
        double v[EPC];
        if constexpr (sizeof(T) == 8) {
          const double2 tv = *reinterpret_cast<const double2*>(cp);
          v[0] = tv.x;
          v[1] = tv.y;
        } else {
          const float4 tv = *reinterpret_cast<const float4*>(cp);
          v[0] = tv.x;
          v[1] = tv.y;
          v[2] = tv.z;
          v[3] = tv.w;
        }
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          const int u = t * U + q * EPC + e;
          reset_if(sa, (starts >> u) & 1u);
          double w = v[e];
          if constexpr (TR && PRE) w *= __ldg(PREp + (kb + u < n ? kb + u : n - 1));
          if constexpr (TR && IDC) w *= id[u];
          pv[u] = sa.step(cfu(u), w);
        }
      }
    }
    // the previous block's store has had the whole causal pass to read out
    if (lane == 0 && bi >= 1) release(bi - 1);

    // ---- anti-causal recursion down the block, results in place
#pragma unroll
    for (int t = NS - 1; t >= 0; --t) {
      unsigned char* rowp = base + t * L::sub + rs * 128;
#pragma unroll
      for (int q = U / EPC - 1; q >= 0; --q) {
        void* cp = rowp + ((q ^ sw) << 4);
        double o[EPC];
#pragma unroll
        for (int e = EPC - 1; e >= 0; --e) {
          const int u = t * U + q * EPC + e;
          const Coef3 c = cfu(u);
          if ((ends >> u) & 1u) {  // segment end: enter from the right ghosts
            if (kb + u < n - 1 && ghosts) {
              const bool s1 = u >= 1 ? ((sb >> (u >= 1 ? u - 1 : 0)) & 1u) : sm1;
              const bool s2 =
                  s1 && (u >= 2 ? ((sb >> (u >= 2 ? u - 2 : 0)) & 1u) : (u == 1 ? sm1 : sm2));
              const Closure M = u == jl ? mpre : load_closure(Mrow + (kb + u) * 10);
              enter(sd, segment_entry<TR, X>(pv, u, r1, r2, r3, s1, s2, c, cfu, M), c);
            } else {
              sd.reset();
            }
          }
          double ov = sd.step(c, c.b * pv[u]);
          if constexpr (!TR && IDC) ov *= id[u];
          if constexpr (POST) ov *= __ldg(POSTp + (kb + u < n ? kb + u : n - 1));
          o[e] = ((sb >> u) & 1u) ? ov : 0.0;
        }
        if constexpr (sizeof(T) == 8) {
          *reinterpret_cast<double2*>(cp) = make_double2(o[0], o[1]);
        } else {
          *reinterpret_cast<float4*>(cp) =
              make_float4(static_cast<float>(o[0]), static_cast<float>(o[1]),
                          static_cast<float>(o[2]), static_cast<float>(o[3]));
        }
      }
    }
    // this warp's [32 planes x 1 row] of the block back to global memory
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (iy < ny && pg * 32 < npl) {
        const int nsub = static_cast<int>((n - kb + U - 1) / U < NS ? (n - kb + U - 1) / U : NS);
        for (int t = 0; t < nsub; ++t)
          tma_store_3d(&tm_out, static_cast<int>(kb + t * U), static_cast<int>(p0 + pg * 32),
                       static_cast<int>(iy), base + t * L::sub + (r * 32 * NWR + pg * 32) * 128,
                       l2_evict_first());
      }
      bulk_commit();
    }
  }
  if (lane == 0) {
    if (NB >= 1) release(NB - 1);
    bulk_wait_all();
  }
}

// Paired-tile variant of C2, x layout (see k_xck2)
template <typename T, bool TR, bool IDC, bool PRE, bool POST, int R, int NWR, int S>
__global__ void __launch_bounds__(32 * R * NWR, 1)
    k_xck2p(StreamArgs a, const double* __restrict__ ck, const __grid_constant__ CUtensorMap tm_in,
           const __grid_constant__ CUtensorMap tm_out, const __grid_constant__ CUtensorMap tm_coef,
           const __grid_constant__ CUtensorMap tm_idc) {
  using L = XC2<T, R, NWR>;
  constexpr int U = L::U, X = L::X, NWC = R * NWR;
  static_assert(L::NS == 1, "paired tiles take one 128 B subtile per block");
  // a tile is two consecutive blocks: [R rows][32*NWR planes][2][X], so every
  // (plane, row) is fetched and stored as one 256 B run (a TMA copy with
  // 128 B runs caps at ~4.9 TB/s, with 256 B runs at ~6.2 TB/s:
  // tools/probe/tma_copy_probe.cu)
  constexpr size_t TF = 2 * L::sub, TC = 2 * L::coef, TI = 2 * L::idc;
  constexpr size_t TB = (TF + TC + TI + 1023) / 1024 * 1024;
  constexpr int ESZ = static_cast<int>(sizeof(T));
  constexpr int EPC = 16 / ESZ;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * TB);
  int* released = reinterpret_cast<int*>(full + S);  // warps done with a buffer

  const int64_t n = a.nx, ny = a.ny, nh = n * ny;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t PB = (planes + 32 * NWR - 1) / (32 * NWR);
  const int64_t iyb = blockIdx.x / PB;
  const int64_t p0 = (blockIdx.x - iyb * PB) * 32 * NWR;
  const int64_t iy0 = iyb * R;
  const int npl = static_cast<int>(planes - p0 < 32 * NWR ? planes - p0 : 32 * NWR);
  const int64_t NB = (n + X - 1) / X;
  const int64_t NT = (NB + 1) / 2;  // tiles
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // No producer warp and no CTA-wide barrier: each warp returns its own
  // [32 planes x 1 row] part of a block with a TMA store, and the last warp
  // to release a buffer (its store read out) issues the buffer's next load.
  auto load_tile = [&](int64_t ti) {
    const int s = static_cast<int>(ti % S);
    const int64_t j = NT - 1 - ti;  // blocks 2j, 2j+1
    unsigned char* base = smem + s * TB;
    const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(TF + TC + (IDC ? TI : 0)));
    tma_load_4d(base, &tm_in, 0, static_cast<int>(2 * j), static_cast<int>(p0), static_cast<int>(iy0),
                &full[s], pol_stream);
    tma_load_2d(base + TF, &tm_coef, static_cast<int>(4 * 2 * j * X), static_cast<int>(iy0),
                &full[s], pol_keep);
    if constexpr (IDC)
      tma_load_2d(base + TF + TC, &tm_idc, static_cast<int>(2 * j * X), static_cast<int>(iy0),
                  &full[s], pol_keep);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0;
    }
    mbar_fence_init();
    tma_prefetch_desc(&tm_in);
    tma_prefetch_desc(&tm_coef);
    for (int64_t ti = 0; ti < S && ti < NT; ++ti) load_tile(ti);
  }
  __syncthreads();
  // lane 0 of each warp: once this warp's store of block `bi` has read its
  // buffer, count the warp out; the last one refills the buffer
  auto release = [&](int64_t ti) {
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    const int s = static_cast<int>(ti % S);
    if (atomicAdd(&released[s], 1) == NWC - 1) {
      released[s] = 0;
      if (ti + S < NT) load_tile(ti + S);
    }
  };

  // consumers: warp -> (row r, 32 planes)
  const int r = warp / NWR;
  const int pg = warp - r * NWR;
  const int pl = pg * 32 + lane;
  const int64_t iy = iy0 + r;
  const bool act = pl < npl && iy < ny;
  const int64_t p = p0 + (pl < npl ? pl : 0);
  const int64_t iyc = iy < ny ? iy : iy0;
  const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
  (void)var;
  const uint64_t* W = a.bitsT + iyc * a.words * a.nlev_all + lev;
  const int64_t ws = a.nlev_all;
  const double* PREp = PRE ? a.pre_scale + lev * nh + iyc * n : nullptr;
  const double* POSTp = POST ? a.post_scale + lev * nh + iyc * n : nullptr;
  const double* Mrow = a.clos + clos_off(a.cls[lev], 0, TR ? 1 : 0, nh, iyc * n);
  const bool ghosts = a.ghost[lev] > 0;
  const int rs0 = (r * 32 * NWR + pl) * 2;  // 128 B row of this chain's first block
  typename std::conditional<TR, AdjA2, FwdA2>::type sa;
  typename std::conditional<TR, AdjD2, FwdD2>::type sd;
  auto meta = [&](int64_t b) {
    return load_meta<X>(ck + ((iy * NB + b) * 3) * planes + p, b > 0 && act, planes, W, ws,
                        b * X, a.words);
  };
  BlockMeta next = meta(NB - 1);

  for (int64_t bi = 0; bi < NB; ++bi) {
    const int64_t b = NB - 1 - bi;
    const int64_t kb = b * X;
    const int h = static_cast<int>(b & 1);
    const int64_t ti = NT - 1 - (b >> 1);
    const int s = static_cast<int>(ti % S);
    const bool tile_first = h == 1 || bi == 0;
    const int rs = rs0 + h;
    const int sw = rs & 7;
    const BlockMeta cur = next;
    if (b > 0) next = meta(b - 1);  // consumed one block from now
    const double r1 = cur.r1, r2 = cur.r2, r3 = cur.r3;
    const BlockBits bb = decode_bits<X>(cur, kb, a.words);
    const uint32_t sb = bb.sb, sm1 = bb.sm1, sm2 = bb.sm2, after = bb.after;
    const uint32_t starts = sb & ~((sb << 1) | sm1);
    const uint32_t ends = sb & ~((sb >> 1) | (after << (X - 1)));
    const int jl = first_end(ends);
    const Closure mpre = prefetch_closure(Mrow + (kb + (jl > 0 ? jl : 0)) * 10,
                                          jl >= 0 && kb + jl < n - 1 && ghosts);
    if (tile_first) mbar_wait(&full[s], static_cast<uint32_t>((ti / S) & 1));
    unsigned char* base = smem + s * TB;
    const Coef3* cf = reinterpret_cast<const Coef3*>(base + TF) + r * 2 * X + h * X;
    const double* id = reinterpret_cast<const double*>(base + TF + TC) + r * 2 * X + h * X;
    auto cfu = [&](int uu) -> Coef3 { return lds_coef(cf + uu); };

    // ---- causal recursion over the block from its checkpoint (registers)
    restore(sa, r1, r2, r3);
    double pv[X];
#pragma unroll
    for (int t = 0; t < 1; ++t) {
      const unsigned char* rowp = base + rs * 128;
#pragma unroll
      for (int q = 0; q < U / EPC; ++q) {
        const void* cp = rowp + ((q ^ sw) << 4);
        double v[EPC];
        if constexpr (sizeof(T) == 8) {
          const double2 tv = *reinterpret_cast<const double2*>(cp);
          v[0] = tv.x;
          v[1] = tv.y;
        } else {
          const float4 tv = *reinterpret_cast<const float4*>(cp);
          v[0] = tv.x;
          v[1] = tv.y;
          v[2] = tv.z;
          v[3] = tv.w;
        }
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          const int u = q * EPC + e;
          reset_if(sa, (starts >> u) & 1u);
          double w = v[e];
          if constexpr (TR && PRE) w *= __ldg(PREp + (kb + u < n ? kb + u : n - 1));
          if constexpr (TR && IDC) w *= id[u];
          pv[u] = sa.step(cfu(u), w);
        }
      }
    }
    // the previous tile's store has had the whole causal pass to read out
    if (lane == 0 && tile_first && ti >= 1) release(ti - 1);

    // ---- anti-causal recursion down the block, results in place
#pragma unroll
    for (int t = 0; t >= 0; --t) {
      unsigned char* rowp = base + rs * 128;
#pragma unroll
      for (int q = U / EPC - 1; q >= 0; --q) {
        void* cp = rowp + ((q ^ sw) << 4);
        double o[EPC];
#pragma unroll
        for (int e = EPC - 1; e >= 0; --e) {
          const int u = q * EPC + e;
          const Coef3 c = cfu(u);
          if ((ends >> u) & 1u) {  // segment end: enter from the right ghosts
            if (kb + u < n - 1 && ghosts) {
              const bool s1 = u >= 1 ? ((sb >> (u >= 1 ? u - 1 : 0)) & 1u) : sm1;
              const bool s2 =
                  s1 && (u >= 2 ? ((sb >> (u >= 2 ? u - 2 : 0)) & 1u) : (u == 1 ? sm1 : sm2));
              const Closure M = u == jl ? mpre : load_closure(Mrow + (kb + u) * 10);
              enter(sd, segment_entry<TR, X>(pv, u, r1, r2, r3, s1, s2, c, cfu, M), c);
            } else {
              sd.reset();
            }
          }
          double ov = sd.step(c, c.b * pv[u]);
          if constexpr (!TR && IDC) ov *= id[u];
          if constexpr (POST) ov *= __ldg(POSTp + (kb + u < n ? kb + u : n - 1));
          o[e] = ((sb >> u) & 1u) ? ov : 0.0;
        }
        if constexpr (sizeof(T) == 8) {
          *reinterpret_cast<double2*>(cp) = make_double2(o[0], o[1]);
        } else {
          *reinterpret_cast<float4*>(cp) =
              make_float4(static_cast<float>(o[0]), static_cast<float>(o[1]),
                          static_cast<float>(o[2]), static_cast<float>(o[3]));
        }
      }
    }
    // tile done (its lower block): this warp's [32 planes x 1 row x 2 blocks]
    // back to global memory as 256 B runs
    if (h == 0) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (iy < ny && pg * 32 < npl)
          tma_store_4d(&tm_out, 0, static_cast<int>(2 * (b >> 1)), static_cast<int>(p0 + pg * 32),
                       static_cast<int>(iy), base + ((r * 32 * NWR + pg * 32) * 2) * 128,
                       l2_evict_first());
        bulk_commit();
      }
    }
  }
  if (lane == 0) {
    if (NT >= 1) release(NT - 1);
    bulk_wait_all();
  }
}


// ============================================================ y-sweep
// Coefficients of the y direction in SoA rows [ny][4][nx] (a1, a2, a3, b):
// lanes = columns read 8 B each, conflict-free.
// staged rows [rows][2][32][2]: (a1, a2) and (a3, b) pairs, 16 B per lane
template <int U>
__device__ __forceinline__ Coef3 coef_soa(const double* cs, int u, int lane) {
  const double* q = cs + u * 128 + lane * 2;
  const double2 lo = lds_f64x2(q), hi = lds_f64x2(q + 64);
  return Coef3{lo.x, lo.y, hi.x, hi.y};
}

template <typename T, int NW, int U>
struct YC1 {
  static constexpr size_t field = size_t(NW) * U * 32 * sizeof(T);
  static constexpr size_t coef = size_t(U) * 4 * 32 * sizeof(double);
  static constexpr size_t idc = size_t(U) * 32 * sizeof(double);
  static constexpr size_t bytes = field + coef + idc;
};

// C1, y: 32 columns x NW planes per CTA, TMA stages of U rows
template <typename T, bool TR, bool IDC, bool VAR, int NW, int U, int S>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    k_yck1(StreamArgs a, double* __restrict__ ck, const __grid_constant__ CUtensorMap tm_field,
           const __grid_constant__ CUtensorMap tm_coef, const __grid_constant__ CUtensorMap tm_idc) {
  using L = YC1<T, NW, U>;
  constexpr int X = ck_y<T>(), SPB = X / U;
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
  const int64_t NB = (ny + X - 1) / X;
  const int64_t nst = (NB - 1) * SPB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwp);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == NW) {  // producer
    if (lane == 0) {
      const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
      tma_prefetch_desc(&tm_field);
      tma_prefetch_desc(&tm_coef);
      // the field box holds box_planes planes (few-plane operators: no zero fill)
      const uint32_t total = static_cast<uint32_t>(
          size_t(a.box_planes) * U * 32 * sizeof(T) + L::coef + (IDC ? L::idc : 0));
      for (int64_t i = 0; i < nst; ++i) {
        const int s = static_cast<int>(i % S);
        const int64_t m = i / S;
        if (m > 0) mbar_wait(&empty[s], static_cast<uint32_t>((m - 1) & 1));
        const int lo = static_cast<int>(i * U);
        unsigned char* base = smem + s * L::bytes;
        mbar_arrive_expect_tx(&full[s], total);
        tma_load_3d(base, &tm_field, static_cast<int>(ix0), lo, static_cast<int>(p0), &full[s],
                    pol_stream);
        tma_load_4d(base + L::field, &tm_coef, 0, static_cast<int>(ix0), 0, lo, &full[s], pol_keep);
        if constexpr (IDC)
          tma_load_2d(base + L::field + L::coef, &tm_idc, static_cast<int>(ix0), lo, &full[s],
                      pol_keep);
      }
    }
    return;
  }
  if (warp >= nwp) return;

  const int64_t p = p0 + warp;
  const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
  const bool act = lane < ncol;
  const int64_t ix = ix0 + (act ? lane : 0);
  const uint64_t* W = a.bitsT + lev * a.words * nx + ix;  // lanes: consecutive words
  const double* PREp = VAR ? a.pre_scale + lev * nh + ix : nullptr;
  WordStream sbw;
  sbw.start(W, nx, a.words);
  typename std::conditional<TR, AdjA2, FwdA2>::type st;
  uint32_t carry = 0;

  for (int64_t i = 0; i < nst; ++i) {
    const int s = static_cast<int>(i % S);
    const int64_t lo = i * U;
    sbw.advance(W, nx, a.words, lo);
    const uint32_t sb = sbw.stage<U>(lo);
    const uint32_t starts = sb & ~((sb << 1) | carry);
    mbar_wait(&full[s], static_cast<uint32_t>((i / S) & 1));
    const unsigned char* base = smem + s * L::bytes;
    const T* fld = reinterpret_cast<const T*>(base) + warp * U * 32 + lane;
    const double* cs = reinterpret_cast<const double*>(base + L::field);
    const double* id = reinterpret_cast<const double*>(base + L::field + L::coef) + lane;
#pragma unroll
    for (int r = 0; r < U; ++r) {
      if ((starts >> r) & 1u) st.reset();
      double w = static_cast<double>(fld[r * 32]);
      if constexpr (TR && VAR) w *= __ldg(PREp + (lo + r < ny ? lo + r : ny - 1) * nx);
      if constexpr (TR && IDC) w *= id[r * 32];
      st.step(coef_soa<U>(cs, r, lane), w);
    }
    carry = (sb >> (U - 1)) & 1u;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if ((i + 1) % SPB == 0 && act) {
      const int64_t b = (i + 1) / SPB;
      const double4 rr = st.raw();
      double* o = ck + ((p * NB + b) * 3) * nx + ix;
      __stcg(o, rr.x);
      __stcg(o + nx, rr.y);
      __stcg(o + 2 * nx, rr.z);
    }
  }
}

template <typename T, int NPL>
struct YC2 {
  static constexpr int X = ck_y<T>();
  static constexpr size_t field = size_t(NPL) * X * 32 * sizeof(T);
  static constexpr size_t coef = size_t(X) * 4 * 32 * sizeof(double);
  static constexpr size_t idc = size_t(X) * 32 * sizeof(double);
  static constexpr size_t bytes = (field + coef + idc + 1023) / 1024 * 1024;
};

// C2, y: blocks of X rows, descending; lanes = columns, each warp carries PPW
// planes (independent chains interleaved: ILP, and one coefficient load
// serves PPW chains); results go straight to global memory (coalesced
// 32-column rows).
template <typename T, bool TR, bool IDC, bool PRE, bool POST, int NW, int PPW, int S, int LG,
          int PD>
__global__ void __launch_bounds__(32 * NW, NW <= 8 ? 2 : 1)
    k_yck2(T* __restrict__ out, StreamArgs a, const double* __restrict__ ck,
           const __grid_constant__ CUtensorMap tm_field, const __grid_constant__ CUtensorMap tm_coef,
           const __grid_constant__ CUtensorMap tm_idc) {
  constexpr int NPL = NW * PPW;  // planes per CTA
  using L = YC2<T, NPL>;
  constexpr int X = L::X;
  // LG > 1: a warp covers 32/LG columns of LG planes (lanes = columns x
  // planes), so one coefficient load serves LG chains and a warp's
  // coefficient LDS.128 touches 32/LG distinct 16 B words instead of 32
  constexpr int CW = 32 / LG;                  // columns per warp
  static_assert(PPW == 1 || LG == 1, "LG > 1 takes one plane per lane");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * L::bytes);
  uint64_t* empty = full + S;

  const int64_t nx = a.nx, ny = a.ny, nh = nx * ny;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t PB = (planes + NPL - 1) / NPL;
  const int64_t tile = blockIdx.x / PB;
  const int64_t p0 = (blockIdx.x - tile * PB) * NPL;
  const int64_t ix0 = tile * 32;
  const int ncol = static_cast<int>(nx - ix0 < 32 ? nx - ix0 : 32);
  const int npl = static_cast<int>(planes - p0 < NPL ? planes - p0 : NPL);
  const int nwp = LG == 1 ? (npl + PPW - 1) / PPW : ((npl + LG - 1) / LG) * LG;
  const int64_t NB = (ny + X - 1) / X;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // no producer warp: thread 0 issues block loads; a buffer is refilled once
  // every warp has finished the block it held (empty barrier)
  const uint32_t total = static_cast<uint32_t>(size_t(a.box_planes) * X * 32 * sizeof(T) +
                                               L::coef + (IDC ? L::idc : 0));
  auto load_block = [&](int64_t bi) {
    const int s = static_cast<int>(bi % S);
    const int lo = static_cast<int>((NB - 1 - bi) * X);
    unsigned char* base = smem + s * L::bytes;
    const uint64_t pol_stream = l2_evict_first(), pol_keep = l2_evict_last();
    mbar_arrive_expect_tx(&full[s], total);
    tma_load_3d(base, &tm_field, static_cast<int>(ix0), lo, static_cast<int>(p0), &full[s],
                pol_stream);
    tma_load_4d(base + L::field, &tm_coef, 0, static_cast<int>(ix0), 0, lo, &full[s], pol_keep);
    if constexpr (IDC)
      tma_load_2d(base + L::field + L::coef, &tm_idc, static_cast<int>(ix0), lo, &full[s],
                  pol_keep);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwp);
    }
    mbar_fence_init();
    tma_prefetch_desc(&tm_field);
    tma_prefetch_desc(&tm_coef);
    for (int64_t bi = 0; bi < S && bi < NB; ++bi) load_block(bi);
  }
  __syncthreads();
  if (warp >= nwp) return;

  // this lane's column in the CTA tile and plane slot
  const int wc = LG == 1 ? 0 : warp % LG;      // column group of the warp
  const int wp = LG == 1 ? warp : warp / LG;   // plane group of the warp
  const int cl = LG == 1 ? lane : wc * CW + lane % CW;  // column in the 32-column tile
  const int ql = LG == 1 ? 0 : lane / CW;      // plane within the warp's group
  const bool colok = cl < ncol;
  const int64_t ix = ix0 + (colok ? cl : 0);
  T* dst[PPW];
  const uint64_t* W[PPW];
  const double* PREp[PPW];
  const double* POSTp[PPW];
  const double* Mcol[PPW];
  bool ghosts[PPW], act[PPW];
  int64_t pp[PPW];
#pragma unroll
  for (int c = 0; c < PPW; ++c) {
    const int pl = LG == 1 ? warp * PPW + c : wp * LG + ql;
    act[c] = colok && pl < npl;
    const int64_t p = p0 + (pl < npl ? pl : 0);
    pp[c] = p;
    const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
    dst[c] = out + p * a.pitch * ny + ix;  // field rows are `pitch` apart
    W[c] = a.bitsT + lev * a.words * nx + ix;
    PREp[c] = PRE ? a.pre_scale + lev * nh + ix : nullptr;
    POSTp[c] = POST ? a.post_scale + lev * nh + ix : nullptr;
    Mcol[c] = a.clos + clos_off(a.cls[lev], 1, TR ? 1 : 0, nh, ix);
    ghosts[c] = a.ghost[lev] > 0;
  }
  typename std::conditional<TR, AdjA2, FwdA2>::type sa[PPW];
  typename std::conditional<TR, AdjD2, FwdD2>::type sd[PPW];
  auto meta = [&](int c, int64_t b) {
    return load_meta<X>(ck + ((pp[c] * NB + b) * 3) * nx + ix, b > 0 && act[c], nx, W[c], nx,
                        b * X, a.words);
  };
  // per-block metadata PD blocks ahead (PD > 1 for the few-plane shape, where
  // no other warp hides the load latency): ring[c][j] = block NB-1-(bi+j)
  BlockMeta ring[PPW][PD];
#pragma unroll
  for (int c = 0; c < PPW; ++c)
#pragma unroll
    for (int j = 0; j < PD; ++j) ring[c][j] = meta(c, NB - 1 - j >= 0 ? NB - 1 - j : 0);

  for (int64_t bi = 0; bi < NB; ++bi) {
    const int s = static_cast<int>(bi % S);
    const int64_t b = NB - 1 - bi;
    const int64_t kb = b * X;
    if (threadIdx.x == 0 && bi >= 1 && bi - 1 + S < NB) {  // refill block bi-1's buffer
      mbar_wait(&empty[(bi - 1) % S], static_cast<uint32_t>(((bi - 1) / S) & 1));
      load_block(bi - 1 + S);
    }
    double r1[PPW], r2[PPW], r3[PPW];
    uint32_t sb[PPW], sm1[PPW], sm2[PPW], starts[PPW], ends[PPW];
    int jl[PPW];
    Closure mpre[PPW];
#pragma unroll
    for (int c = 0; c < PPW; ++c) {
      const BlockMeta cur = ring[c][0];
#pragma unroll
      for (int j = 0; j + 1 < PD; ++j) ring[c][j] = ring[c][j + 1];
      ring[c][PD - 1] = meta(c, b - PD >= 0 ? b - PD : 0);  // consumed PD blocks from now
      r1[c] = cur.r1;
      r2[c] = cur.r2;
      r3[c] = cur.r3;
      const BlockBits bb = decode_bits<X>(cur, kb, a.words);
      sb[c] = bb.sb;
      sm1[c] = bb.sm1;
      sm2[c] = bb.sm2;
      starts[c] = bb.sb & ~((bb.sb << 1) | bb.sm1);
      ends[c] = bb.sb & ~((bb.sb >> 1) | (bb.after << (X - 1)));
      jl[c] = first_end(ends[c]);
      mpre[c] = prefetch_closure(Mcol[c] + (kb + (jl[c] > 0 ? jl[c] : 0)) * nx * 10,
                                 jl[c] >= 0 && kb + jl[c] < ny - 1 && ghosts[c]);
    }
    mbar_wait(&full[s], static_cast<uint32_t>((bi / S) & 1));
    const unsigned char* base = smem + s * L::bytes;
    const T* fld = reinterpret_cast<const T*>(base) +
                   (LG == 1 ? warp * PPW : wp * LG + ql) * X * 32 + cl;
    const double* cs = reinterpret_cast<const double*>(base + L::field);
    const double* id = reinterpret_cast<const double*>(base + L::field + L::coef) + cl;
    auto cfu = [&](int uu) -> Coef3 { return coef_soa<X>(cs, uu, cl); };

#pragma unroll
    for (int c = 0; c < PPW; ++c) restore(sa[c], r1[c], r2[c], r3[c]);
    double pv[PPW][X];
#pragma unroll
    for (int u = 0; u < X; ++u) {
      const Coef3 cu = cfu(u);
      double idu = 1.0;
      if constexpr (TR && IDC) idu = id[u * 32];
#pragma unroll
      for (int c = 0; c < PPW; ++c) {
        reset_if(sa[c], (starts[c] >> u) & 1u);
        double w = static_cast<double>(fld[(c * X + u) * 32]);
        if constexpr (TR && PRE) w *= __ldg(PREp[c] + (kb + u < ny ? kb + u : ny - 1) * nx);
        if constexpr (TR && IDC) w *= idu;
        pv[c][u] = sa[c].step(cu, w);
      }
    }

    const int rvalid = colok ? static_cast<int>(ny - kb < X ? ny - kb : X) : 0;
    T* dp[PPW];
#pragma unroll
    for (int c = 0; c < PPW; ++c) dp[c] = dst[c] + (kb + X - 1) * a.pitch;  // walked down
#pragma unroll
    for (int u = X - 1; u >= 0; --u) {
      const Coef3 cu = cfu(u);
      double idu = 1.0;
      if constexpr (!TR && IDC) idu = id[u * 32];
#pragma unroll
      for (int c = 0; c < PPW; ++c) {
        if ((ends[c] >> u) & 1u) {
          if (kb + u < ny - 1 && ghosts[c]) {
            const bool s1 = u >= 1 ? ((sb[c] >> (u >= 1 ? u - 1 : 0)) & 1u) : sm1[c];
            const bool s2 = s1 && (u >= 2 ? ((sb[c] >> (u >= 2 ? u - 2 : 0)) & 1u)
                                          : (u == 1 ? sm1[c] : sm2[c]));
            const Closure M =
                u == jl[c] ? mpre[c] : load_closure(Mcol[c] + (kb + u) * nx * 10);
            enter(sd[c], segment_entry<TR, X>(pv[c], u, r1[c], r2[c], r3[c], s1, s2, cu, cfu, M),
                  cu);
          } else {
            sd[c].reset();
          }
        }
        double o = sd[c].step(cu, cu.b * pv[c][u]);
        if constexpr (!TR && IDC) o *= idu;
        if constexpr (POST) o *= __ldg(POSTp[c] + (kb + u < ny ? kb + u : ny - 1) * nx);
        st_cs_if(dp[c], ((sb[c] >> u) & 1u) ? o : 0.0, act[c] && u < rvalid);
        dp[c] -= a.pitch;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

constexpr int kYc1NW = 16, kYc1U = 8, kYc1S = 4;
// C2 shapes (measured on C5 fp64, ncu): x 4 rows x 128 planes, 16 warps,
// 3 buffers (3.33 ms; 3 rows/4 buffers 3.47, 2 rows/5 buffers 4.26); y 12
// planes, 12 warps, 3 buffers (3.52 ms; 16 warps/2 buffers 3.81, 10/3
// 3.74, 8/4 3.83, 13/3 4.22)
template <typename T>
struct C2Shape {
  static constexpr bool f64 = sizeof(T) == 8;
  static constexpr int yNW = 8, yPPW = 1, yS = 2, yLG = 1;
  static constexpr int xR = 4, xNWR = 4, xS = 3;
  static constexpr int pR = 3, pNWR = 4, pS = 2;  // paired x tiles: 98 KB each
};
constexpr int kXc1NW = 4, kXc1S = 4;


// ------------------------------------------------------------- launchers
template <typename T>
int64_t ckpt_doubles(const StreamArgs& a) {
  const int64_t planes = a.nvar * a.nlev;
  if (a.dir == 0) return a.ny * ((a.nx + ck_x<T>() - 1) / ck_x<T>()) * 3 * planes;
  return planes * ((a.ny + ck_y<T>() - 1) / ck_y<T>()) * 3 * a.nx;
}

template <typename T, bool TR, bool IDC, bool VAR, int NW, int S>
void launch_xck1_shape(const T* in, const StreamArgs& a, double* ck, cudaStream_t st) {
  using L = XT<T, NW, false>;
  const size_t smem = S * L::bytes + 2 * S * sizeof(uint64_t) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_xck1<T, TR, IDC, VAR, NW, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    attr = true;
  }
  const int64_t planes = a.nvar * a.nlev;
  const uint64_t sz = sizeof(T);
  const uint64_t fd[3] = {uint64_t(a.nx), uint64_t(a.ny), uint64_t(planes)};
  const uint64_t fs[2] = {uint64_t(a.pitch) * sz, uint64_t(a.pitch * a.ny) * sz};
  const uint32_t fb[3] = {uint32_t(L::U), 1, uint32_t(32 * NW)};
  const CUtensorMap tin = make_tmap(in, tma_dtype<T>(), 3, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
  const uint64_t cd[2] = {uint64_t(4 * a.nx), uint64_t(a.ny)};
  const uint64_t cs[1] = {uint64_t(4 * a.nx) * 8};
  const uint32_t cb[2] = {uint32_t(4 * L::U), 1};
  const CUtensorMap tc =
      make_tmap(a.c3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, cd, cs, cb, CU_TENSOR_MAP_SWIZZLE_NONE);
  const uint64_t id[2] = {uint64_t(a.nx), uint64_t(a.ny)};
  const uint64_t is[1] = {uint64_t(a.ipitch) * 8};  // TMA: 16 B multiple
  const uint32_t ib[2] = {uint32_t(L::U), 1};
  const CUtensorMap ti = IDC ? make_tmap(a.idcp, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, id, is, ib,
                                         CU_TENSOR_MAP_SWIZZLE_NONE)
                             : tc;
  const int64_t PB = (planes + 32 * NW - 1) / (32 * NW);
  k_xck1<T, TR, IDC, VAR, NW, S><<<a.ny * PB, 32 * (NW + 1), smem, st>>>(a, ck, tin, tc, ti);
}

template <typename T, bool TR, bool IDC, bool VAR, int NW, int S>
void launch_xck1p_shape(const T* in, const StreamArgs& a, double* ck, cudaStream_t st) {
  using L = XT<T, NW, false>;
  constexpr int U = L::U;
  constexpr size_t PBYTES = (2 * (L::field + L::coef + L::idc) + 1023) / 1024 * 1024;
  const size_t smem = S * PBYTES + 2 * S * sizeof(uint64_t) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_xck1p<T, TR, IDC, VAR, NW, S>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  const int64_t planes = a.nvar * a.nlev;
  const uint64_t sz = sizeof(T);
  // dims (x within a block, block, row, plane): stages land as [plane][2][U]
  const uint64_t fd[4] = {uint64_t(U), uint64_t(a.nx / U), uint64_t(a.ny), uint64_t(planes)};
  const uint64_t fs[3] = {uint64_t(U) * sz, uint64_t(a.pitch) * sz, uint64_t(a.pitch * a.ny) * sz};
  const uint32_t fb[4] = {uint32_t(U), 2, 1, uint32_t(32 * NW)};
  const CUtensorMap tin = make_tmap(in, tma_dtype<T>(), 4, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  const uint64_t cd[2] = {uint64_t(4 * a.nx), uint64_t(a.ny)};
  const uint64_t cs[1] = {uint64_t(4 * a.nx) * 8};
  const uint32_t cb[2] = {uint32_t(4 * 2 * U), 1};
  const CUtensorMap tc =
      make_tmap(a.c3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, cd, cs, cb, CU_TENSOR_MAP_SWIZZLE_NONE);
  const uint64_t id[2] = {uint64_t(a.nx), uint64_t(a.ny)};
  const uint64_t is[1] = {uint64_t(a.ipitch) * 8};
  const uint32_t ib[2] = {uint32_t(2 * U), 1};
  const CUtensorMap ti = IDC ? make_tmap(a.idcp, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, id, is, ib,
                                         CU_TENSOR_MAP_SWIZZLE_NONE)
                             : tc;
  const int64_t PB = (planes + 32 * NW - 1) / (32 * NW);
  k_xck1p<T, TR, IDC, VAR, NW, S><<<a.ny * PB, 32 * (NW + 1), smem, st>>>(a, ck, tin, tc, ti);
}

template <typename T, bool TR, bool IDC, bool VAR>
void launch_xck1(const T* in, const StreamArgs& a, double* ck, cudaStream_t st) {
  static const bool pair_env = [] {
    const char* e = std::getenv("RGF_B200_XPAIR");
    return !(e && e[0] == '0');
  }();
  if (pair_env && a.nx % ck_x<T>() == 0) {  // paired stages: 256 B runs
    launch_xck1p_shape<T, TR, IDC, VAR, kXc1NW, 2>(in, a, ck, st);
    return;
  }
  // 4 stages, 3 CTAs/SM (1.75 ms on C5 fp64; 6 stages 1.90, 8 or 12 stages
  // at 1 CTA/SM ~3 ms)
  launch_xck1_shape<T, TR, IDC, VAR, kXc1NW, kXc1S>(in, a, ck, st);
}

template <typename T, bool TR, bool IDC, bool PRE, bool POST, int R, int NWR, int S>
void launch_xck2_shape(const T* in, T* out, const StreamArgs& a, const double* ck,
                       cudaStream_t st) {
  using L = XC2<T, R, NWR>;
  const size_t smem = S * L::bytes + 2 * S * sizeof(uint64_t) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_xck2<T, TR, IDC, PRE, POST, R, NWR, S>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  const int64_t planes = a.nvar * a.nlev;
  const uint64_t sz = sizeof(T);
  // dims (x, plane, row): box rows land in smem as [row][plane][x]
  const uint64_t fd[3] = {uint64_t(a.nx), uint64_t(planes), uint64_t(a.ny)};
  const uint64_t fs[2] = {uint64_t(a.pitch * a.ny) * sz, uint64_t(a.pitch) * sz};
  const uint32_t fb[3] = {uint32_t(L::U), uint32_t(32 * NWR), uint32_t(R)};
  const CUtensorMap tin = make_tmap(in, tma_dtype<T>(), 3, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
  const uint32_t fbo[3] = {uint32_t(L::U), 32, 1};  // one warp's part
  const CUtensorMap tout = make_tmap(out, tma_dtype<T>(), 3, fd, fs, fbo,
                                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
  const uint64_t cd[2] = {uint64_t(4 * a.nx), uint64_t(a.ny)};
  const uint64_t cs[1] = {uint64_t(4 * a.nx) * 8};
  const uint32_t cb[2] = {uint32_t(4 * L::X), uint32_t(R)};
  const CUtensorMap tc =
      make_tmap(a.c3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, cd, cs, cb, CU_TENSOR_MAP_SWIZZLE_NONE);
  const uint64_t id[2] = {uint64_t(a.nx), uint64_t(a.ny)};
  const uint64_t is[1] = {uint64_t(a.ipitch) * 8};  // TMA: 16 B multiple
  const uint32_t ib[2] = {uint32_t(L::X), uint32_t(R)};
  const CUtensorMap ti = IDC ? make_tmap(a.idcp, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, id, is, ib,
                                         CU_TENSOR_MAP_SWIZZLE_NONE)
                             : tc;
  const int64_t PB = (planes + 32 * NWR - 1) / (32 * NWR);
  const int64_t blocks = ((a.ny + R - 1) / R) * PB;
  k_xck2<T, TR, IDC, PRE, POST, R, NWR, S><<<blocks, 32 * R * NWR, smem, st>>>(a, ck, tin, tout,
                                                                               tc, ti);
}

template <typename T, bool TR, bool IDC, bool PRE, bool POST, int R, int NWR, int S>
void launch_xck2p_shape(const T* in, T* out, const StreamArgs& a, const double* ck,
                        cudaStream_t st) {
  using L = XC2<T, R, NWR>;
  constexpr int X = L::X;
  constexpr size_t TB = (2 * (L::sub + L::coef + L::idc) + 1023) / 1024 * 1024;
  const size_t smem = S * TB + 2 * S * sizeof(uint64_t) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_xck2p<T, TR, IDC, PRE, POST, R, NWR, S>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  const int64_t planes = a.nvar * a.nlev;
  const uint64_t sz = sizeof(T);
  // dims (x within a block, block, plane, row): tiles land as [row][plane][2][X]
  const uint64_t fd[4] = {uint64_t(X), uint64_t(a.nx / X), uint64_t(planes), uint64_t(a.ny)};
  const uint64_t fs[3] = {uint64_t(X) * sz, uint64_t(a.pitch * a.ny) * sz, uint64_t(a.pitch) * sz};
  const uint32_t fb[4] = {uint32_t(X), 2, uint32_t(32 * NWR), uint32_t(R)};
  const CUtensorMap tin = make_tmap(in, tma_dtype<T>(), 4, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  const uint32_t fbo[4] = {uint32_t(X), 2, 32, 1};  // one warp's part
  const CUtensorMap tout = make_tmap(out, tma_dtype<T>(), 4, fd, fs, fbo,
                                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  const uint64_t cd[2] = {uint64_t(4 * a.nx), uint64_t(a.ny)};
  const uint64_t cs[1] = {uint64_t(4 * a.nx) * 8};
  const uint32_t cb[2] = {uint32_t(4 * 2 * X), uint32_t(R)};
  const CUtensorMap tc =
      make_tmap(a.c3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, cd, cs, cb, CU_TENSOR_MAP_SWIZZLE_NONE);
  const uint64_t id[2] = {uint64_t(a.nx), uint64_t(a.ny)};
  const uint64_t is[1] = {uint64_t(a.ipitch) * 8};
  const uint32_t ib[2] = {uint32_t(2 * X), uint32_t(R)};
  const CUtensorMap ti = IDC ? make_tmap(a.idcp, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, id, is, ib,
                                         CU_TENSOR_MAP_SWIZZLE_NONE)
                             : tc;
  const int64_t PB = (planes + 32 * NWR - 1) / (32 * NWR);
  const int64_t blocks = ((a.ny + R - 1) / R) * PB;
  k_xck2p<T, TR, IDC, PRE, POST, R, NWR, S><<<blocks, 32 * R * NWR, smem, st>>>(a, ck, tin, tout,
                                                                                tc, ti);
}

template <typename T, bool TR, bool IDC, bool PRE, bool POST>
void launch_xck2(const T* in, T* out, const StreamArgs& a, const double* ck, cudaStream_t st) {
  // rows whole blocks long: paired tiles (256 B runs), unless RGF_B200_XPAIR=0
  static const bool pair_env = [] {
    const char* e = std::getenv("RGF_B200_XPAIR");
    return !(e && e[0] == '0');
  }();
  if (pair_env && a.nx % ck_x<T>() == 0) {
    launch_xck2p_shape<T, TR, IDC, PRE, POST, C2Shape<T>::pR, C2Shape<T>::pNWR, C2Shape<T>::pS>(
        in, out, a, ck, st);
    return;
  }
  launch_xck2_shape<T, TR, IDC, PRE, POST, C2Shape<T>::xR, C2Shape<T>::xNWR, C2Shape<T>::xS>(
      in, out, a, ck, st);
}

// paired coefficient map for the y kernels: [ny][2][nx][2] as dims
// {2, nx, 2, ny}, box {2, 32, 2, rows}
inline CUtensorMap coef_soa_map(const StreamArgs& a, uint32_t rows) {
  const uint64_t d[4] = {2, uint64_t(a.nx), 2, uint64_t(a.ny)};
  const uint64_t s[3] = {16, uint64_t(a.nx) * 16, uint64_t(a.nx) * 32};
  const uint32_t b[4] = {2, 32, 2, rows};
  return make_tmap(a.c3s, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, s, b, CU_TENSOR_MAP_SWIZZLE_NONE);
}

template <typename T, bool TR, bool IDC, bool VAR, int NW, int U, int S>
void launch_yck1_shape(const T* in, const StreamArgs& a0, double* ck, cudaStream_t st) {
  using L = YC1<T, NW, U>;
  const size_t smem = S * L::bytes + 2 * S * sizeof(uint64_t) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_yck1<T, TR, IDC, VAR, NW, U, S>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  const int64_t planes = a0.nvar * a0.nlev;
  StreamArgs a = a0;
  a.box_planes = static_cast<int>(planes < NW ? planes : NW);
  const uint64_t sz = sizeof(T);
  const uint64_t fd[3] = {uint64_t(a.nx), uint64_t(a.ny), uint64_t(planes)};
  const uint64_t fs[2] = {uint64_t(a.pitch) * sz, uint64_t(a.pitch * a.ny) * sz};
  const uint32_t fb[3] = {32, uint32_t(U), uint32_t(a.box_planes)};
  const CUtensorMap tf = make_tmap(in, tma_dtype<T>(), 3, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_NONE);
  const CUtensorMap tc = coef_soa_map(a, U);
  const uint64_t id[2] = {uint64_t(a.nx), uint64_t(a.ny)};
  const uint64_t is[1] = {uint64_t(a.ipitch) * 8};  // TMA: 16 B multiple
  const uint32_t ib[2] = {32, uint32_t(U)};
  const CUtensorMap ti = IDC ? make_tmap(a.idcp, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, id, is, ib,
                                         CU_TENSOR_MAP_SWIZZLE_NONE)
                             : tc;
  const int64_t blocks = ((a.nx + 31) / 32) * ((planes + NW - 1) / NW);
  k_yck1<T, TR, IDC, VAR, NW, U, S><<<blocks, 32 * (NW + 1), smem, st>>>(a, ck, tf, tc, ti);
}

// few planes (a single level: the reference's own 2-D operator, the CG
// solver): 4-plane CTAs with an 8-deep stage ring, so the serial walk down a
// column is not latency-bound on the box round trips
template <typename T, bool TR, bool IDC, bool VAR>
void launch_yck1(const T* in, const StreamArgs& a, double* ck, cudaStream_t st) {
  if (a.nvar * a.nlev <= 4)
    launch_yck1_shape<T, TR, IDC, VAR, 4, kYc1U, 12>(in, a, ck, st);
  else
    launch_yck1_shape<T, TR, IDC, VAR, kYc1NW, kYc1U, kYc1S>(in, a, ck, st);
}

template <typename T, bool TR, bool IDC, bool PRE, bool POST, int NW, int PPW, int S, int LG = 1,
          int PD = 1>
void launch_yck2_shape(const T* in, T* out, const StreamArgs& a0, const double* ck,
                       cudaStream_t st) {
  constexpr int NPL = NW * PPW;
  using L = YC2<T, NPL>;
  const size_t smem = S * L::bytes + 2 * S * sizeof(uint64_t) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_yck2<T, TR, IDC, PRE, POST, NW, PPW, S, LG, PD>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  const int64_t planes = a0.nvar * a0.nlev;
  StreamArgs a = a0;
  a.box_planes = static_cast<int>(planes < NPL ? planes : NPL);
  const uint64_t sz = sizeof(T);
  const uint64_t fd[3] = {uint64_t(a.nx), uint64_t(a.ny), uint64_t(planes)};
  const uint64_t fs[2] = {uint64_t(a.pitch) * sz, uint64_t(a.pitch * a.ny) * sz};
  const uint32_t fb[3] = {32, uint32_t(L::X), uint32_t(a.box_planes)};
  const CUtensorMap tf = make_tmap(in, tma_dtype<T>(), 3, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_NONE);
  const CUtensorMap tc = coef_soa_map(a, L::X);
  const uint64_t id[2] = {uint64_t(a.nx), uint64_t(a.ny)};
  const uint64_t is[1] = {uint64_t(a.ipitch) * 8};  // TMA: 16 B multiple
  const uint32_t ib[2] = {32, uint32_t(L::X)};
  const CUtensorMap ti = IDC ? make_tmap(a.idcp, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, id, is, ib,
                                         CU_TENSOR_MAP_SWIZZLE_NONE)
                             : tc;
  const int64_t blocks = ((a.nx + 31) / 32) * ((planes + NPL - 1) / NPL);
  k_yck2<T, TR, IDC, PRE, POST, NW, PPW, S, LG, PD><<<blocks, 32 * NW, smem, st>>>(out, a, ck, tf,
                                                                              tc, ti);
}

template <typename T, bool TR, bool IDC, bool PRE, bool POST>
void launch_yck2(const T* in, T* out, const StreamArgs& a, const double* ck, cudaStream_t st) {
  if (a.nvar * a.nlev <= 2) {  // few planes: 2-plane CTAs, 6 buffers in flight
    launch_yck2_shape<T, TR, IDC, PRE, POST, 2, 1, 6, 1, 4>(in, out, a, ck, st);
    return;
  }
  launch_yck2_shape<T, TR, IDC, PRE, POST, C2Shape<T>::yNW, C2Shape<T>::yPPW, C2Shape<T>::yS,
                    C2Shape<T>::yLG>(in, out, a, ck, st);
}

// runtime flags -> template flags; returns kernel launches
template <typename T, bool TR>
int launch_ck_dir(const T* in, T* out, const StreamArgs& a, double* ck, cudaStream_t st) {
  const bool idc = a.idc != nullptr;
  const bool pre = TR && a.pre_scale != nullptr;
  const bool post = a.post_scale != nullptr;
  const int64_t n = a.dir == 0 ? a.nx : a.ny;
  const int64_t X = a.dir == 0 ? ck_x<T>() : ck_y<T>();
  int launches = 0;
  // C1 (skipped when the line is a single block)
  if (n > X) {
    const bool i1 = TR && idc;
#define RGFB_C1(I, V)                                         \
  if (a.dir == 0) launch_xck1<T, TR, I, V>(in, a, ck, st);    \
  else launch_yck1<T, TR, I, V>(in, a, ck, st);
    if (i1) {
      if (pre) { RGFB_C1(true, true) } else { RGFB_C1(true, false) }
    } else {
      if (pre) { RGFB_C1(false, true) } else { RGFB_C1(false, false) }
    }
#undef RGFB_C1
    ++launches;
  }
#define RGFB_C2(I, P, Q)                                             \
  if (a.dir == 0) launch_xck2<T, TR, I, P, Q>(in, out, a, ck, st);   \
  else launch_yck2<T, TR, I, P, Q>(in, out, a, ck, st);
  if (idc) {
    if (pre) {
      if (post) { RGFB_C2(true, true, true) } else { RGFB_C2(true, true, false) }
    } else {
      if (post) { RGFB_C2(true, false, true) } else { RGFB_C2(true, false, false) }
    }
  } else {
    if (pre) {
      if (post) { RGFB_C2(false, true, true) } else { RGFB_C2(false, true, false) }
    } else {
      if (post) { RGFB_C2(false, false, true) } else { RGFB_C2(false, false, false) }
    }
  }
#undef RGFB_C2
  return launches + 1;
}

template <typename T>
int launch_ckpt_sweep(const T* in, T* out, const StreamArgs& a, double* ck, cudaStream_t st) {
  return a.transpose ? launch_ck_dir<T, true>(in, out, a, ck, st)
                     : launch_ck_dir<T, false>(in, out, a, ck, st);
}

// bits[dir] -> chain-minor words: x [lev][iy][w] -> [iy][w][lev];
// y [lev][ix][w] -> [lev][w][ix]
__global__ void k_bits_transpose(const uint64_t* __restrict__ bits, int dir, int64_t nx, int64_t ny,
                                 int64_t nlev, int64_t words, uint64_t* __restrict__ out) {
  const int64_t nlines = dir == 0 ? ny : nx;
  const int64_t total = nlev * nlines * words;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = t % words, ln = t / words;
    const int64_t lev = ln / nlines, line = ln - lev * nlines;
    const int64_t o = dir == 0 ? (line * words + w) * nlev + lev : (lev * words + w) * nlines + line;
    out[o] = bits[t];
  }
}

// AoS [nh][4] -> paired rows [ny][2][nx][2]: (a1, a2), (a3, b)
__global__ void k_coef_soa(const Coef3* __restrict__ c3, int64_t nx, int64_t ny,
                           double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nx * ny;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t y = t / nx, x = t - y * nx;
    const Coef3 c = c3[t];
    double* o = out + (y * 2 * nx + x) * 2;
    o[0] = c.a1;
    o[1] = c.a2;
    o[2 * nx] = c.a3;
    o[2 * nx + 1] = c.b;
  }
}

}  // namespace rgfb
