// Single-pass 3rd-RF sweeps ("ring" kernels): one field read and one field
// write per direction.
//
// The checkpointed sweep (sweep_ckpt.cuh) reads every element twice because
// a chain is walked in two kernels. Here a warp owns one line and 32 planes
// (x: one row x 32 planes; y: 16/8 planes x 2/4 adjacent columns) and walks
// it once, ascending, in blocks of X points staged by TMA into a per-warp
// ring of NSLOT shared-memory slots:
//
//  * causal recursion over block b (rf3.hpp:217-239; state reset at segment
//    starts = the reference's zero startup rows), the values kept in
//    registers;
//  * every segment that ENDS in block b is finished at once: the
//    anti-causal recursion (rf3.hpp:241-262) is entered from the right-ghost
//    closure M_j (closures.cuh; covariance.cpp:271-273 with the G ghost
//    steps collapsed) and runs down to the segment's start, through older
//    ring slots that still hold the segment's causal values;
//  * points of a segment that has not ended yet stay in the ring as causal
//    values; a block whose points are all final is returned with one TMA
//    store and its slot refilled.
//
// Lanes are planes of the same line, so with level-invariant masks (C3-C5)
// all lanes meet their segment ends together; with masks that differ per
// level (C2: land grows with depth) the warp runs the union of the lanes'
// ranges with per-lane predicates. A segment longer than the ring (rare:
// ~1% of C5 points) spills its oldest block's causal values to the output
// buffer and finishes those points from global memory later.
//
// The arithmetic per step is the checkpointed kernels' (same FMA order, same
// closure products); the adjoint (rf3.hpp:264-286) uses the same structure
// in gather form (AdjA2 / AdjD2). fp32 fields keep fp64 coefficients and
// registers; causal values parked in the ring are stored as T.
#pragma once
#include <climits>

#include "sweep_ckpt.cuh"

namespace rgfb {

// Section timers (compile with -DRGF_RING_PROF): cycles per section summed
// over warps, read back with rgf_debug_ring_prof().
#ifdef RGF_RING_PROF
__device__ unsigned long long g_ring_prof[8];
#define RING_T0() long long rp_t = clock64()
#define RING_TS(i)                                  \
  {                                                 \
    const long long rp_n = clock64();               \
    rp_acc[i] += static_cast<unsigned long long>(rp_n - rp_t); \
    rp_t = rp_n;                                    \
  }
#else
#define RING_T0()
#define RING_TS(i)
#endif

template <typename T, int DIR>
struct RingL {
  static constexpr int X = 128 / int(sizeof(T));                // points per block
  static constexpr int K = DIR == 0 ? 1 : 16 / int(sizeof(T));  // lines per warp
  static constexpr int P = 32 / K;                              // planes per warp
  static constexpr int FB = X * 32 * int(sizeof(T));            // field slot: 4 KB
  static constexpr int CB = X * K * int(sizeof(Coef3));         // coefficient slot
  static constexpr int IB = X * K * 8;                          // inv_dc slot
};
template <typename T, int DIR, bool IDC, int NSLOT>
constexpr size_t ring_warp_bytes() {
  using L = RingL<T, DIR>;
  return (size_t(NSLOT) * (L::FB + L::CB + (IDC ? L::IB : 0)) + size_t(NSLOT) * 12 + 1023) / 1024 *
         1024;
}

// lane's X values of a field slot. x: [32 planes][128 B], 128 B swizzled
// (lane = plane reads 16 B chunks conflict-free); y: [X rows][32 lanes].
template <typename T, int DIR, int X>
__device__ __forceinline__ void ring_ld(const unsigned char* fs, int lane, double (&v)[X]) {
  if constexpr (DIR == 0) {
    constexpr int EPC = 16 / int(sizeof(T));
    const unsigned char* rowp = fs + lane * 128;
    const int sw = lane & 7;
#pragma unroll
    for (int q = 0; q < X / EPC; ++q) {
      const void* cp = rowp + ((q ^ sw) << 4);
      if constexpr (sizeof(T) == 8) {
        const double2 t = *reinterpret_cast<const double2*>(cp);
        v[2 * q] = t.x;
        v[2 * q + 1] = t.y;
      } else {
        const float4 t = *reinterpret_cast<const float4*>(cp);
        v[4 * q] = t.x;
        v[4 * q + 1] = t.y;
        v[4 * q + 2] = t.z;
        v[4 * q + 3] = t.w;
      }
    }
  } else {
    const T* f = reinterpret_cast<const T*>(fs) + lane;
#pragma unroll
    for (int u = 0; u < X; ++u) v[u] = static_cast<double>(f[u * 32]);
  }
}
template <typename T, int DIR, int X>
__device__ __forceinline__ void ring_st(unsigned char* fs, int lane, const double (&v)[X]) {
  if constexpr (DIR == 0) {
    constexpr int EPC = 16 / int(sizeof(T));
    unsigned char* rowp = fs + lane * 128;
    const int sw = lane & 7;
#pragma unroll
    for (int q = 0; q < X / EPC; ++q) {
      void* cp = rowp + ((q ^ sw) << 4);
      if constexpr (sizeof(T) == 8) {
        *reinterpret_cast<double2*>(cp) = make_double2(v[2 * q], v[2 * q + 1]);
      } else {
        *reinterpret_cast<float4*>(cp) =
            make_float4(static_cast<float>(v[4 * q]), static_cast<float>(v[4 * q + 1]),
                        static_cast<float>(v[4 * q + 2]), static_cast<float>(v[4 * q + 3]));
      }
    }
  } else {
    T* f = reinterpret_cast<T*>(fs) + lane;
#pragma unroll
    for (int u = 0; u < X; ++u) f[u * 32] = static_cast<T>(v[u]);
  }
}

// block bits of one lane: sea bits, starts, ends (+ the two bits before)
struct RingBits {
  uint32_t sb, sm1, sm2, after;
};

template <typename T, int DIR, bool TR, bool IDC, bool PRE, bool POST, int NW, int NSLOT>
__global__ void __launch_bounds__(32 * NW)
    k_ring(T* __restrict__ out, StreamArgs a, const __grid_constant__ CUtensorMap tm_in,
           const __grid_constant__ CUtensorMap tm_out, const __grid_constant__ CUtensorMap tm_coef,
           const __grid_constant__ CUtensorMap tm_idc) {
  using L = RingL<T, DIR>;
  constexpr int X = L::X, K = L::K, P = L::P;
  constexpr int FB = L::FB, CB = L::CB, IB = IDC ? L::IB : 0;
  constexpr size_t WB = ring_warp_bytes<T, DIR, IDC, NSLOT>();
  constexpr uint32_t MSK = X == 32 ? 0xffffffffu : ((1u << X) - 1u);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* fld = smem + warp * WB;  // NSLOT field slots
  unsigned char* cfs = fld + NSLOT * FB;  // NSLOT coefficient slots
  unsigned char* ids = cfs + NSLOT * CB;  // NSLOT inv_dc slots
  uint64_t* full = reinterpret_cast<uint64_t*>(ids + NSLOT * IB);

  const int64_t nx = a.nx, ny = a.ny, nh = nx * ny;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t PG = (planes + P - 1) / P;
  const int64_t lines = DIR == 0 ? ny : (nx + K - 1) / K;
  const int64_t unit = static_cast<int64_t>(blockIdx.x) * NW + warp;
  if (unit >= lines * PG) return;  // warp-uniform; nothing CTA-wide follows
  const int64_t ln = unit / PG, pg = unit - ln * PG;
  const int64_t p0 = pg * P;
  const int n = static_cast<int>(DIR == 0 ? nx : ny);
  const int NB = (n + X - 1) / X;
  const int lp = lane / K, lc = lane % K;
  const int64_t iy = DIR == 0 ? ln : 0;
  const int64_t ix0 = DIR == 0 ? 0 : ln * K;
  const int64_t ix = ix0 + lc;
  const bool act = p0 + lp < planes && (DIR == 0 || ix < nx);
  const int64_t p = p0 + (p0 + lp < planes ? lp : 0);
  const int64_t ixc = DIR == 0 ? 0 : (ix < nx ? ix : nx - 1);
  const int64_t lev = a.lev0 + p % a.nlev;
  const uint64_t* W = DIR == 0 ? a.bitsT + iy * a.words * a.nlev_all + lev
                               : a.bitsT + lev * a.words * nx + ixc;
  const int64_t ws = DIR == 0 ? a.nlev_all : nx;
  const int64_t hb = DIR == 0 ? iy * nx : ixc;  // horizontal index of line position i: hb + i*hs
  const int64_t hs = DIR == 0 ? 1 : nx;
  T* gp = out + (DIR == 0 ? (p * ny + iy) * a.pitch : p * ny * a.pitch + ixc);
  const int64_t gs = DIR == 0 ? 1 : a.pitch;
  const double* PREp = PRE ? a.pre_scale + lev * nh + hb : nullptr;
  const double* POSTp = POST ? a.post_scale + lev * nh + hb : nullptr;
  const double* Mb = a.clos + clos_off(a.cls[lev], DIR, TR ? 1 : 0, nh, hb);
  const int64_t Ms = hs * 10;
  const bool ghosts = a.ghost[lev] > 0;
  const int64_t words = a.words;

  if (lane == 0) {
    for (int s = 0; s < NSLOT; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
    tma_prefetch_desc(&tm_in);
    tma_prefetch_desc(&tm_coef);
  }
  __syncwarp();

  int loaded = 0;   // next block to load
  int ob = 0;       // oldest block still held in the ring (not stored, not spilled)
  // y: a warp's field rows are 16-32 B wide; the neighbouring columns' warps
  // read the rest of each sector soon after, so y data stays evict-normal
  const uint64_t pol_stream = DIR == 0 ? l2_evict_first() : l2_evict_normal();
  const uint64_t pol_keep = l2_evict_last();
  auto issue_load = [&](int k) {  // lane 0
    const int s = k % NSLOT;
    mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(FB + CB + IB));
    const int kb = k * X;
    if constexpr (DIR == 0) {
      tma_load_3d(fld + s * FB, &tm_in, kb, static_cast<int>(p0), static_cast<int>(iy), &full[s],
                  pol_stream);
      tma_load_2d(cfs + s * CB, &tm_coef, 4 * kb, static_cast<int>(iy), &full[s], pol_keep);
      if constexpr (IDC)
        tma_load_2d(ids + s * IB, &tm_idc, kb, static_cast<int>(iy), &full[s], pol_keep);
    } else {
      tma_load_3d(fld + s * FB, &tm_in, static_cast<int>(ix0), static_cast<int>(p0), kb, &full[s],
                  pol_stream);
      tma_load_2d(cfs + s * CB, &tm_coef, static_cast<int>(4 * ix0), kb, &full[s], pol_keep);
      if constexpr (IDC)
        tma_load_2d(ids + s * IB, &tm_idc, static_cast<int>(ix0), kb, &full[s], pol_keep);
    }
  };
  // Block k of the ring back to global memory with generic 16 B stores, read
  // out of the slot transposed so one warp store covers whole 128 B lines
  // (x: 4 planes x 128 B; y: 2 rows x 16 planes x 16 B). Finished blocks and
  // ring overflow (spill: pending lanes park their causal values in `out`)
  // take the same path; no async-proxy store, hence no proxy fence.
  auto store_block = [&](int k) {
    const unsigned char* f = fld + (k % NSLOT) * FB;
    const int kb = k * X;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int q = i * 32 + lane;
      int4 v;
      T* g;
      bool on;
      if constexpr (DIR == 0) {  // chunk c of plane row pl
        const int pl = q >> 3, c = q & 7;
        v = *reinterpret_cast<const int4*>(f + pl * 128 + ((c ^ (pl & 7)) << 4));
        const int e = kb + c * (16 / int(sizeof(T)));
        on = p0 + pl < planes && e < n;
        g = out + ((p0 + (on ? pl : 0)) * ny + iy) * a.pitch + (on ? e : 0);
      } else {  // plane pl's K columns in slot row r
        const int r = q / P, pl = q % P;
        v = *reinterpret_cast<const int4*>(f + r * 32 * int(sizeof(T)) + pl * 16);
        on = p0 + pl < planes && kb + r < n && ix0 < nx;
        g = out + ((p0 + (on ? pl : 0)) * ny + (on ? kb + r : 0)) * a.pitch + ix0;
      }
      if (on) *reinterpret_cast<int4*>(g) = v;
    }
    __syncwarp();
  };
  auto cfl = [&](const unsigned char* cs, int u) -> Coef3 {
    return lds_coef(reinterpret_cast<const Coef3*>(cs) + (DIR == 0 ? u : u * K + lc));
  };
  auto idl = [&](const unsigned char* is, int u) -> double {
    return reinterpret_cast<const double*>(is)[DIR == 0 ? u : u * K + lc];
  };
  auto clampi = [&](int i) -> int64_t { return i < n ? i : n - 1; };

  // mask window: words wi-1, wi, wi+1 of the lane's line (wi+1 arrived a
  // word ago; wi+2 is in flight), so no bit extraction waits on a load
  uint64_t wprev = 0, wcur = ldw(W, 0), wnxt = words > 1 ? ldw(W, ws) : 0ull;
  uint64_t wraw = ldw(W, (words > 2 ? 2 : words - 1) * ws);
  int64_t wi = 0;
  auto bits_of = [&](int kb) -> RingBits {  // block at kb within words wi, wi+1
    const int64_t w = kb >> 6;
    const uint64_t c = w == wi ? wcur : wnxt;
    const uint64_t pv = w == wi ? wprev : wcur;
    const uint64_t nx2 = w == wi ? wnxt : 0ull;  // after-bit of a block ending word wi
    const int off = kb & 63;
    RingBits r;
    r.sb = static_cast<uint32_t>(c >> off) & MSK;
    r.sm1 = off ? static_cast<uint32_t>(c >> (off - 1)) & 1u : static_cast<uint32_t>(pv >> 63);
    r.sm2 = off ? static_cast<uint32_t>(c >> (off - 2)) & 1u
                : static_cast<uint32_t>(pv >> 62) & 1u;
    r.after = off + X < 64 ? static_cast<uint32_t>(c >> (off + X)) & 1u
                           : static_cast<uint32_t>(nx2) & 1u;
    return r;
  };
  auto ends_of = [&](const RingBits& r) -> uint32_t {
    return r.sb & ~((r.sb >> 1) | (r.after << (X - 1)));
  };
  // closure of the highest segment end of block k (predicated prefetch)
  // (mpos: the line position it was fetched for, -1 if none)
  auto prefetch_for = [&](int k, uint32_t e, int& mpos) -> Closure {
    const int j = first_end(e);
    const int pos = k * X + (j > 0 ? j : 0);
    const bool on = k < NB && j >= 0 && pos < n - 1 && ghosts;
    mpos = on ? pos : -1;
    return prefetch_closure(Mb + static_cast<int64_t>(pos < n ? pos : 0) * Ms, on);
  };
  // closures fetched PFD blocks ahead (PFD+1 blocks fit in words wi, wi+1)
  constexpr int PFD = 64 / X / 2;
  Closure mq[PFD];
  int mqpos[PFD];
#pragma unroll
  for (int d = 0; d < PFD; ++d)
    mq[d] = prefetch_for(d, d < NB ? ends_of(bits_of(d * X)) : 0u, mqpos[d]);

  typename std::conditional<TR, AdjA2, FwdA2>::type sa;
  typename std::conditional<TR, AdjD2, FwdD2>::type sd;
  int segst = 0;  // start of the lane's current (latest) segment
  int fin = 0;    // every line position < fin is final (in the ring or in global memory)

#ifdef RGF_RING_PROF
  unsigned long long rp_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  RING_T0();
  for (int b = 0; b < NB; ++b) {
    const int kb = b * X;
    // ---- keep the ring fed; spill the oldest blocks if block b has no slot
    while (loaded < NB && loaded - NSLOT < ob) {
      if (lane == 0) issue_load(loaded);
      ++loaded;
    }
    while (loaded <= b) {
      while (loaded - NSLOT >= ob) store_block(ob++);  // spill
      if (lane == 0) issue_load(loaded);
      ++loaded;
    }
    RING_TS(0)
    // ---- mask bits of this block and the next (closure prefetch)
    if ((kb >> 6) != wi) {
      wi = kb >> 6;
      wprev = wcur;
      wcur = wnxt;
      wnxt = wi + 1 < words ? wraw : 0ull;
      const int64_t w2 = wi + 2 < words ? wi + 2 : words - 1;
      wraw = ldw(W, w2 * ws);
    }
    const RingBits rb = bits_of(kb);
    const uint32_t sb = rb.sb;
    const uint32_t starts = sb & ~((sb << 1) | rb.sm1);
    const uint32_t ends = ends_of(rb);
    const int jl = first_end(ends);
    int mpos_next;
    const Closure mnext =
        prefetch_for(b + PFD, b + PFD < NB ? ends_of(bits_of(kb + PFD * X)) : 0u, mpos_next);
    const int mpos = mqpos[0];

    const int s = b % NSLOT;
    unsigned char* fs = fld + s * FB;
    const unsigned char* cs = cfs + s * CB;
    const unsigned char* is = ids + s * IB;
    RING_TS(1)
    mbar_wait(&full[s], static_cast<uint32_t>((b / NSLOT) & 1));
    RING_TS(2)

    // ---- causal recursion over the block (values in registers)
    const double4 rin = sa.raw();  // raw state entering the block
    double pv[X];
    {
      double v[X];
      ring_ld<T, DIR, X>(fs, lane, v);
      // coefficient loads are issued two steps ahead (volatile: in this order)
      Coef3 ca = cfl(cs, 0), cb = cfl(cs, 1);
      if (__any_sync(0xffffffffu, starts != 0u)) {
#pragma unroll
        for (int u = 0; u < X; ++u) {
          const Coef3 cc = cfl(cs, u + 2 < X ? u + 2 : X - 1);
          reset_if(sa, (starts >> u) & 1u);
          double w = v[u];
          if constexpr (TR && PRE) w = __dmul_rn(w, __ldg(PREp + clampi(kb + u) * hs));
          if constexpr (TR && IDC) w = __dmul_rn(w, idl(is, u));
          pv[u] = sa.step(ca, w);
          ca = cb;
          cb = cc;
        }
      } else {  // no segment starts in this block (most blocks): no resets
#pragma unroll
        for (int u = 0; u < X; ++u) {
          const Coef3 cc = cfl(cs, u + 2 < X ? u + 2 : X - 1);
          double w = v[u];
          if constexpr (TR && PRE) w = __dmul_rn(w, __ldg(PREp + clampi(kb + u) * hs));
          if constexpr (TR && IDC) w = __dmul_rn(w, idl(is, u));
          pv[u] = sa.step(ca, w);
          ca = cb;
          cb = cc;
        }
      }
    }
    if (starts) segst = kb + 31 - __clz(starts);
    RING_TS(3)

    // ---- segments ending in this block: anti-causal recursion from their ends
    const bool any = __any_sync(0xffffffffu, ends != 0u);
    double o[X];
    if (any) {
      auto cfu = [&](int uu) -> Coef3 { return cfl(cs, uu); };
      sd.reset();
      Coef3 ca = cfl(cs, X - 1), cb = cfl(cs, X - 2);
#pragma unroll
      for (int u = X - 1; u >= 0; --u) {
        const Coef3 c = ca;
        const Coef3 cc = cfl(cs, u >= 2 ? u - 2 : 0);
        ca = cb;
        cb = cc;
        if ((ends >> u) & 1u) {
          if (kb + u < n - 1 && ghosts) {
            const bool s1 = u >= 1 ? ((sb >> (u >= 1 ? u - 1 : 0)) & 1u) : rb.sm1;
            const bool s2 =
                s1 && (u >= 2 ? ((sb >> (u >= 2 ? u - 2 : 0)) & 1u) : (u == 1 ? rb.sm1 : rb.sm2));
            const Closure M =
                kb + u == mpos ? mq[0] : load_closure(Mb + static_cast<int64_t>(kb + u) * Ms);
            enter(sd, segment_entry<TR, X>(pv, u, rin.x, rin.y, rin.z, s1, s2, c, cfu, M), c);
          } else {
            sd.reset();
          }
        }
        double ov = sd.step(c, c.b * pv[u]);
        if constexpr (!TR && IDC) ov *= idl(is, u);
        if constexpr (POST) ov *= __ldg(POSTp + clampi(kb + u) * hs);
        const bool sea = (sb >> u) & 1u;
        o[u] = sea ? (jl >= u ? ov : pv[u]) : 0.0;
      }
      ring_st<T, DIR, X>(fs, lane, o);
    } else if (__all_sync(0xffffffffu, sb == MSK)) {
      ring_st<T, DIR, X>(fs, lane, pv);  // all sea, nothing final yet
    } else {
#pragma unroll
      for (int u = 0; u < X; ++u) o[u] = ((sb >> u) & 1u) ? pv[u] : 0.0;
      ring_st<T, DIR, X>(fs, lane, o);
    }

    RING_TS(4)
    // ---- ... and down through the older blocks of those segments
    const bool fl = jl >= 0;
    const int mfin = static_cast<int>(
        __reduce_min_sync(0xffffffffu, static_cast<unsigned>(fl && act ? fin : INT_MAX)));
    if (any && mfin < kb) {
      for (int k = b - 1; k >= mfin / X; --k) {
        const int kk = k * X;
        if (k >= ob) {  // still in the ring
          const int s2 = k % NSLOT;
          unsigned char* f2 = fld + s2 * FB;
          const unsigned char* c2 = cfs + s2 * CB;
          const unsigned char* i2 = ids + s2 * IB;
          double v[X];
          ring_ld<T, DIR, X>(f2, lane, v);
          Coef3 ca = cfl(c2, X - 1), cb = cfl(c2, X - 2);
#pragma unroll
          for (int u = X - 1; u >= 0; --u) {
            const Coef3 c = ca;
            const Coef3 cc = cfl(c2, u >= 2 ? u - 2 : 0);
            ca = cb;
            cb = cc;
            double ov = sd.step(c, c.b * v[u]);
            if constexpr (!TR && IDC) ov *= idl(i2, u);
            if constexpr (POST) ov *= __ldg(POSTp + static_cast<int64_t>(kk + u) * hs);
            v[u] = (fl && kk + u >= fin) ? ov : v[u];
          }
          ring_st<T, DIR, X>(f2, lane, v);
        } else {  // spilled: causal values in global memory (all loads first)
          double v[X];
#pragma unroll
          for (int u = 0; u < X; ++u) v[u] = static_cast<double>(gp[static_cast<int64_t>(kk + u) * gs]);
#pragma unroll
          for (int u = X - 1; u >= 0; --u) {
            const int64_t i = kk + u;
            const Coef3 c = ldc(a.c3 + hb + i * hs);
            double ov = sd.step(c, c.b * v[u]);
            if constexpr (!TR && IDC) ov *= __ldg(a.idc + hb + i * hs);
            if constexpr (POST) ov *= __ldg(POSTp + i * hs);
            v[u] = ov;
          }
          if (act && fl) {
#pragma unroll
            for (int u = 0; u < X; ++u)
              if (kk + u >= fin) gp[static_cast<int64_t>(kk + u) * gs] = static_cast<T>(v[u]);
          }
        }
      }
    }

    RING_TS(5)
    // ---- bookkeeping: what is final, return finished blocks
    const bool open = ((sb >> (X - 1)) & 1u) && rb.after;
    fin = open ? segst : kb + X;
    const int m = static_cast<int>(
        __reduce_min_sync(0xffffffffu, static_cast<unsigned>(act ? fin : INT_MAX)));
    __syncwarp();
    while (ob <= b && (ob + 1) * X <= m) store_block(ob++);
#pragma unroll
    for (int d = 0; d + 1 < PFD; ++d) {
      mq[d] = mq[d + 1];
      mqpos[d] = mqpos[d + 1];
    }
    mq[PFD - 1] = mnext;
    mqpos[PFD - 1] = mpos_next;
    RING_TS(6)
  }
#ifdef RGF_RING_PROF
  if (lane == 0) {
    RING_TS(7)
    for (int i = 0; i < 8; ++i) atomicAdd(&g_ring_prof[i], rp_acc[i]);
  }
#endif
}

// ------------------------------------------------------------- launchers
// Shapes: four independent warps per CTA (one per SM sub-partition), one CTA
// per SM. Measured on C5 fp64 x (ncu / clock64 section timers):
// 1 warp x 15 slots x 3 CTAs/SM 8.5 ms, 4 warps x 11 slots 7.2 ms, 4 warps x
// 5 slots x 2 CTAs/SM 6.9 ms (26% of points spilled): the kernel issues
// ~1000 instructions per 16-point block at ~1.2 IPC per SM whatever the warp
// count, against 5.1 ms for the checkpointed pair. Kept as an experimental
// path (RGF_B200_SWEEP=ring).
template <typename T, int DIR>
struct RingShape {
  static constexpr int NW = 4;
  static constexpr int NSLOT = DIR == 0 ? (sizeof(T) == 8 ? 11 : 9) : (sizeof(T) == 8 ? 9 : 5);
};

template <typename T, int DIR, bool TR, bool IDC, bool PRE, bool POST>
void launch_ring_dir(const T* in, T* out, const StreamArgs& a, cudaStream_t st) {
  constexpr int NW = RingShape<T, DIR>::NW, NSLOT = RingShape<T, DIR>::NSLOT;
  using L = RingL<T, DIR>;
  constexpr size_t smem = NW * ring_warp_bytes<T, DIR, IDC, NSLOT>() + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ring<T, DIR, TR, IDC, PRE, POST, NW, NSLOT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  const int64_t planes = a.nvar * a.nlev;
  const uint64_t sz = sizeof(T);
  // field dims (x, plane, row)
  const uint64_t fd[3] = {uint64_t(a.nx), uint64_t(planes), uint64_t(a.ny)};
  const uint64_t fs[2] = {uint64_t(a.pitch * a.ny) * sz, uint64_t(a.pitch) * sz};
  const uint32_t fb[3] = {DIR == 0 ? uint32_t(L::X) : uint32_t(L::K), uint32_t(L::P),
                          DIR == 0 ? 1u : uint32_t(L::X)};
  const CUtensorMapSwizzle sw = DIR == 0 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
  // y boxes are K columns (16-32 B) wide: no L2 promotion (a 128 B fill per
  // 16 B row read the field 8 times over)
  const CUtensorMapL2promotion pr =
      DIR == 0 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  const CUtensorMap tin = make_tmap(in, tma_dtype<T>(), 3, fd, fs, fb, sw, pr);
  const CUtensorMap tout = make_tmap(out, tma_dtype<T>(), 3, fd, fs, fb, sw, pr);
  const uint64_t cd[2] = {uint64_t(4 * a.nx), uint64_t(a.ny)};
  const uint64_t cst[1] = {uint64_t(4 * a.nx) * 8};
  const uint32_t cb[2] = {DIR == 0 ? uint32_t(4 * L::X) : uint32_t(4 * L::K),
                          DIR == 0 ? 1u : uint32_t(L::X)};
  const CUtensorMap tc =
      make_tmap(a.c3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, cd, cst, cb, CU_TENSOR_MAP_SWIZZLE_NONE);
  const uint64_t id[2] = {uint64_t(a.nx), uint64_t(a.ny)};
  const uint64_t is[1] = {uint64_t(a.ipitch) * 8};  // TMA: 16 B multiple
  const uint32_t ib[2] = {DIR == 0 ? uint32_t(L::X) : uint32_t(L::K),
                          DIR == 0 ? 1u : uint32_t(L::X)};
  const CUtensorMap ti = IDC ? make_tmap(a.idcp, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, id, is, ib,
                                         CU_TENSOR_MAP_SWIZZLE_NONE)
                             : tc;
  const int64_t PG = (planes + L::P - 1) / L::P;
  const int64_t lines = DIR == 0 ? a.ny : (a.nx + L::K - 1) / L::K;
  const int64_t blocks = (lines * PG + NW - 1) / NW;
  k_ring<T, DIR, TR, IDC, PRE, POST, NW, NSLOT><<<blocks, 32 * NW, smem, st>>>(out, a, tin, tout,
                                                                               tc, ti);
}

template <typename T, bool TR>
int launch_ring_tr(const T* in, T* out, const StreamArgs& a, cudaStream_t st) {
  const bool idc = a.idc != nullptr;
  const bool pre = TR && a.pre_scale != nullptr;
  const bool post = a.post_scale != nullptr;
#define RGFB_RING(I, P, Q)                                          \
  if (a.dir == 0) launch_ring_dir<T, 0, TR, I, P, Q>(in, out, a, st); \
  else launch_ring_dir<T, 1, TR, I, P, Q>(in, out, a, st);
  if (idc) {
    if (pre) {
      if (post) { RGFB_RING(true, true, true) } else { RGFB_RING(true, true, false) }
    } else {
      if (post) { RGFB_RING(true, false, true) } else { RGFB_RING(true, false, false) }
    }
  } else {
    if (pre) {
      if (post) { RGFB_RING(false, true, true) } else { RGFB_RING(false, true, false) }
    } else {
      if (post) { RGFB_RING(false, false, true) } else { RGFB_RING(false, false, false) }
    }
  }
#undef RGFB_RING
  return 1;
}

// one directional sweep, one launch; returns kernel launches
template <typename T>
int launch_ring_sweep(const T* in, T* out, const StreamArgs& a, cudaStream_t st) {
  return a.transpose ? launch_ring_tr<T, true>(in, out, a, st)
                     : launch_ring_tr<T, false>(in, out, a, st);
}

}  // namespace rgfb
