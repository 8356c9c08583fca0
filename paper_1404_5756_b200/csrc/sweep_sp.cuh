// Single-pass 3rd-RF x-sweep: one field read and one field write per sweep.
//
// A row (x-line) of every plane is cut into CS chunks of at most RC points,
// one chunk per CTA of a thread-block cluster (cluster = one row x one plane
// group, CTA rank = chunk). Lanes are planes, so with level-invariant masks
// (one mask class, one ghost width: C1, C3-C5) the masks, segment ends,
// coefficients and every table below are warp-uniform broadcast reads.
//
// The reference's per-segment sequence (covariance.cpp:271-349: causal
// recursion rf3.hpp:217-239 from a zero state at the segment start, the right
// ghosts collapsed into the closure M_j at the segment end, anti-causal
// recursion rf3.hpp:241-262, unit-DC, land = 0) is linear in the data, so a
// chunk only needs two 3-vectors from outside:
//   S_c  the raw causal state entering the chunk (from the chunks on the left)
//   T_c  the raw anti-causal state entering it from the right.
// Per CTA:
//   F0  causal recursion over the chunk (staged in shared memory by TMA, one
//       mbarrier per 16-point sub-tile so it starts on the first sub-tile),
//       zero entry state; p is kept in shared memory in place of the input.
//       Its exit state b_c is published in shared memory.
//   cluster barrier 1; S_c = fold over j < c of S <- A_j S + b_j (DSMEM
//       reads of the peers' b_j; A_j = the chunk's homogeneous causal
//       transfer, precomputed).
//   p += Phi S_c over the chunk's first segment (Phi: homogeneous causal
//       response to S, precomputed; zero after the first segment start).
//   B0  anti-causal recursion down the chunk with a zero entry state, closure
//       entries at segment ends from the now exact p (and S_c for the two
//       points before the chunk). Exit state e_c published.
//   cluster barrier 2; T_c = fold over j > c of T <- B_j T + e_j.
//   o += Psi T_c over the chunk's last segment (Psi: homogeneous anti-causal
//       response to T), unit-DC / variance, land = 0, TMA store.
// A_j, B_j, Phi, Psi and the chunk's closure rows depend only on the
// coefficients and the mask, so they are built once per operator
// (k_xsp_tables) with the same state arithmetic as the kernel. Field traffic:
// one read and one write; everything else is per (row, x) and shared by the
// plane group (and by the cluster's row through L2).
#pragma once
#include "sweep_ckpt.cuh"

namespace rgfb {

namespace sp {
constexpr int NW = 4;             // warps per CTA; each owns a sub-chunk of RW points
constexpr int RCMAX = 272;        // max points per CTA chunk (17 sub-tiles of 16)
constexpr int NSUB = RCMAX / 16;  // TMA sub-tiles per CTA
constexpr int MAXE = 12;          // closure rows staged per sub-chunk (more: read from L2)
constexpr int CHKW = 24;          // per sub-chunk: A[9], B[9], phi_len, psi_start, nends, pad
constexpr int MAXCS = 16;         // CTAs per row (non-portable cluster size)
constexpr int SUBB = 32 * 128;    // sub-tile bytes: 32 plane slots x 16 doubles

struct Layout {
  static constexpr size_t tile = size_t(NSUB) * SUBB;
  static constexpr size_t coef = tile;
  static constexpr size_t idc = coef + size_t(RCMAX) * 32;
  static constexpr size_t tab = idc + size_t(RCMAX) * 8;          // [u][6]: Phi, Psi
  static constexpr size_t chk = tab + size_t(RCMAX) * 48;         // this CTA's sub-chunks
  static constexpr size_t ccta = chk + size_t(NW) * CHKW * 8;     // the row's CTA transfers
  static constexpr size_t cl = ccta + size_t(MAXCS) * CHKW * 8;   // closures per sub-chunk
  static constexpr size_t xw = cl + size_t(NW) * MAXE * 80;       // warp exits [w][lane][6]
  static constexpr size_t xc = xw + size_t(NW) * 32 * 48;         // CTA exits [lane][6]
  static constexpr size_t words = xc + 32 * 48;                   // mask words
  static constexpr size_t bars = words + 16 * 8;
  static constexpr size_t bytes = bars + (NSUB + 1) * 8;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// a double in CTA `rank`'s shared memory at the address of `local` in ours
__device__ __forceinline__ double ld_peer(const double* local, uint32_t rank) {
  uint32_t r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
  double v;  // volatile: kept after the cluster barrier; no clobber, so loads batch
  asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(r));
  return v;
}

// raw anti-causal state: what the chunk on the left needs to continue
// (forward: q_{k+1..k+3}; adjoint: pending sums into u_k, u_{k-1}, u_{k-2})
__device__ __forceinline__ void restore_d(FwdD2& s, double t0, double t1, double t2) {
  s.q1 = t0;
  s.q2 = t1;
  s.q3 = t2;
}
__device__ __forceinline__ void restore_d(AdjD2& s, double t0, double t1, double t2) {
  s.U1 = 0.0;
  s.X1 = 0.0;
  s.Y22 = 0.0;
  s.Y21 = 0.0;
  s.Y33 = t0;
  s.Y32 = t1;
  s.Y31 = t2;
}
__device__ __forceinline__ double3 raw_d(const FwdD2& s) { return make_double3(s.q1, s.q2, s.q3); }
__device__ __forceinline__ double3 raw_d(const AdjD2& s) {
  return make_double3(fma(s.X1, s.U1, s.Y33 + s.Y22), s.Y32 + s.Y21, s.Y31);
}
__device__ __forceinline__ double3 raw_a(const FwdA2& s) { return make_double3(s.p1, s.p2, s.p3); }
__device__ __forceinline__ double3 raw_a(const AdjA2& s) {
  const double4 r = s.raw();
  return make_double3(r.x, r.y, r.z);
}
// y = M x + v for a row-major 3x3 M
__device__ __forceinline__ double3 affine3(const double* M, double3 x, double3 v) {
  return make_double3(fma(M[0], x.x, fma(M[1], x.y, fma(M[2], x.z, v.x))),
                      fma(M[3], x.x, fma(M[4], x.y, fma(M[5], x.z, v.y))),
                      fma(M[6], x.x, fma(M[7], x.y, fma(M[8], x.z, v.z))));
}

// closure-entry raw state at a segment end u of the chunk (segment_entry's
// arithmetic with the chunk entry S in place of a checkpoint). pu/pm1/pm2:
// the stored causal values at u, u-1, u-2 (valid when u >= 1 / u >= 2).
template <bool TR>
__device__ __forceinline__ double3 end_raw(int u, double pu, double pm1, double pm2, double3 S,
                                           bool s1, bool s2, const Coef3& c, const Coef3& c1,
                                           const Coef3& c2) {
  if constexpr (!TR) {
    const double x1 = s1 ? (u >= 1 ? pm1 : S.x) : 0.0;
    const double x2 = s2 ? (u >= 2 ? pm2 : (u == 1 ? S.x : S.y)) : 0.0;
    return make_double3(pu, x1, x2);
  } else {
    double t1, t2, t3;
    if (u >= 2) {
      t1 = c1.a2 * pm1;
      t2 = c1.a3 * pm1;
      t3 = c2.a3 * pm2;
    } else if (u == 1) {
      t1 = c1.a2 * pm1;
      t2 = c1.a3 * pm1;
      t3 = S.z;
    } else {
      t1 = S.y;
      t2 = S.z;
      t3 = 0.0;
    }
    if (!s1) t1 = t2 = t3 = 0.0;
    if (!s2) t3 = 0.0;
    return make_double3(fma(c.a1, pu, t3 + t1), t2 + c.a2 * pu, c.a3 * pu);
  }
}
}  // namespace sp

struct XspArgs {
  int64_t nx, ny, planes, nlev, lev0, pitch, nh;
  int ppc, PB, RW, RC, CS;
  int64_t words;
  const uint64_t* bits;  // level-major packed bits of the class's representative level
  int ghosts;
  const Coef3* c3;
  const double* idc;  // rows `ipitch` apart
  int64_t ipitch;
  const double* clos;  // closure rows [nh][10] of this class / part
  const double* tab;   // [ny][nx][6]: Phi[3], Psi[3] (relative to the point's sub-chunk)
  const double* chk;   // [ny][CS*NW][CHKW] per sub-chunk
  const double* ccta;  // [ny][CS][CHKW]: Acta[9], Bcta[9] per CTA chunk
  const double* cl;    // [ny][CS*NW][MAXE][10] closure rows of each sub-chunk's ends
  const double* pre_scale;
  const double* post_scale;
};

// ------------------------------------------------------------ tables
// One thread per (row, CTA chunk): for each of its NW sub-chunks the
// homogeneous responses of the kernel's own recursions (zero input) to the
// three unit entry states, then the chunk's composed transfers.
template <bool TR>
__global__ void k_xsp_tables(XspArgs a, double* tab, double* chk, double* ccta, double* cl) {
  using A2 = typename std::conditional<TR, AdjA2, FwdA2>::type;
  using D2 = typename std::conditional<TR, AdjD2, FwdD2>::type;
  const int64_t nx = a.nx;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < a.ny * a.CS;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t iy = t / a.CS;
    const int c = static_cast<int>(t - iy * a.CS);
    const uint64_t* W = a.bits + iy * a.words;
    auto bit = [&](int64_t x) -> bool {
      return x >= 0 && x < nx && ((W[x >> 6] >> (x & 63)) & 1ull);
    };
    const Coef3* cr = a.c3 + iy * nx;
    double* tb = tab + iy * nx * 6;
    double Ac[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, Bc[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    for (int w = 0; w < sp::NW; ++w) {
      const int64_t g = t * sp::NW + w;
      const int64_t xs = int64_t(c) * a.RC + int64_t(w) * a.RW;
      const int Lw = static_cast<int>(xs >= nx ? 0 : (nx - xs < a.RW ? nx - xs : a.RW));
      double* ck = chk + g * sp::CHKW;
      double* cls = cl + g * sp::MAXE * 10;
      double A[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, B[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
      int phi_len = 0, psi_start = 0, nends = 0;
      if (Lw > 0) {
        // causal: Phi and A
        A2 s[3];
        for (int k = 0; k < 3; ++k) restore(s[k], k == 0, k == 1, k == 2);
        for (int u = 0; u < Lw; ++u) {
          const int64_t x = xs + u;
          const bool sea = bit(x);
          if (sea && !bit(x - 1))
            for (int k = 0; k < 3; ++k) s[k].reset();
          bool nz = false;
          for (int k = 0; k < 3; ++k) {
            const double o = s[k].step(cr[x], 0.0);
            tb[x * 6 + k] = sea ? o : 0.0;
            nz |= sea && o != 0.0;
          }
          if (nz) phi_len = u + 1;
        }
        const bool last_sea = bit(xs + Lw - 1);
        for (int k = 0; k < 3; ++k) {
          const double3 r = sp::raw_a(s[k]);
          A[0 * 3 + k] = last_sea ? r.x : 0.0;
          A[1 * 3 + k] = last_sea ? r.y : 0.0;
          A[2 * 3 + k] = last_sea ? r.z : 0.0;
        }
        // anti-causal: Psi, B and the closure rows met (descending order)
        D2 d[3];
        for (int k = 0; k < 3; ++k) sp::restore_d(d[k], k == 0, k == 1, k == 2);
        psi_start = Lw;
        for (int u = Lw - 1; u >= 0; --u) {
          const int64_t x = xs + u;
          const bool sea = bit(x);
          if (sea && !bit(x + 1)) {  // segment end: closure entry of a zero raw state
            for (int k = 0; k < 3; ++k) d[k].reset();
            if (x < nx - 1 && a.ghosts) {
              if (nends < sp::MAXE)
                for (int m = 0; m < 10; ++m) cls[nends * 10 + m] = a.clos[(iy * nx + x) * 10 + m];
              ++nends;
            }
          }
          bool nz = false;
          for (int k = 0; k < 3; ++k) {
            const double o = d[k].step(cr[x], cr[x].b * 0.0);
            tb[x * 6 + 3 + k] = sea ? o : 0.0;
            nz |= sea && o != 0.0;
          }
          if (nz) psi_start = u;
        }
        const bool first_sea = bit(xs);
        for (int k = 0; k < 3; ++k) {
          const double3 r = sp::raw_d(d[k]);
          B[0 * 3 + k] = first_sea ? r.x : 0.0;
          B[1 * 3 + k] = first_sea ? r.y : 0.0;
          B[2 * 3 + k] = first_sea ? r.z : 0.0;
        }
      }
      for (int m = 0; m < 9; ++m) {
        ck[m] = A[m];
        ck[9 + m] = B[m];
      }
      ck[18] = phi_len;
      ck[19] = psi_start;
      ck[20] = nends;
      ck[21] = ck[22] = ck[23] = 0.0;
      // chunk transfers: Acta <- A Acta (sub-chunks in order), Bcta <- Bcta B
      double N[9];
      for (int r = 0; r < 3; ++r)
        for (int q = 0; q < 3; ++q)
          N[r * 3 + q] = A[r * 3 + 0] * Ac[0 * 3 + q] + A[r * 3 + 1] * Ac[1 * 3 + q] +
                         A[r * 3 + 2] * Ac[2 * 3 + q];
      for (int m = 0; m < 9; ++m) Ac[m] = N[m];
      for (int r = 0; r < 3; ++r)
        for (int q = 0; q < 3; ++q)
          N[r * 3 + q] = Bc[r * 3 + 0] * B[0 * 3 + q] + Bc[r * 3 + 1] * B[1 * 3 + q] +
                         Bc[r * 3 + 2] * B[2 * 3 + q];
      for (int m = 0; m < 9; ++m) Bc[m] = N[m];
    }
    double* cc = ccta + t * sp::CHKW;
    for (int m = 0; m < 9; ++m) {
      cc[m] = Ac[m];
      cc[9 + m] = Bc[m];
    }
    for (int m = 18; m < sp::CHKW; ++m) cc[m] = 0.0;
  }
}

// ------------------------------------------------------------ the sweep
// NW warps per CTA (lanes = up to 32 planes of one row; warp w owns the
// sub-chunk [w*RW, (w+1)*RW) of the CTA's chunk), two CTAs per SM. Carries
// are folded in two levels: warps inside the CTA through shared memory, CTAs
// of the cluster through distributed shared memory.
template <bool TR, bool IDC, bool PRE, bool POST>
__global__ void __launch_bounds__(32 * sp::NW, 2)
    k_xsp(XspArgs a, const __grid_constant__ CUtensorMap tm_in,
          const __grid_constant__ CUtensorMap tm_out) {
  using L = sp::Layout;
  using A2 = typename std::conditional<TR, AdjA2, FwdA2>::type;
  using D2 = typename std::conditional<TR, AdjD2, FwdD2>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const Coef3* cf = reinterpret_cast<const Coef3*>(smem + L::coef);
  const double* id = reinterpret_cast<const double*>(smem + L::idc);
  const double* tb = reinterpret_cast<const double*>(smem + L::tab);
  const double* ck = reinterpret_cast<const double*>(smem + L::chk);
  const double* cc = reinterpret_cast<const double*>(smem + L::ccta);
  const double* cls = reinterpret_cast<const double*>(smem + L::cl);
  double* xw = reinterpret_cast<double*>(smem + L::xw);
  double* xc = reinterpret_cast<double*>(smem + L::xc);
  uint64_t* mw = reinterpret_cast<uint64_t*>(smem + L::words);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::bars);  // [NSUB] field, [NSUB] tables

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = static_cast<int>(sp::cluster_rank());
  const int64_t cid = blockIdx.x / a.CS;
  const int64_t iy = cid / a.PB;
  const int pg = static_cast<int>(cid - iy * a.PB);
  const int64_t p0 = int64_t(pg) * a.ppc;
  const int npl = static_cast<int>(a.planes - p0 < a.ppc ? a.planes - p0 : a.ppc);
  const int64_t nx = a.nx;
  const int64_t X0 = int64_t(c) * a.RC;
  const int Lc = static_cast<int>(nx - X0 < a.RC ? nx - X0 : a.RC);
  const int nsub = (Lc + 15) / 16;
  const int64_t t_chunk = iy * a.CS + c;
  const int64_t w0 = (X0 >> 6) - 1;  // mask word in slot 0

  if (threadIdx.x == 0) {
    for (int t = 0; t <= sp::NSUB; ++t) mbar_init(&bars[t], 1);
    mbar_fence_init();
    const uint64_t pol_stream = l2_evict_first();
    tma_prefetch_desc(&tm_in);
    const uint32_t cb = uint32_t(Lc) * 32, ib = uint32_t((Lc + 1) & ~1) * 8, tbb = uint32_t(Lc) * 48;
    const uint32_t kb = sp::NW * sp::CHKW * 8, kcb = uint32_t(a.CS) * sp::CHKW * 8;
    const uint32_t lb = sp::NW * sp::MAXE * 80;
    mbar_arrive_expect_tx(&bars[sp::NSUB], cb + (IDC ? ib : 0) + tbb + kb + kcb + lb);
    bulk_g2s(smem + L::coef, a.c3 + iy * nx + X0, cb, &bars[sp::NSUB]);
    if constexpr (IDC) bulk_g2s(smem + L::idc, a.idc + iy * a.ipitch + X0, ib, &bars[sp::NSUB]);
    bulk_g2s(smem + L::tab, a.tab + (iy * nx + X0) * 6, tbb, &bars[sp::NSUB]);
    bulk_g2s(smem + L::chk, a.chk + t_chunk * sp::NW * sp::CHKW, kb, &bars[sp::NSUB]);
    bulk_g2s(smem + L::ccta, a.ccta + iy * a.CS * sp::CHKW, kcb, &bars[sp::NSUB]);
    bulk_g2s(smem + L::cl, a.cl + t_chunk * sp::NW * sp::MAXE * 10, lb, &bars[sp::NSUB]);
    for (int t = 0; t < nsub; ++t) {
      mbar_arrive_expect_tx(&bars[t], uint32_t(a.ppc) * 128);
      tma_load_3d(smem + t * sp::SUBB, &tm_in, static_cast<int>(X0 + 16 * t),
                  static_cast<int>(p0), static_cast<int>(iy), &bars[t], pol_stream);
    }
  }
  if (warp == 0 && lane < 16) {  // the chunk's mask words (one mask class: warp-uniform)
    const int64_t wi = w0 + lane;
    mw[lane] = (wi >= 0 && wi < a.words) ? ldw(a.bits + iy * a.words, wi) : 0ull;
  }
  __syncthreads();

  const int pl = lane;
  const int64_t p = p0 + (pl < npl ? pl : 0);
  const int64_t lev = a.lev0 + p % a.nlev;
  const int sw = pl & 7;
  const int us = warp * a.RW;  // this warp's sub-chunk [us, us + Lw) of the chunk
  const int Lw = Lc - us <= 0 ? 0 : (Lc - us < a.RW ? Lc - us : a.RW);
  const double* ckw = ck + warp * sp::CHKW;
  auto bits16 = [&](int u) -> uint32_t {  // bits of chunk points u..u+15 (0 past the line)
    const int64_t x = X0 + u;
    const int64_t i = (x >> 6) - w0;
    const int s = static_cast<int>(x & 63);
    uint64_t v = mw[i] >> s;
    if (s > 48) v |= mw[i + 1] << (64 - s);
    return static_cast<uint32_t>(v & 0xffffull);
  };
  auto bit = [&](int u) -> uint32_t {
    const int64_t x = X0 + u;
    return (x >= 0 && x < nx) ? static_cast<uint32_t>((mw[(x >> 6) - w0] >> (x & 63)) & 1ull) : 0u;
  };
  auto pair_at = [&](int u) -> double2* {  // this lane's points u, u+1 (u even)
    return reinterpret_cast<double2*>(smem + (u >> 4) * sp::SUBB + pl * 128 +
                                      ((((u & 15) >> 1) ^ sw) << 4));
  };
  auto elem = [&](int u) -> double* {
    return reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(pair_at(u & ~1)) +
                                     (u & 1) * 8);
  };
  const double* PREp = PRE ? a.pre_scale + lev * a.nh + iy * nx + X0 : nullptr;
  const double* POSTp = POST ? a.post_scale + lev * a.nh + iy * nx + X0 : nullptr;

  mbar_wait(&bars[sp::NSUB], 0);

  // ---- F0: causal recursion over the sub-chunk, zero entry, p in place
  A2 sa;
  {
    uint32_t carry = bit(us - 1);
    auto step_pair = [&](int u, uint32_t rs0, uint32_t rs1, bool two) {
      double2* cp = pair_at(u);
      const double2 v = *cp;
      double w0v = v.x, w1v = v.y;
      if constexpr (TR && PRE) {
        w0v *= __ldg(PREp + u);
        if (two) w1v *= __ldg(PREp + u + 1);
      }
      if constexpr (TR && IDC) {
        w0v *= id[u];
        w1v *= id[u + 1];
      }
      reset_if(sa, rs0);
      const double r0 = sa.step(cf[u], w0v);
      double r1 = v.y;
      if (two) {
        reset_if(sa, rs1);
        r1 = sa.step(cf[u + 1], w1v);
      }
      *cp = make_double2(r0, r1);
    };
    int u0 = us;
    for (; u0 + 16 <= us + Lw; u0 += 16) {
      const uint32_t sb = bits16(u0);
      const uint32_t starts = sb & ~((sb << 1) | carry);
      carry = (sb >> 15) & 1u;
      mbar_wait(&bars[u0 >> 4], 0);
      mbar_wait(&bars[(u0 + 15) >> 4], 0);
      if (starts == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) step_pair(u0 + 2 * k, 0u, 0u, true);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          step_pair(u0 + 2 * k, (starts >> (2 * k)) & 1u, (starts >> (2 * k + 1)) & 1u, true);
      }
    }
    for (; u0 < us + Lw; u0 += 2) {  // tail (pairs; a last single point when Lw is odd)
      const bool two = u0 + 1 < us + Lw;
      const uint32_t b0 = bit(u0), b1 = bit(u0 + 1);
      mbar_wait(&bars[u0 >> 4], 0);
      step_pair(u0, b0 & ~carry, b1 & ~b0, two);
      carry = two ? b1 : b0;
    }
  }
  {
    const double3 b = sp::raw_a(sa);
    const bool ls = Lw > 0 && bit(us + Lw - 1);
    double* o = xw + (warp * 32 + pl) * 6;
    o[0] = ls ? b.x : 0.0;
    o[1] = ls ? b.y : 0.0;
    o[2] = ls ? b.z : 0.0;
  }
  __syncthreads();
  if (warp == sp::NW - 1) {  // the chunk's exit from a zero entry, for the CTAs on the right
    double3 bc = make_double3(0.0, 0.0, 0.0);
#pragma unroll
    for (int w = 0; w < sp::NW; ++w) {
      const double* bw = xw + (w * 32 + pl) * 6;
      bc = sp::affine3(ck + w * sp::CHKW, bc, make_double3(bw[0], bw[1], bw[2]));
    }
    xc[pl * 6 + 0] = bc.x;
    xc[pl * 6 + 1] = bc.y;
    xc[pl * 6 + 2] = bc.z;
  }
  sp::cluster_arrive();
  sp::cluster_wait();

  // ---- S for this warp: CTAs on the left (DSMEM), then warps on the left
  double3 S = make_double3(0.0, 0.0, 0.0);
  {
    double pb[sp::MAXCS][3];  // all peers' exits first (independent loads), then the fold
#pragma unroll
    for (int j = 0; j < sp::MAXCS; ++j)
#pragma unroll
      for (int k = 0; k < 3; ++k) pb[j][k] = j < c ? sp::ld_peer(xc + pl * 6 + k, j) : 0.0;
#pragma unroll
    for (int j = 0; j < sp::MAXCS; ++j)
      if (j < c) S = sp::affine3(cc + j * sp::CHKW, S, make_double3(pb[j][0], pb[j][1], pb[j][2]));
    for (int w = 0; w < warp; ++w) {
      const double* bw = xw + (w * 32 + pl) * 6;
      S = sp::affine3(ck + w * sp::CHKW, S, make_double3(bw[0], bw[1], bw[2]));
    }
  }
  // p += Phi S over the sub-chunk's first segment
  {
    const int phi_len = static_cast<int>(ckw[18]);
    for (int u = us; u < us + phi_len; ++u) {
      double* q = elem(u);
      const double* f = tb + u * 6;
      *q = fma(f[0], S.x, fma(f[1], S.y, fma(f[2], S.z, *q)));
    }
  }
  __syncwarp();

  // ---- B0: anti-causal recursion down the sub-chunk, zero entry state
  D2 sd;
  {
    int ei = 0;
    const double* clw = cls + warp * sp::MAXE * 10;
    // one point; `end` = segment end here, sb/sbit helpers for s1/s2
    auto point = [&](int u, double pu, bool end) -> double {
      const Coef3 cu = cf[u];
      if (end) {
        const int64_t x = X0 + u;
        if (x < nx - 1 && a.ghosts) {
          const int ur = u - us;
          const bool s1 = bit(u - 1) != 0u;
          const bool s2 = s1 && bit(u - 2) != 0u;
          const double pm1 = ur >= 1 ? *elem(u - 1) : 0.0;
          const double pm2 = ur >= 2 ? *elem(u - 2) : 0.0;
          const Coef3 c1 = cf[ur >= 1 ? u - 1 : u], c2 = cf[ur >= 2 ? u - 2 : u];
          const double3 r = sp::end_raw<TR>(ur, pu, pm1, pm2, S, s1, s2, cu, c1, c2);
          const double* Mp = ei < sp::MAXE ? clw + ei * 10 : a.clos + (iy * nx + x) * 10;
          Closure M;
#pragma unroll
          for (int m = 0; m < 9; ++m) M.m[m] = Mp[m];
          ++ei;
          enter(sd, apply_m(M, r.x, r.y, r.z), cu);
        } else {
          sd.reset();
        }
      }
      return sd.step(cu, cu.b * pu);
    };
    int u1 = us + Lw;  // exclusive end of the unprocessed range
    // tail first (descending): points beyond the last full group of 16
    const int nfull = Lw / 16;
    const int ufull = us + nfull * 16;
    while (u1 > ufull) {
      const int u = u1 - 1;
      const bool end = bit(u) && !bit(u + 1);
      double* q = elem(u);
      *q = point(u, *q, end);
      u1 = u;
    }
    for (int u0 = ufull - 16; u0 >= us; u0 -= 16) {
      const uint32_t sb = bits16(u0);
      const uint32_t after = bit(u0 + 16);
      const uint32_t ends = sb & ~((sb >> 1) | (after << 15));
      if (ends == 0) {
#pragma unroll
        for (int k = 7; k >= 0; --k) {
          double2* cp = pair_at(u0 + 2 * k);
          const double2 v = *cp;
          const Coef3 c1 = cf[u0 + 2 * k + 1], c0 = cf[u0 + 2 * k];
          const double o1 = sd.step(c1, c1.b * v.y);
          const double o0 = sd.step(c0, c0.b * v.x);
          *cp = make_double2(o0, o1);
        }
      } else {
#pragma unroll 1
        for (int k = 7; k >= 0; --k) {
          double2* cp = pair_at(u0 + 2 * k);
          const double2 v = *cp;
          const double o1 = point(u0 + 2 * k + 1, v.y, (ends >> (2 * k + 1)) & 1u);
          const double o0 = point(u0 + 2 * k, v.x, (ends >> (2 * k)) & 1u);
          *cp = make_double2(o0, o1);
        }
      }
    }
  }
  {
    const double3 e = sp::raw_d(sd);
    const bool fs = Lw > 0 && bit(us);
    double* o = xw + (warp * 32 + pl) * 6;
    o[3] = fs ? e.x : 0.0;
    o[4] = fs ? e.y : 0.0;
    o[5] = fs ? e.z : 0.0;
  }
  __syncthreads();
  if (warp == 0) {  // the chunk's exit from a zero right entry, for the CTAs on the left
    double3 ec = make_double3(0.0, 0.0, 0.0);
#pragma unroll
    for (int w = sp::NW - 1; w >= 0; --w) {
      const double* ew = xw + (w * 32 + pl) * 6 + 3;
      ec = sp::affine3(ck + w * sp::CHKW + 9, ec, make_double3(ew[0], ew[1], ew[2]));
    }
    xc[pl * 6 + 3] = ec.x;
    xc[pl * 6 + 4] = ec.y;
    xc[pl * 6 + 5] = ec.z;
  }
  sp::cluster_arrive();
  sp::cluster_wait();

  // ---- T for this warp: CTAs on the right (DSMEM), then warps on the right
  double3 T = make_double3(0.0, 0.0, 0.0);
  {
    double pe[sp::MAXCS][3];
#pragma unroll
    for (int j = 0; j < sp::MAXCS; ++j)
#pragma unroll
      for (int k = 0; k < 3; ++k)
        pe[j][k] = (j > c && j < a.CS) ? sp::ld_peer(xc + pl * 6 + 3 + k, j) : 0.0;
#pragma unroll
    for (int j = sp::MAXCS - 1; j >= 0; --j)
      if (j > c && j < a.CS)
        T = sp::affine3(cc + j * sp::CHKW + 9, T, make_double3(pe[j][0], pe[j][1], pe[j][2]));
    for (int w = sp::NW - 1; w > warp; --w) {
      const double* ew = xw + (w * 32 + pl) * 6 + 3;
      T = sp::affine3(ck + w * sp::CHKW + 9, T, make_double3(ew[0], ew[1], ew[2]));
    }
  }
  sp::cluster_arrive();  // done with the peers' shared memory (waited before exit)

  // ---- o += Psi T over the last segment; unit-DC, variance, land = 0
  {
    const int psi = us + static_cast<int>(ckw[19]);
    auto fin = [&](int u, double o, uint32_t sea) -> double {
      if (u >= psi) {
        const double* f = tb + u * 6 + 3;
        o = fma(f[0], T.x, fma(f[1], T.y, fma(f[2], T.z, o)));
      }
      if constexpr (!TR && IDC) o *= id[u];
      if constexpr (POST) o *= __ldg(POSTp + u);
      return sea ? o : 0.0;
    };
    int u0 = us;
    for (; u0 + 16 <= us + Lw; u0 += 16) {
      const uint32_t sb = bits16(u0);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        double2* cp = pair_at(u0 + 2 * k);
        const double2 v = *cp;
        *cp = make_double2(fin(u0 + 2 * k, v.x, (sb >> (2 * k)) & 1u),
                           fin(u0 + 2 * k + 1, v.y, (sb >> (2 * k + 1)) & 1u));
      }
    }
    for (; u0 < us + Lw; ++u0) {
      double* q = elem(u0);
      *q = fin(u0, *q, bit(u0));
    }
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t pol = l2_evict_first();
    for (int t = 0; t < nsub; ++t)
      tma_store_3d(&tm_out, static_cast<int>(X0 + 16 * t), static_cast<int>(p0),
                   static_cast<int>(iy), smem + t * sp::SUBB, pol);
    bulk_commit();
    bulk_wait_read_all();
  }
  __syncthreads();
  sp::cluster_wait();
}

// ------------------------------------------------------------ launcher
// Chunking of a row of nx points: CS CTAs of RC = NW*RW points (RW a
// multiple of 4, so chunk starts are 16-point aligned). False when the
// single-pass path does not apply (rows longer than MAXCS*RCMAX).
inline bool xsp_chunking(int64_t nx, int& RW, int& RC, int& CS) {
  if (nx < 16) return false;
  const int64_t cs = (nx + sp::RCMAX - 1) / sp::RCMAX;
  if (cs > sp::MAXCS) return false;
  const int64_t rw = ((nx + cs * sp::NW - 1) / (cs * sp::NW) + 3) / 4 * 4;
  RW = static_cast<int>(rw);
  RC = static_cast<int>(rw * sp::NW);
  CS = static_cast<int>((nx + RC - 1) / RC);
  return RC <= sp::RCMAX && CS <= sp::MAXCS;
}

template <bool TR, bool IDC, bool PRE, bool POST>
bool launch_xsp_k(const double* in, double* out, const XspArgs& a, cudaStream_t st) {
  auto kern = k_xsp<TR, IDC, PRE, POST>;
  const size_t smem = sp::Layout::bytes + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  const uint64_t fd[3] = {uint64_t(a.nx), uint64_t(a.planes), uint64_t(a.ny)};
  const uint64_t fs[2] = {uint64_t(a.pitch * a.ny) * 8, uint64_t(a.pitch) * 8};
  const uint32_t fb[3] = {16, uint32_t(a.ppc), 1};
  const CUtensorMap tin = make_tmap(in, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, fd, fs, fb,
                                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  const CUtensorMap tout = make_tmap(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, fd, fs, fb,
                                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(int64_t(a.CS) * a.ny * a.PB));
  cfg.blockDim = dim3(32 * sp::NW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = static_cast<unsigned>(a.CS);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, tin, tout) == cudaSuccess;
}

inline bool launch_xsp(const double* in, double* out, const XspArgs& a, bool tr, bool idc,
                       bool pre, bool post, cudaStream_t st) {
#define RGFB_XSP(T_, I_, P_, Q_) return launch_xsp_k<T_, I_, P_, Q_>(in, out, a, st);
  if (tr) {
    if (idc) {
      if (pre) { RGFB_XSP(true, true, true, false) } else { RGFB_XSP(true, true, false, false) }
    } else {
      if (pre) { RGFB_XSP(true, false, true, false) } else { RGFB_XSP(true, false, false, false) }
    }
  } else {
    if (idc) {
      if (post) { RGFB_XSP(false, true, false, true) } else { RGFB_XSP(false, true, false, false) }
    } else {
      if (post) { RGFB_XSP(false, false, false, true) } else { RGFB_XSP(false, false, false, false) }
    }
  }
#undef RGFB_XSP
}

}  // namespace rgfb
