// Chunked sweep for single-level operators (the reference's own 2-D operator:
// the acceptance case, the CG solver).
//
// With one plane the checkpointed kernels have one warp per 32-column tile
// walking the whole line, ~84 cycles per row of issue-bound latency
// (DESIGN §3.9). Here a CTA owns a 32-column tile and its NW warps own NW
// chunks of the lines (rows [w R, (w+1) R)); the chunks run their
// recursions from zero entry states at the same time and exchange 3-value
// carries through shared memory, exactly as the cluster kernel of round 2
// did across CTAs, but inside one CTA:
//   F0  causal recursion over the chunk from a zero state (resets at segment
//       starts), p written to an fp64 scratch plane; exit b_w -> smem;
//   S_w = fold over w' < w of  S <- A_w' S + b_w'   (A: the chunk's
//       homogeneous causal transfer, precomputed);
//   p += Phi S_w over the chunk's first segment (Phi: homogeneous response);
//   B0  anti-causal recursion down the chunk from a zero state, closure entries
//       at segment ends (covariance.cpp:271-349 with the right ghosts
//       collapsed, closures.cuh), o written over p; exit e_w -> smem;
//   T_w = fold over w' > w of  T <- B_w' T + e_w';
//   o += Psi T_w over the chunk's last segment; unit-DC / variance, land = 0.
// The data of a single level is L2-resident, so the extra scratch passes cost
// L2 bandwidth only. Lanes are columns: every load and store is a coalesced
// 32-column row. The tables (A, B, Phi, Psi per level, chunk and column)
// come from k_yfew_tables, which runs the kernel's own step arithmetic on unit
// entry states. Results match the checkpointed kernels to rounding
// (reassociated chunk entries), not bit for bit.
#pragma once
#include "sweep_ckpt.cuh"

namespace rgfb {

namespace few {
constexpr int NW = 16;   // chunks (warps) per column tile
constexpr int CHKW = 20; // per (level, chunk, column): A[9], B[9], phi_len, psi_start

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
// closure-entry raw state at a segment end u rows into the chunk (the
// checkpointed kernels' segment_entry with the chunk entry S as checkpoint)
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
__device__ __forceinline__ double3 affine3(const double* M, int64_t ms, double3 x, double3 v) {
  return make_double3(fma(M[0], x.x, fma(M[ms], x.y, fma(M[2 * ms], x.z, v.x))),
                      fma(M[3 * ms], x.x, fma(M[4 * ms], x.y, fma(M[5 * ms], x.z, v.y))),
                      fma(M[6 * ms], x.x, fma(M[7 * ms], x.y, fma(M[8 * ms], x.z, v.z))));
}
}  // namespace few

// Inputs of a few-plane sweep in the frame where lines are columns (the y
// frame, or the transposed x frame): nx columns, ny rows.
struct FewArgs {
  int64_t nx, ny, pitch, nh;
  int64_t planes, nlev, lev0;
  int R;                    // rows per chunk
  int CS;                   // CTAs per column tile (a thread-block cluster; NW chunks each)
  int words;                // mask words per column
  const uint64_t* bits;     // [lev][column][word], bit = row
  const Coef3* c3;          // [row][column]
  const double* c3s;        // [row][2][column][2]: (a1, a2), (a3, b)
  const double* idc;        // rows idc_pitch apart, or null
  int64_t idc_pitch;
  const double* clos;       // closures of dir 1 / part: + clos_off(cls, 1, part, nh, h)
  int part;
  const int* ghost;
  const int* cls;
  const double* tab;        // [lev][row][6][column]: Phi[3], Psi[3]
  const double* chk;        // [lev][chunk][CHKW][column], chunk = cta * NW + warp
  const double* chk_cta;    // [lev][cta][18][column]: the CTA's composed A, B
  const double* pre_scale;  // [lev][row][column] or null
  const double* post_scale;
};

// ------------------------------------------------------------ tables
// One thread per (level, column, chunk): homogeneous responses (zero input)
// of the kernel's own recursions to the three unit entry states.
template <bool TR>
__global__ void k_yfew_tables(FewArgs a, double* tab, double* chk) {
  using A2 = typename std::conditional<TR, AdjA2, FwdA2>::type;
  using D2 = typename std::conditional<TR, AdjD2, FwdD2>::type;
  const int64_t nx = a.nx, ny = a.ny;
  const int NC = a.CS * few::NW;  // chunks per line
  const int64_t total = a.nlev * nx * NC;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int w = static_cast<int>(t % NC);
    const int64_t ix = (t / NC) % nx;
    const int64_t lev = t / (int64_t(NC) * nx);
    const int64_t r0 = int64_t(w) * a.R;
    const int L = static_cast<int>(r0 >= ny ? 0 : (ny - r0 < a.R ? ny - r0 : a.R));
    const uint64_t* W = a.bits + (lev * nx + ix) * a.words;
    auto bit = [&](int64_t r) -> bool {
      return r >= 0 && r < ny && ((W[r >> 6] >> (r & 63)) & 1ull);
    };
    auto cf = [&](int64_t r) -> Coef3 { return a.c3[r * nx + ix]; };
    double* tb = tab + lev * ny * 6 * nx + ix;  // [row][6][column]
    double* ck = chk + (lev * NC + w) * few::CHKW * nx + ix;
    double A[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, B[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    int phi_len = 0, psi_start = 0;
    if (L > 0) {
      A2 s[3];
      for (int k = 0; k < 3; ++k) restore(s[k], k == 0, k == 1, k == 2);
      for (int u = 0; u < L; ++u) {
        const int64_t r = r0 + u;
        const bool sea = bit(r);
        if (sea && !bit(r - 1))
          for (int k = 0; k < 3; ++k) s[k].reset();
        bool nz = false;
        const Coef3 c = cf(r);
        for (int k = 0; k < 3; ++k) {
          const double o = s[k].step(c, 0.0);
          tb[(r * 6 + k) * nx] = sea ? o : 0.0;
          nz |= sea && o != 0.0;
        }
        if (nz) phi_len = u + 1;
      }
      const bool ls = bit(r0 + L - 1);
      for (int k = 0; k < 3; ++k) {
        const double3 v = few::raw_a(s[k]);
        A[0 * 3 + k] = ls ? v.x : 0.0;
        A[1 * 3 + k] = ls ? v.y : 0.0;
        A[2 * 3 + k] = ls ? v.z : 0.0;
      }
      D2 d[3];
      for (int k = 0; k < 3; ++k) few::restore_d(d[k], k == 0, k == 1, k == 2);
      psi_start = L;
      for (int u = L - 1; u >= 0; --u) {
        const int64_t r = r0 + u;
        const bool sea = bit(r);
        if (sea && !bit(r + 1))  // segment end: entry from a zero raw state
          for (int k = 0; k < 3; ++k) d[k].reset();
        bool nz = false;
        const Coef3 c = cf(r);
        for (int k = 0; k < 3; ++k) {
          const double o = d[k].step(c, c.b * 0.0);
          tb[(r * 6 + 3 + k) * nx] = sea ? o : 0.0;
          nz |= sea && o != 0.0;
        }
        if (nz) psi_start = u;
      }
      const bool fs = bit(r0);
      for (int k = 0; k < 3; ++k) {
        const double3 v = few::raw_d(d[k]);
        B[0 * 3 + k] = fs ? v.x : 0.0;
        B[1 * 3 + k] = fs ? v.y : 0.0;
        B[2 * 3 + k] = fs ? v.z : 0.0;
      }
    }
    for (int m = 0; m < 9; ++m) {
      ck[m * nx] = A[m];
      ck[(9 + m) * nx] = B[m];
    }
    ck[18 * nx] = phi_len;
    ck[19 * nx] = psi_start;
  }
}

// The CTA-level transfers: Acta = A_{NW-1} ... A_0, Bcta = B_0 ... B_{NW-1}
// over the CTA's NW chunks (one thread per level, column and CTA).
__global__ void k_yfew_cta(FewArgs a, const double* chk, double* chk_cta) {
  const int64_t nx = a.nx;
  const int NC = a.CS * few::NW;
  const int64_t total = a.nlev * nx * a.CS;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(t % a.CS);
    const int64_t ix = (t / a.CS) % nx;
    const int64_t lev = t / (int64_t(a.CS) * nx);
    double Ac[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, Bc[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, N[9];
    for (int w = 0; w < few::NW; ++w) {
      const double* ck = chk + (lev * NC + c * few::NW + w) * few::CHKW * nx + ix;
      for (int r = 0; r < 3; ++r)
        for (int q = 0; q < 3; ++q)
          N[r * 3 + q] = ck[(r * 3 + 0) * nx] * Ac[0 * 3 + q] + ck[(r * 3 + 1) * nx] * Ac[1 * 3 + q] +
                         ck[(r * 3 + 2) * nx] * Ac[2 * 3 + q];
      for (int m = 0; m < 9; ++m) Ac[m] = N[m];
      for (int r = 0; r < 3; ++r)
        for (int q = 0; q < 3; ++q)
          N[r * 3 + q] = Bc[r * 3 + 0] * ck[(9 + 0 * 3 + q) * nx] +
                         Bc[r * 3 + 1] * ck[(9 + 1 * 3 + q) * nx] +
                         Bc[r * 3 + 2] * ck[(9 + 2 * 3 + q) * nx];
      for (int m = 0; m < 9; ++m) Bc[m] = N[m];
    }
    double* o = chk_cta + ((lev * a.CS + c) * 18) * nx + ix;
    for (int m = 0; m < 9; ++m) {
      o[m * nx] = Ac[m];
      o[(9 + m) * nx] = Bc[m];
    }
  }
}

__device__ __forceinline__ uint32_t few_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void few_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}
__device__ __forceinline__ void few_cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void few_cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ double few_ld_peer(const double* local, uint32_t rank) {
  uint32_t r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(r));
  return v;
}

// ------------------------------------------------------------ the sweep
template <typename T, bool TR, bool IDC, bool PRE, bool POST>
__global__ void __launch_bounds__(32 * few::NW, 1)
    k_yfew(const T* __restrict__ in, T* __restrict__ out, double* __restrict__ scr, FewArgs a) {
  using A2 = typename std::conditional<TR, AdjA2, FwdA2>::type;
  using D2 = typename std::conditional<TR, AdjD2, FwdD2>::type;
  __shared__ double xw[few::NW][32][6];  // chunk exits: b (causal), e (anti-causal)
  __shared__ double xc[32][6];           // this CTA's exits, read by the cluster's peers
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nx = a.nx, ny = a.ny;
  const int64_t ix0 = int64_t(blockIdx.x) * 32;
  const bool act = ix0 + lane < nx;
  const int64_t ix = act ? ix0 + lane : nx - 1;
  const int c = a.CS > 1 ? static_cast<int>(few_cluster_rank()) : 0;  // CTA in the cluster
  const int64_t p = blockIdx.y / a.CS;  // plane
  const int64_t lev = a.lev0 + p % a.nlev;
  const int NC = a.CS * few::NW;
  const int g = c * few::NW + warp;  // this warp's chunk of the line
  const int64_t r0 = int64_t(g) * a.R;
  const int L = static_cast<int>(r0 >= ny ? 0 : (ny - r0 < a.R ? ny - r0 : a.R));
  // restrict-qualified locals: the loads of later rows may be hoisted above
  // this row's scratch store (each step is otherwise an L2 round trip)
  const T* __restrict__ src = in + p * ny * a.pitch + ix;
  T* __restrict__ dst = out + p * ny * a.pitch + ix;
  double* __restrict__ sp = scr + p * ny * nx + ix;  // fp64 scratch: p, then o before scaling
  const double* __restrict__ c3s = a.c3s;
  const double* __restrict__ idc = a.idc;
  const uint64_t* __restrict__ W = a.bits + (lev * nx + ix) * a.words;
  auto bit = [&](int64_t r) -> uint32_t {
    return (r >= 0 && r < ny) ? static_cast<uint32_t>((__ldg(W + (r >> 6)) >> (r & 63)) & 1ull) : 0u;
  };
  auto bits8 = [&](int64_t r) -> uint32_t {  // mask bits of rows r..r+7 (0 outside the line)
    uint32_t v = 0;
    if (r >= 0) {
      const int64_t i = r >> 6;
      const int sh = static_cast<int>(r & 63);
      uint64_t w = __ldg(W + i) >> sh;
      if (sh > 56 && (i + 1) * 64 < ny) w |= __ldg(W + i + 1) << (64 - sh);
      v = static_cast<uint32_t>(w & 0xffull);
    }
    return v;
  };
  auto coef = [&](int64_t r) -> Coef3 {
    const double2 lo = __ldg(reinterpret_cast<const double2*>(c3s + (r * 2 * nx + ix) * 2));
    const double2 hi = __ldg(reinterpret_cast<const double2*>(c3s + (r * 2 * nx + ix) * 2 + 2 * nx));
    return Coef3{lo.x, lo.y, hi.x, hi.y};
  };
  const double* ckl = a.chk + lev * NC * few::CHKW * nx + ix;       // + (chunk*CHKW + m)*nx
  const double* ccl = a.chk_cta + lev * a.CS * 18 * nx + ix;        // + (cta*18 + m)*nx
  const double* tbl = a.tab + lev * ny * 6 * nx + ix;               // + (r*6 + k)*nx
  const double* PREp = PRE ? a.pre_scale + lev * a.nh + ix : nullptr;
  const double* POSTp = POST ? a.post_scale + lev * a.nh + ix : nullptr;

  // ---- F0: causal recursion from a zero state, p -> scratch. Rows go in
  // groups of G whose loads are all issued before the group's recursion, so a
  // group pays one L2 round trip instead of one per row.
  constexpr int G = 4;
  A2 sa;
  {
    uint32_t prev = bit(r0 - 1);
    for (int u0 = 0; u0 < L; u0 += G) {
      const int64_t rb = r0 + u0;
      const uint32_t sb = bits8(rb);
      double wv[G];
      Coef3 cv[G];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int64_t r = u0 + j < L ? rb + j : rb;  // clamped: tail rows unused
        wv[j] = static_cast<double>(__ldg(src + r * a.pitch));
        if constexpr (TR && PRE) wv[j] *= __ldg(PREp + r * nx);
        if constexpr (TR && IDC) wv[j] *= __ldg(idc + r * a.idc_pitch + ix);
        cv[j] = coef(r);
      }
#pragma unroll
      for (int j = 0; j < G; ++j) {
        if (u0 + j < L) {
          const uint32_t sea = (sb >> j) & 1u;
          reset_if(sa, sea & ~prev);
          sp[(rb + j) * nx] = sa.step(cv[j], wv[j]);
          prev = sea;
        }
      }
    }
  }
  {
    const double3 b = few::raw_a(sa);
    const bool ls = L > 0 && bit(r0 + L - 1);
    xw[warp][lane][0] = ls ? b.x : 0.0;
    xw[warp][lane][1] = ls ? b.y : 0.0;
    xw[warp][lane][2] = ls ? b.z : 0.0;
  }
  __syncthreads();
  if (a.CS > 1) {  // the CTA's exit from a zero entry, for the CTAs below
    if (warp == few::NW - 1) {
      double3 bc = make_double3(0.0, 0.0, 0.0);
      for (int w = 0; w < few::NW; ++w)
        bc = few::affine3(ckl + int64_t(c * few::NW + w) * few::CHKW * nx, nx, bc,
                          make_double3(xw[w][lane][0], xw[w][lane][1], xw[w][lane][2]));
      xc[lane][0] = bc.x;
      xc[lane][1] = bc.y;
      xc[lane][2] = bc.z;
    }
    few_cluster_sync();
  }
  double3 S = make_double3(0.0, 0.0, 0.0);
  for (int j = 0; j < c; ++j)  // CTAs above (DSMEM)
    S = few::affine3(ccl + int64_t(j) * 18 * nx, nx, S,
                     make_double3(few_ld_peer(&xc[lane][0], j), few_ld_peer(&xc[lane][1], j),
                                  few_ld_peer(&xc[lane][2], j)));
  for (int w = 0; w < warp; ++w)
    S = few::affine3(ckl + int64_t(c * few::NW + w) * few::CHKW * nx, nx, S,
                     make_double3(xw[w][lane][0], xw[w][lane][1], xw[w][lane][2]));
  {  // p += Phi S over the chunk's first segment
    const int phi_len = static_cast<int>(ckl[(int64_t(g) * few::CHKW + 18) * nx]);
    for (int u = 0; u < phi_len; ++u) {
      const int64_t r = r0 + u;
      const double* f = tbl + r * 6 * nx;
      sp[r * nx] = fma(f[0], S.x, fma(f[nx], S.y, fma(f[2 * nx], S.z, sp[r * nx])));
    }
  }

  // ---- B0: anti-causal recursion down the chunk from a zero state (groups
  // of G rows, descending, loads first)
  D2 sd;
  {
    const bool ghosts = a.ghost[lev] > 0;
    const double* Mcol = a.clos + clos_off(a.cls[lev], 1, a.part, a.nh, ix);
    const int ng = (L + G - 1) / G;
    uint32_t after = bit(r0 + L);  // row below the chunk's last (in line order: after)
    for (int g = ng - 1; g >= 0; --g) {
      const int u0 = g * G;
      const int64_t rb = r0 + u0;
      const uint32_t sb = bits8(rb);
      const uint32_t bm1 = bit(rb - 1), bm2 = bit(rb - 2);
      double pv[G];
      Coef3 cv[G];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int64_t r = u0 + j < L ? rb + j : rb;
        pv[j] = sp[r * nx];
        cv[j] = coef(r);
      }
      // rows j of the group whose successor is land or past the chunk's data:
      // the successor of the group's last valid row is `after`
      const int nv = L - u0 < G ? L - u0 : G;
      const uint32_t succ = (sb >> 1) | (after << (nv - 1));
      const uint32_t ends = sb & ~succ & ((1u << nv) - 1u);
#pragma unroll
      for (int j = G - 1; j >= 0; --j) {
        if (j < nv) {
          const int u = u0 + j;
          const int64_t r = rb + j;
          if ((ends >> j) & 1u) {
            if (r < ny - 1 && ghosts) {
              const bool s1 = (j >= 1 ? ((sb >> (j >= 1 ? j - 1 : 0)) & 1u) : bm1) != 0u;
              const bool s2 = s1 && (j >= 2 ? ((sb >> (j >= 2 ? j - 2 : 0)) & 1u)
                                            : (j == 1 ? bm1 : bm2)) != 0u;
              const double pm1 = u >= 1 ? (j >= 1 ? pv[j >= 1 ? j - 1 : 0] : sp[(r - 1) * nx]) : 0.0;
              const double pm2 = u >= 2 ? (j >= 2 ? pv[j >= 2 ? j - 2 : 0] : sp[(r - 2) * nx]) : 0.0;
              const Coef3 c1 = j >= 1 ? cv[j >= 1 ? j - 1 : 0] : coef(u >= 1 ? r - 1 : r);
              const Coef3 c2 = j >= 2 ? cv[j >= 2 ? j - 2 : 0] : coef(u >= 2 ? r - 2 : r);
              const double3 raw = few::end_raw<TR>(u, pv[j], pm1, pm2, S, s1, s2, cv[j], c1, c2);
              const Closure M = load_closure(Mcol + r * nx * 10);
              enter(sd, apply_m(M, raw.x, raw.y, raw.z), cv[j]);
            } else {
              sd.reset();
            }
          }
          sp[r * nx] = sd.step(cv[j], cv[j].b * pv[j]);
        }
      }
      after = sb & 1u;
    }
  }
  {
    const double3 e = few::raw_d(sd);
    const bool fs = L > 0 && bit(r0);
    xw[warp][lane][3] = fs ? e.x : 0.0;
    xw[warp][lane][4] = fs ? e.y : 0.0;
    xw[warp][lane][5] = fs ? e.z : 0.0;
  }
  __syncthreads();
  if (a.CS > 1) {  // the CTA's exit from a zero right entry, for the CTAs above
    if (warp == 0) {
      double3 ec = make_double3(0.0, 0.0, 0.0);
      for (int w = few::NW - 1; w >= 0; --w)
        ec = few::affine3(ckl + (int64_t(c * few::NW + w) * few::CHKW + 9) * nx, nx, ec,
                          make_double3(xw[w][lane][3], xw[w][lane][4], xw[w][lane][5]));
      xc[lane][3] = ec.x;
      xc[lane][4] = ec.y;
      xc[lane][5] = ec.z;
    }
    few_cluster_sync();
  }
  double3 Tin = make_double3(0.0, 0.0, 0.0);
  for (int j = a.CS - 1; j > c; --j)  // CTAs below (DSMEM)
    Tin = few::affine3(ccl + (int64_t(j) * 18 + 9) * nx, nx, Tin,
                       make_double3(few_ld_peer(&xc[lane][3], j), few_ld_peer(&xc[lane][4], j),
                                    few_ld_peer(&xc[lane][5], j)));
  for (int w = few::NW - 1; w > warp; --w)
    Tin = few::affine3(ckl + (int64_t(c * few::NW + w) * few::CHKW + 9) * nx, nx, Tin,
                       make_double3(xw[w][lane][3], xw[w][lane][4], xw[w][lane][5]));
  if (a.CS > 1) few_cluster_arrive();  // done with the peers' shared memory

  // ---- o += Psi T over the last segment; unit-DC, variance, land = 0
  {
    const int psi = static_cast<int>(ckl[(int64_t(g) * few::CHKW + 19) * nx]);
    for (int u0 = 0; u0 < L; u0 += G) {
      const int64_t rb = r0 + u0;
      const uint32_t sb = bits8(rb);
      double ov[G], sc[G];
#pragma unroll
      for (int j = 0; j < G; ++j) {
        const int64_t r = u0 + j < L ? rb + j : rb;
        ov[j] = sp[r * nx];
        if (u0 + j >= psi) {
          const double* f = tbl + (r * 6 + 3) * nx;
          ov[j] = fma(f[0], Tin.x, fma(f[nx], Tin.y, fma(f[2 * nx], Tin.z, ov[j])));
        }
        sc[j] = 1.0;
        if constexpr (!TR && IDC) sc[j] = __ldg(idc + r * a.idc_pitch + ix);
        if constexpr (POST) sc[j] *= __ldg(POSTp + r * nx);
      }
#pragma unroll
      for (int j = 0; j < G; ++j)
        if (u0 + j < L && act)
          dst[(rb + j) * a.pitch] = static_cast<T>(((sb >> j) & 1u) ? ov[j] * sc[j] : 0.0);
    }
  }
  if (a.CS > 1) few_cluster_wait();  // no CTA leaves while a peer may read its exits
}

template <typename T, bool TR, bool IDC, bool PRE, bool POST>
void launch_yfew_k(const T* in, T* out, double* scr, const FewArgs& a, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>((a.nx + 31) / 32), static_cast<unsigned>(a.planes * a.CS));
  cfg.blockDim = dim3(32 * few::NW);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = static_cast<unsigned>(a.CS);
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_yfew<T, TR, IDC, PRE, POST>, in, out, scr, a);
  if (e != cudaSuccess)
    throw std::runtime_error(std::string("few-plane sweep launch: ") + cudaGetErrorString(e));
}

template <typename T>
void launch_yfew(const T* in, T* out, double* scr, const FewArgs& a, bool tr, bool idc, bool pre,
                 bool post, cudaStream_t st) {
#define RGFB_FEW(TR_, I_, P_, Q_) launch_yfew_k<T, TR_, I_, P_, Q_>(in, out, scr, a, st)
  if (tr) {
    if (idc) {
      if (pre) RGFB_FEW(true, true, true, false); else RGFB_FEW(true, true, false, false);
    } else {
      if (pre) RGFB_FEW(true, false, true, false); else RGFB_FEW(true, false, false, false);
    }
  } else {
    if (idc) {
      if (post) RGFB_FEW(false, true, false, true); else RGFB_FEW(false, true, false, false);
    } else {
      if (post) RGFB_FEW(false, false, false, true); else RGFB_FEW(false, false, false, false);
    }
  }
#undef RGFB_FEW
}

}  // namespace rgfb
