// Construction-time kernels of the streaming 3rd-RF path: the right-ghost
// closure tables and the bit-packed per-level masks (sweep_stream.cuh).
#pragma once
#include "common.cuh"

namespace rgfb {

// ------------------------------------------------------------ closures
// Per point p (horizontal), ghost width G, coefficients c = c3[p]:
//  M (forward op): state (p_j, p_{j-1}, p_{j-2}) -> (q_{j+1}, q_{j+2}, q_{j+3})
//    by G causal ghost steps with zero input, then the anti-causal pass from
//    the far end with zero state (the reference's startup rows).
//  Mt (adjoint): pending contributions (P1, P2, P3) into u_{j+1..j+3} ->
//    (u'_{j+1}, u'_{j+2}, u'_{j+3}) by the causal-transpose gather over the
//    ghosts, beta scaling, and the anti-causal-transpose gather back.
// Ghost recursions use the reference's unfused left-to-right order.
// Output layout: `out` = forward part [nh][10], `out + nh*10` = adjoint part
// [nh][10] (9 matrix entries, one pad: 80 B rows, TMA-loadable).
__global__ void k_closures(const Coef3* c3, int64_t nh, int G, double* out, double* scratch,
                           int64_t slab) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double* g = scratch + tid * slab;
  for (int64_t p = tid; p < nh; p += (int64_t)gridDim.x * blockDim.x) {
    const Coef3 c = c3[p];
    double* o = out + p * 10;
    double* oa = out + nh * 10 + p * 10;
    o[9] = 0.0;
    oa[9] = 0.0;
    for (int m = 0; m < 3; ++m) {
      // forward closure, basis state e_m over (p_j, p_{j-1}, p_{j-2})
      double pm1 = m == 0, pm2 = m == 1, pm3 = m == 2;
      for (int k = 0; k < G; ++k) {
        const double t = dadd(dadd(dmul(c.a1, pm1), dmul(c.a2, pm2)), dmul(c.a3, pm3));
        pm3 = pm2;
        pm2 = pm1;
        pm1 = t;
        g[k] = t;
      }
      double q1 = 0.0, q2 = 0.0, q3 = 0.0;
      double r[3] = {0.0, 0.0, 0.0};
      for (int k = G - 1; k >= 0; --k) {
        const double t = dadd(dadd(dadd(dmul(c.b, g[k]), dmul(c.a1, q1)), dmul(c.a2, q2)),
                              dmul(c.a3, q3));
        q3 = q2;
        q2 = q1;
        q1 = t;
        if (k < 3) r[k] = t;
      }
      o[0 + m] = r[0];
      o[3 + m] = r[1];
      o[6 + m] = r[2];

      // adjoint closure, basis pending contributions e_m over (P1, P2, P3)
      const double P1 = m == 0, P2 = m == 1, P3 = m == 2;
      double u1 = 0.0, u2 = 0.0, u3 = 0.0;  // u_{k-1}, u_{k-2}, u_{k-3} (ghosts)
      for (int k = 0; k < G; ++k) {
        double u;
        if (k == 0)
          u = P1;
        else if (k == 1)
          u = dadd(P2, dmul(c.a1, u1));
        else if (k == 2)
          u = dadd(dadd(P3, dmul(c.a2, u2)), dmul(c.a1, u1));
        else
          u = dadd(dadd(dmul(c.a3, u3), dmul(c.a2, u2)), dmul(c.a1, u1));
        u3 = u2;
        u2 = u1;
        u1 = u;
        g[k] = dmul(c.b, u);  // v_{j+1+k}
      }
      double w1 = 0.0, w2 = 0.0, w3 = 0.0;  // u'_{k+1}, u'_{k+2}, u'_{k+3}
      double s[3] = {0.0, 0.0, 0.0};
      for (int k = G - 1; k >= 0; --k) {
        const double u = dadd(dadd(dadd(g[k], dmul(c.a3, w3)), dmul(c.a2, w2)), dmul(c.a1, w1));
        w3 = w2;
        w2 = w1;
        w1 = u;
        if (k < 3) s[k] = u;
      }
      oa[0 + m] = s[0];
      oa[3 + m] = s[1];
      oa[6 + m] = s[2];
    }
  }
}

// Bit-packed masks per direction: dir 0 words[(lev*ny+iy)*W + ix/64],
// dir 1 words[(lev*nx+ix)*W + iy/64]; bit k = sea at line position k.
__global__ void k_pack_bits(const uint8_t* mask, int dir, int64_t nx, int64_t ny, int64_t nlev,
                            int64_t words, uint64_t* bits) {
  const int64_t nlines = dir == 0 ? ny : nx;
  const int64_t n = dir == 0 ? nx : ny;
  const int64_t total = nlev * nlines * words;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t wi = t % words;
    const int64_t ln = t / words;  // lev*nlines + line
    const int64_t lev = ln / nlines, line = ln - lev * nlines;
    uint64_t v = 0;
    for (int b = 0; b < 64; ++b) {
      const int64_t k = wi * 64 + b;
      if (k >= n) break;
      const int64_t idx = dir == 0 ? (lev * ny + line) * nx + k : (lev * ny + k) * nx + line;
      if (mask[idx]) v |= (1ull << b);
    }
    bits[t] = v;
  }
}

}  // namespace rgfb
