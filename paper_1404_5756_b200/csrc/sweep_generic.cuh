// Segment-serial sweep: one thread per (var, level, line), walking the line's
// sea-segment descriptors exactly as HorizontalCovarianceOp::sweep_line does
// (covariance.cpp:228-352), with the reference's unfused left-to-right
// arithmetic (__dmul_rn/__dadd_rn). It serves the paths the streaming
// kernels do not cover (1st-RF, whose K>=2 iterations make both ghost zones
// live) and is bit-identical to the reference for identical
// coefficients. The extended segment lives in a per-thread fp64 scratch
// slab (the reference's thread_local SweepScratch, covariance.cpp:21-34).
#pragma once
#include "common.cuh"

namespace rgfb {

struct SweepArgs {
  int dir;        // 0 = x lines (rows), 1 = y lines (columns)
  int transpose;  // apply_g*_transpose
  int order;      // 1 | 3
  int k;          // 1st-RF iterations
  int unit_dc;    // 3rd-RF unit-DC rescaling
  int64_t nx, ny, nlev, nvar;
  int64_t lev0;   // first global level of this launch (level-chunked host pipeline)
  const Coef3* c3;     // rf3 table (dir's), nx*ny
  const double2* c1;   // rf1 table {alpha, beta}
  const double* idc;   // inv_dc table
  const int64_t* seg_off;  // per (lev, line) prefix offsets
  const int2* segs;        // (start, len)
  const int* ghost;        // per level
  const double* pre_scale; // optional per-(lev,point) multiplier applied to the input (variance), or NULL
  const double* post_scale;// optional multiplier applied to the output
  double* scratch;
  int64_t slab;  // doubles per thread slab
};

// rf3.hpp:217-239 with coefficients through accessor C (covariance.cpp:313-314)
template <class C>
__device__ void g_rf3_forward(double* s, const C& c, int64_t m) {
  double pm1 = dmul(c.b(0), s[0]);
  s[0] = pm1;
  double t = dadd(dmul(c.b(1), s[1]), dmul(c.a1(1), pm1));
  s[1] = t;
  double pm2 = pm1;
  pm1 = t;
  t = dadd(dadd(dmul(c.b(2), s[2]), dmul(c.a1(2), pm1)), dmul(c.a2(2), pm2));
  s[2] = t;
  double pm3 = pm2;
  pm2 = pm1;
  pm1 = t;
  for (int64_t i = 3; i < m; ++i) {
    t = dadd(dadd(dadd(dmul(c.b(i), s[i]), dmul(c.a1(i), pm1)), dmul(c.a2(i), pm2)),
             dmul(c.a3(i), pm3));
    pm3 = pm2;
    pm2 = pm1;
    pm1 = t;
    s[i] = t;
  }
}

// rf3.hpp:241-262
template <class C>
__device__ void g_rf3_backward(double* s, const C& c, int64_t m) {
  double pm1 = dmul(c.b(m - 1), s[m - 1]);
  s[m - 1] = pm1;
  double t = dadd(dmul(c.b(m - 2), s[m - 2]), dmul(c.a1(m - 2), pm1));
  s[m - 2] = t;
  double pm2 = pm1;
  pm1 = t;
  t = dadd(dadd(dmul(c.b(m - 3), s[m - 3]), dmul(c.a1(m - 3), pm1)), dmul(c.a2(m - 3), pm2));
  s[m - 3] = t;
  double pm3 = pm2;
  pm2 = pm1;
  pm1 = t;
  for (int64_t i = m - 4; i >= 0; --i) {
    t = dadd(dadd(dadd(dmul(c.b(i), s[i]), dmul(c.a1(i), pm1)), dmul(c.a2(i), pm2)),
             dmul(c.a3(i), pm3));
    pm3 = pm2;
    pm2 = pm1;
    pm1 = t;
    s[i] = t;
  }
}

// rf3.hpp:264-274
template <class C>
__device__ void g_rf3_forward_transpose(double* w, const C& c, int64_t m) {
  for (int64_t i = m - 1; i >= 0; --i) {
    const double wi = w[i];
    if (i >= 1) w[i - 1] = dadd(w[i - 1], dmul(c.a1(i), wi));
    if (i >= 2) w[i - 2] = dadd(w[i - 2], dmul(c.a2(i), wi));
    if (i >= 3) w[i - 3] = dadd(w[i - 3], dmul(c.a3(i), wi));
    w[i] = dmul(c.b(i), wi);
  }
}

// rf3.hpp:276-286
template <class C>
__device__ void g_rf3_backward_transpose(double* w, const C& c, int64_t m) {
  for (int64_t i = 0; i < m; ++i) {
    const double wi = w[i];
    if (i + 1 < m) w[i + 1] = dadd(w[i + 1], dmul(c.a1(i), wi));
    if (i + 2 < m) w[i + 2] = dadd(w[i + 2], dmul(c.a2(i), wi));
    if (i + 3 < m) w[i + 3] = dadd(w[i + 3], dmul(c.a3(i), wi));
    w[i] = dmul(c.b(i), wi);
  }
}

// rf1.hpp:20-63
template <class C>
__device__ void g_rf1_forward(double* s, const C& c, int64_t m) {
  double prev = dmul(c.b(0), s[0]);
  s[0] = prev;
  for (int64_t i = 1; i < m; ++i) {
    prev = dadd(dmul(c.b(i), s[i]), dmul(c.a1(i), prev));
    s[i] = prev;
  }
}
template <class C>
__device__ void g_rf1_backward(double* s, const C& c, int64_t m) {
  double prev = dmul(c.b(m - 1), s[m - 1]);
  s[m - 1] = prev;
  for (int64_t i = m - 2; i >= 0; --i) {
    prev = dadd(dmul(c.b(i), s[i]), dmul(c.a1(i), prev));
    s[i] = prev;
  }
}
template <class C>
__device__ void g_rf1_forward_transpose(double* w, const C& c, int64_t m) {
  double prev = w[m - 1];
  w[m - 1] = dmul(c.b(m - 1), prev);
  for (int64_t i = m - 2; i >= 0; --i) {
    const double cur = dadd(w[i], dmul(c.a1(i + 1), prev));
    w[i] = dmul(c.b(i), cur);
    prev = cur;
  }
}
template <class C>
__device__ void g_rf1_backward_transpose(double* w, const C& c, int64_t m) {
  double prev = w[0];
  w[0] = dmul(c.b(0), prev);
  for (int64_t i = 1; i < m; ++i) {
    const double cur = dadd(w[i], dmul(c.a1(i - 1), prev));
    w[i] = dmul(c.b(i), cur);
    prev = cur;
  }
}

// Coefficients of the extended segment: ghost cells replicate the segment's
// end points (covariance.cpp:38-44 gather_with_ghosts).
struct SegCoef3 {
  const Coef3* t;
  int64_t base, stride;  // flat horizontal index of line element k = base + k*stride
  int64_t start, len, gl;
  __device__ __forceinline__ int64_t at(int64_t e) const {
    int64_t k = e - gl;
    k = k < 0 ? 0 : (k >= len ? len - 1 : k);
    return base + (start + k) * stride;
  }
  __device__ __forceinline__ double a1(int64_t e) const { return t[at(e)].a1; }
  __device__ __forceinline__ double a2(int64_t e) const { return t[at(e)].a2; }
  __device__ __forceinline__ double a3(int64_t e) const { return t[at(e)].a3; }
  __device__ __forceinline__ double b(int64_t e) const { return t[at(e)].b; }
};
struct SegCoef1 {
  const double2* t;
  int64_t base, stride, start, len, gl;
  __device__ __forceinline__ int64_t at(int64_t e) const {
    int64_t k = e - gl;
    k = k < 0 ? 0 : (k >= len ? len - 1 : k);
    return base + (start + k) * stride;
  }
  __device__ __forceinline__ double a1(int64_t e) const { return t[at(e)].x; }
  __device__ __forceinline__ double b(int64_t e) const { return t[at(e)].y; }
};

template <typename T>
__global__ void k_sweep_generic(const T* __restrict__ in, T* __restrict__ out, SweepArgs a) {
  const int64_t n = a.dir == 0 ? a.nx : a.ny;            // line length
  const int64_t lines_per_level = a.dir == 0 ? a.ny : a.nx;
  const int64_t nh = a.nx * a.ny;
  const int64_t total = a.nvar * a.nlev * lines_per_level;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double* v = a.scratch + tid * a.slab;
  const bool third = a.order == 3;
  const bool udc = third && a.unit_dc;
  const int64_t min_len = third ? 4 : 2;

  for (int64_t lid = tid; lid < total; lid += (int64_t)gridDim.x * blockDim.x) {
    const int64_t var = lid / (a.nlev * lines_per_level);
    const int64_t rem = lid - var * a.nlev * lines_per_level;
    const int64_t lev = rem / lines_per_level;
    const int64_t line = rem - lev * lines_per_level;
    const int64_t plane = (var * a.nlev + lev) * nh;
    const int64_t glev = a.lev0 + lev;  // metadata are indexed by global level
    const int64_t hbase = a.dir == 0 ? line * a.nx : line;  // horizontal flat index of k=0
    const int64_t stride = a.dir == 0 ? 1 : a.nx;
    const T* src = in + plane + hbase;
    T* dst = out + plane + hbase;
    const double* pre = a.pre_scale ? a.pre_scale + glev * nh + hbase : nullptr;
    const double* post = a.post_scale ? a.post_scale + glev * nh + hbase : nullptr;
    const int64_t G = a.ghost[glev];
    const int64_t s0 = a.seg_off[glev * lines_per_level + line];
    const int64_t s1 = a.seg_off[glev * lines_per_level + line + 1];

    int64_t cursor = 0;  // land before the next segment stays exactly 0
    for (int64_t s = s0; s < s1; ++s) {
      const int2 sg = a.segs[s];
      const int64_t i = sg.x, len = sg.y, j = i + len - 1;
      for (; cursor < i; ++cursor) dst[cursor * stride] = T(0);
      cursor = j + 1;
      const int64_t gl = i > 0 ? G : 0;
      const int64_t gr = j < n - 1 ? G : 0;
      const int64_t ext = len + gl + gr;
      if (ext < min_len) {  // covariance.cpp:260-269 pass-through
        for (int64_t k = 0; k < len; ++k) {
          double x = double(src[(i + k) * stride]);
          if (pre) x = dmul(x, pre[(i + k) * stride]);
          if (post) x = dmul(x, post[(i + k) * stride]);
          dst[(i + k) * stride] = T(x);
        }
        continue;
      }
      for (int64_t e = 0; e < ext; ++e) v[e] = 0.0;
      for (int64_t k = 0; k < len; ++k) {
        double x = double(src[(i + k) * stride]);
        if (pre) x = dmul(x, pre[(i + k) * stride]);
        v[gl + k] = x;
      }
      if (third) {
        const SegCoef3 c{a.c3, hbase, stride, i, len, gl};
        if (!a.transpose) {
          g_rf3_forward(v, c, ext);
          g_rf3_backward(v, c, ext);
          if (udc)
            for (int64_t e = 0; e < ext; ++e) v[e] = dmul(v[e], a.idc[c.at(e)]);
        } else {
          if (udc)
            for (int64_t e = 0; e < ext; ++e) v[e] = dmul(v[e], a.idc[c.at(e)]);
          g_rf3_backward_transpose(v, c, ext);
          g_rf3_forward_transpose(v, c, ext);
        }
      } else {
        const SegCoef1 c{a.c1, hbase, stride, i, len, gl};
        for (int it = 0; it < a.k; ++it) {
          if (!a.transpose) {
            g_rf1_forward(v, c, ext);
            g_rf1_backward(v, c, ext);
          } else {
            g_rf1_backward_transpose(v, c, ext);
            g_rf1_forward_transpose(v, c, ext);
          }
        }
      }
      for (int64_t k = 0; k < len; ++k) {
        double x = v[gl + k];
        if (post) x = dmul(x, post[(i + k) * stride]);
        dst[(i + k) * stride] = T(x);
      }
    }
    for (; cursor < n; ++cursor) dst[cursor * stride] = T(0);
  }
}

// 1-D entry points (rf3.hpp:292-334, rf1.hpp:113-155): whole vector, no
// ghosts, per-point coefficient arrays shared by the batch of lines.
__global__ void k_apply_1d(const double* in, double* out, const Coef3* c3, const double2* c1,
                           int64_t m, int64_t nlines, int order, int k, int transpose,
                           double* scratch) {
  const int64_t lid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (lid >= nlines) return;
  double* v = scratch + lid * m;
  for (int64_t e = 0; e < m; ++e) v[e] = in[lid * m + e];
  if (order == 3) {
    const SegCoef3 c{c3, 0, 1, 0, m, 0};
    if (!transpose) {
      g_rf3_forward(v, c, m);
      g_rf3_backward(v, c, m);
    } else {
      g_rf3_backward_transpose(v, c, m);
      g_rf3_forward_transpose(v, c, m);
    }
  } else {
    const SegCoef1 c{c1, 0, 1, 0, m, 0};
    for (int it = 0; it < k; ++it) {
      if (!transpose) {
        g_rf1_forward(v, c, m);
        g_rf1_backward(v, c, m);
      } else {
        g_rf1_backward_transpose(v, c, m);
        g_rf1_forward_transpose(v, c, m);
      }
    }
  }
  for (int64_t e = 0; e < m; ++e) out[lid * m + e] = v[e];
}

__global__ void k_coefficients_1d(const double* sigma, int64_t m, int order, int k,
                                  int calibration, Coef3* c3, double2* c1) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (order == 1) {
      const double a = rf1_alpha(sigma[p], k);
      c1[p] = make_double2(a, dsub(1.0, a));
    } else {
      const Scal3 f = rf3_filter_scalars(sigma[p], calibration);
      c3[p] = Coef3{f.alpha1, f.alpha2, f.alpha3, f.beta};
    }
  }
}

// caller-supplied tables -> the device layouts k_apply_1d reads
__global__ void k_pack_tables_1d(const double* a1, const double* a2, const double* a3,
                                 const double* b, int64_t m, Coef3* c3, double2* c1) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (c3) c3[p] = Coef3{a1[p], a2[p], a3[p], b[p]};
    if (c1) c1[p] = make_double2(a1[p], b[p]);
  }
}

// scalar helpers: out[0] = rf3_cascade_variance(x) (mode 0) or
// rf3_length_scale_argument(x, calibration) (mode 1)
__global__ void k_scalar_helper(double x, int calibration, int mode, double* out) {
  if (threadIdx.x != 0) return;
  out[0] = mode == 0 ? rf3_cascade_variance(x) : rf3_length_scale_argument(x, calibration);
}

// coefficient tables of m points, unpacked (rf3_filter_coefficients /
// rf1_coefficients table overload)
__global__ void k_unpack_tables_1d(const Coef3* c3, const double2* c1, int64_t m, double* a1,
                                   double* a2, double* a3, double* b) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < m;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (c3) {
      a1[p] = c3[p].a1;
      a2[p] = c3[p].a2;
      a3[p] = c3[p].a3;
      b[p] = c3[p].b;
    } else {
      a1[p] = c1[p].x;
      b[p] = c1[p].y;
    }
  }
}

}  // namespace rgfb
