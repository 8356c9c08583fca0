// Line-resident 1st-RF: all K iterations of a line in one pass over HBM.
//
// The streaming 1st-RF (rf1_stream.cuh) runs 2K passes over the field, each
// reading and writing every element (C5 fp64 K=5: 20 passes x 3.5 ms). But a
// sea segment's K iterations depend only on the segment itself: its values,
// its coefficients and its two ghost zones, which rf1_stream.cuh already
// reduces to the per-segment responses hL / cR (k_rf1_zones) and the
// boundary histories x_j, y_j:
//   ascending pass of iteration it enters with  E_L(it) = sum_{j<it}  hL[it-j] x_j
//   descending pass of iteration it enters with E_R(it) = sum_{j<=it} cR[it-j] y_j
// (rf1.hpp:113-137 with the ghost steps collapsed, covariance.cpp:283-286).
//
// So a CTA stages one line group (x: a row; y: KC adjacent columns) of one
// plane in shared memory with one bulk/TMA copy, the lanes of a warp take the
// line's segments, each lane runs its segment's 2K first-order passes
// in place, land is set to 0 (covariance.cpp:355), and the line goes back with
// one copy: one field read and one field write per sweep instead of 2K.
// Every warp works on its own plane; the coefficients (alpha, beta) of the
// line group are staged once per CTA and shared by all planes.
//
// The per-point arithmetic, the entry sums and the per-pass rounding of the
// stored values to T are the streaming kernels' (Rf1Asc), so results are
// bit-identical to them.
#pragma once
#include "rf1_stream.cuh"

namespace rgfb {

constexpr int kRf1SegKMax = 8;  // iterations supported by the line-resident kernel

template <typename T, int DIR>
struct Rf1SegL {
  static constexpr int KC = DIR == 0 ? 1 : 16 / int(sizeof(T));  // lines per group
};

// rows held per line group: y boxes are 256 rows (TMA fills past the end)
template <int DIR>
__host__ __device__ __forceinline__ int64_t rf1_seg_rows(int64_t n) {
  return DIR == 0 ? n : (n + 255) / 256 * 256;
}
// smem: coefficients [rows][KC] double2, then NW line buffers [rows][KC] T,
// then NW + 1 mbarriers
template <typename T, int DIR>
__host__ __device__ __forceinline__ size_t rf1_seg_coef_bytes(int64_t n) {
  return static_cast<size_t>(rf1_seg_rows<DIR>(n)) * Rf1SegL<T, DIR>::KC * 16;
}
template <typename T, int DIR>
__host__ __device__ __forceinline__ size_t rf1_seg_line_bytes(int64_t n) {
  return (static_cast<size_t>(rf1_seg_rows<DIR>(n)) * Rf1SegL<T, DIR>::KC * sizeof(T) + 127) /
         128 * 128;
}
template <typename T, int DIR>
size_t rf1_seg_smem(int64_t n, int nw) {
  return 1024 + rf1_seg_coef_bytes<T, DIR>(n) + nw * rf1_seg_line_bytes<T, DIR>(n) + (nw + 1) * 8;
}

template <typename T, int DIR, bool TR, bool PRE, bool POST, int KM>
__global__ void __launch_bounds__(256) k_rf1_seg(Rf1Args a, const __grid_constant__ CUtensorMap tm_in,
                                                 const __grid_constant__ CUtensorMap tm_out,
                                                 const __grid_constant__ CUtensorMap tm_coef,
                                                 const T* in, T* out) {
  constexpr int KC = Rf1SegL<T, DIR>::KC;
  constexpr int RB = 256;  // rows per y box
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int NW = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nx = a.nx, ny = a.ny, nh = nx * ny;
  const int n = static_cast<int>(DIR == 0 ? nx : ny);
  const int K = a.k;
  const int64_t planes = a.nvar * a.nlev;
  const size_t coef_bytes = rf1_seg_coef_bytes<T, DIR>(n);
  const size_t line_bytes = rf1_seg_line_bytes<T, DIR>(n);
  double2* cf = reinterpret_cast<double2*>(smem);
  T* buf = reinterpret_cast<T*>(smem + coef_bytes + warp * line_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + coef_bytes + NW * line_bytes);
  uint64_t* cbar = bars + NW;
  uint64_t* lbar = bars + warp;

  const int64_t g = blockIdx.x;  // line group: x row iy, y columns [ix0, ix0 + KC)
  const int64_t iy = DIR == 0 ? g : 0;
  const int64_t ix0 = DIR == 0 ? 0 : g * KC;
  const int ncol = DIR == 0 ? 1 : static_cast<int>(nx - ix0 < KC ? nx - ix0 : KC);
  const int64_t nlines = DIR == 0 ? ny : nx;
  const int64_t words = (n + 63) / 64;
  const int64_t hstride = DIR == 0 ? 1 : nx;  // horizontal index of position i: hb(c) + i*hstride
  auto hb = [&](int c) -> int64_t { return DIR == 0 ? iy * nx : ix0 + c; };
  auto el = [&](int i, int c) -> int { return DIR == 0 ? i : i * KC + c; };

  if (threadIdx.x == 0) {
    for (int w = 0; w < NW + 1; ++w) mbar_init(&bars[w], 1);
    mbar_fence_init();
  }
  __syncthreads();
  // the group's coefficients, once per CTA
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(cbar, static_cast<uint32_t>(coef_bytes));
    if constexpr (DIR == 0) {
      bulk_g2s(cf, a.c1 + iy * nx, static_cast<uint32_t>(coef_bytes), cbar);  // dense rows
    } else {
      for (int r = 0; r < n; r += RB)
        tma_load_2d(cf + r * KC, &tm_coef, static_cast<int>(2 * ix0), r, cbar, l2_evict_last());
    }
  }
  // the plane's line group into this warp's buffer
  auto issue_load = [&](int64_t p) {  // lane 0
    if constexpr (DIR == 0) {
      mbar_arrive_expect_tx(lbar, static_cast<uint32_t>(n * sizeof(T)));
      bulk_g2s(buf, in + (p * ny + iy) * nx, static_cast<uint32_t>(n * sizeof(T)), lbar);
    } else {
      const int nbox = (n + RB - 1) / RB;
      mbar_arrive_expect_tx(lbar, static_cast<uint32_t>(nbox * RB * KC * sizeof(T)));
      for (int r = 0; r < n; r += RB)
        tma_load_3d(buf + r * KC, &tm_in, static_cast<int>(ix0), r, static_cast<int>(p), lbar,
                    l2_evict_first());
    }
  };
  int64_t p = warp;
  int phase = 0;
  if (lane == 0 && p < planes) issue_load(p);
  mbar_wait(cbar, 0);

  for (; p < planes; p += NW, phase ^= 1) {
    const int64_t var = p / a.nlev, lev = a.lev0 + (p - var * a.nlev);
    (void)var;
    mbar_wait(lbar, static_cast<uint32_t>(phase));

    // ---- land = 0 (covariance.cpp:355): each lane takes whole mask words
    for (int c = 0; c < ncol; ++c) {
      const uint64_t* W = a.bits + (lev * nlines + (DIR == 0 ? iy : ix0 + c)) * words;
      for (int64_t w = lane; w < words; w += 32) {
        uint64_t land = ~ldw(W, w);
        const int lim = static_cast<int>(n - w * 64 < 64 ? n - w * 64 : 64);
        if (lim < 64) land &= (1ull << lim) - 1ull;
        while (land) {
          const int b = __ffsll(static_cast<long long>(land)) - 1;
          land &= land - 1ull;
          buf[el(static_cast<int>(w * 64 + b), c)] = static_cast<T>(0.0);
        }
      }
    }

    // ---- the group's segments in rounds: the line's segments sorted longest
    // first (k_rf1_sort, construction) and dealt to the B = 32/KC lanes of
    // each column, one per lane per round. Within a round every lane runs the
    // same K iterations x 2 passes x (longest length of the round) steps under
    // a predicate, so control flow is uniform and the step loop is tight;
    // sorting keeps the lengths of a round close.
    {
      constexpr int B = 32 / KC;  // lanes per line
      constexpr int U = 8;        // steps per load batch
      const int c = lane / B, bin = lane - (lane / B) * B;
      const int64_t line = DIR == 0 ? iy : ix0 + c;
      const bool okc = c < ncol;
      const int64_t lg = lev * nlines + line;
      const int64_t sbase = okc ? a.seg_off[lg] : 0;
      const int64_t scnt = okc ? a.seg_off[lg + 1] - sbase : 0;
      const int rounds = static_cast<int>(
          __reduce_max_sync(0xffffffffu, static_cast<unsigned>((scnt + B - 1) / B)));
      const int64_t h0 = hb(okc ? c : 0);
      for (int r = 0; r < rounds; ++r) {
        const int64_t k = static_cast<int64_t>(r) * B + bin;
        const bool has = k < scnt;
        int2 sg = make_int2(0, 1);
        double z[2 * KM];
        {
          const int64_t sx = has ? a.lpt_ord[sbase + k] : 0;
          if (has) sg = a.segs[sx];
#pragma unroll
          for (int d = 0; d < 2 * KM; ++d)
            z[d] = (has && (d < KM ? d < K : d - KM < K))
                       ? __ldg(a.zone + (d < KM ? d : K + d - KM) * a.nsegs + sx)
                       : 0.0;
        }
        const int len = has ? sg.y : 0;
        const int L = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(len)));
        const int i0 = sg.x, i1 = sg.x + sg.y - 1;
        const double a0 = cf[el(i0, c)].x, a1 = cf[el(i1, c)].x;
        double xh[KM], yh[KM];
#pragma unroll
        for (int j = 0; j < KM; ++j) xh[j] = yh[j] = 0.0;
        Rf1Asc st;
#pragma unroll 1
        for (int it = 1; it <= K; ++it) {
          // ascending pass (rf1_forward / rf1_backward_transpose)
          {
            double e = 0.0;
#pragma unroll
            for (int j = 1; j < KM; ++j)
#pragma unroll
              for (int m = 1; m < KM; ++m)
                if (j + m == it) e = fma(z[m], xh[j - 1], e);
            st.st = e;
            st.ap = a0;
          }
          // steps in chunks of U: all loads first (clamped into the segment),
          // then the recursion, then the predicated stores
          for (int u0 = 0; u0 < L; u0 += U) {
            int q[U];
            double2 cc[U];
            double w[U];
#pragma unroll
            for (int t = 0; t < U; ++t) {
              const int uu = u0 + t < len ? u0 + t : (len > 0 ? len - 1 : 0);
              q[t] = el(i0 + uu, c);
              cc[t] = cf[q[t]];
              w[t] = static_cast<double>(buf[q[t]]);
            }
#pragma unroll
            for (int t = 0; t < U; ++t) {
              if (u0 + t < len) {
                double wt = w[t];
                if constexpr (TR && PRE)
                  if (it == 1) wt *= __ldg(a.pre_scale + lev * nh + h0 + (i0 + u0 + t) * hstride);
                buf[q[t]] = static_cast<T>(st.template step<TR>(cc[t].x, cc[t].y, wt));
              }
            }
          }
          {
            double e = 0.0;
#pragma unroll
            for (int j = 0; j < KM; ++j)
              if (j == it - 1) yh[j] = st.st;
#pragma unroll
            for (int j = 1; j <= KM; ++j)  // j ascending; m = it - j (static indices)
#pragma unroll
              for (int m = 0; m < KM; ++m)
                if (j + m == it) e = fma(z[KM + m], yh[j - 1], e);
            st.st = e;
            st.ap = a1;
          }
          // descending pass (rf1_backward / rf1_forward_transpose)
          for (int u0 = 0; u0 < L; u0 += U) {
            int q[U];
            double2 cc[U];
            double w[U];
#pragma unroll
            for (int t = 0; t < U; ++t) {
              const int uu = u0 + t < len ? u0 + t : (len > 0 ? len - 1 : 0);
              q[t] = el(i1 - uu, c);
              cc[t] = cf[q[t]];
              w[t] = static_cast<double>(buf[q[t]]);
            }
#pragma unroll
            for (int t = 0; t < U; ++t) {
              if (u0 + t < len) {
                double o = st.template step<TR>(cc[t].x, cc[t].y, w[t]);
                if constexpr (POST)
                  if (it == K) o *= __ldg(a.post_scale + lev * nh + h0 + (i1 - u0 - t) * hstride);
                buf[q[t]] = static_cast<T>(o);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < KM; ++j)
            if (j == it - 1) xh[j] = st.st;
        }
      }
    }
    __syncwarp();

    // ---- the line group back to HBM; then this buffer takes the next plane
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      if constexpr (DIR == 0) {
        bulk_s2g(out + (p * ny + iy) * nx, buf, static_cast<uint32_t>(n * sizeof(T)));
      } else {
        for (int r = 0; r < n; r += RB)
          tma_store_3d(&tm_out, static_cast<int>(ix0), r, static_cast<int>(p), buf + r * KC,
                       l2_evict_first());
      }
      bulk_commit();
      if (p + NW < planes) {
        bulk_wait_read_all();
        issue_load(p + NW);
      }
    }
    __syncwarp();
  }
  if (lane == 0) bulk_wait_all();
}

// Construction: per (level, line), the line's segments sorted longest first
// (stable), written into ord[seg_off[line] ...). One thread per line.
__global__ void k_rf1_sort(const int64_t* __restrict__ seg_off, const int2* __restrict__ segs,
                           int64_t lines, int32_t* __restrict__ ord) {
  for (int64_t ln = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ln < lines;
       ln += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s0 = seg_off[ln], cnt = seg_off[ln + 1] - s0;
    int32_t* o = ord + s0;
    for (int64_t k = 0; k < cnt; ++k) {  // insertion sort on the output slots
      const int len = segs[s0 + k].y;
      int64_t j = k;
      while (j > 0 && segs[o[j - 1]].y < len) {
        o[j] = o[j - 1];
        --j;
      }
      o[j] = static_cast<int32_t>(s0 + k);
    }
  }
}

// Launch if the line group fits (returns false to fall back on the streaming
// passes): dense rows 16 B aligned, K <= kRf1SegKMax, coefficients + >= 1
// line buffer within the shared-memory budget.
template <typename T, int DIR, bool TR, bool PRE, bool POST>
void launch_rf1_seg_dir(const T* in, T* out, const Rf1Args& a, int nw, cudaStream_t st) {
  constexpr int KC = Rf1SegL<T, DIR>::KC;
  const int64_t n = DIR == 0 ? a.nx : a.ny;
  const size_t smem = rf1_seg_smem<T, DIR>(n, nw);
  auto kern = a.k <= 5 ? k_rf1_seg<T, DIR, TR, PRE, POST, 5> : k_rf1_seg<T, DIR, TR, PRE, POST, 8>;
  static size_t attr5 = 0, attr8 = 0;
  size_t& attr = a.k <= 5 ? attr5 : attr8;
  if (attr < smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = smem;
  }
  const int64_t planes = a.nvar * a.nlev;
  const uint64_t sz = sizeof(T);
  CUtensorMap tin{}, tout{}, tc{};
  if (DIR == 1) {
    // field (x, y, plane); box {KC, 256 rows, 1}
    const uint64_t fd[3] = {uint64_t(a.nx), uint64_t(a.ny), uint64_t(planes)};
    const uint64_t fs[2] = {uint64_t(a.nx) * sz, uint64_t(a.nx * a.ny) * sz};
    const uint32_t fb[3] = {uint32_t(KC), 256u, 1u};
    tin = make_tmap(in, tma_dtype<T>(), 3, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_NONE);
    tout = make_tmap(out, tma_dtype<T>(), 3, fd, fs, fb, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE);
    // coefficients [ny][nx] (alpha, beta) as doubles [ny][2 nx]; box {2 KC, 256}
    const uint64_t cd[2] = {uint64_t(2 * a.nx), uint64_t(a.ny)};
    const uint64_t cs[1] = {uint64_t(2 * a.nx) * 8};
    const uint32_t cb[2] = {uint32_t(2 * KC), 256u};
    tc = make_tmap(a.c1, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, cd, cs, cb, CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  const int64_t groups = DIR == 0 ? a.ny : (a.nx + KC - 1) / KC;
  kern<<<groups, 32 * nw, smem, st>>>(a, tin, tout, tc, in, out);
}

// warps per CTA for the line-resident kernel (0: does not fit)
template <typename T>
int rf1_seg_warps(const Rf1Args& a) {
  const int64_t n = a.dir == 0 ? a.nx : a.ny;
  constexpr size_t budget = 227 * 1024;
  const int64_t planes = a.nvar * a.nlev;
  for (int nw = 8; nw >= 1; nw /= 2) {
    if (nw > 1 && nw > planes) continue;
    const size_t s = a.dir == 0 ? rf1_seg_smem<T, 0>(n, nw) : rf1_seg_smem<T, 1>(n, nw);
    if (s <= budget) return nw;
  }
  return 0;
}

template <typename T>
bool launch_rf1_seg(const T* in, T* out, const Rf1Args& a, cudaStream_t st) {
  if (a.k > kRf1SegKMax || a.k < 1 || a.segs == nullptr || a.lpt_ord == nullptr) return false;
  if (!tma_supported(in, out, a.nx)) return false;
  const int64_t n = a.dir == 0 ? a.nx : a.ny;
  if (n > (int64_t(1) << 24)) return false;
  const int nw = rf1_seg_warps<T>(a);
  if (nw == 0) return false;
  const bool pre = a.transpose && a.pre_scale != nullptr;
  const bool post = a.post_scale != nullptr;
#define RGFB_SEG(D, TR, P, Q) launch_rf1_seg_dir<T, D, TR, P, Q>(in, out, a, nw, st);
#define RGFB_SEG_D(TR, P, Q)  \
  if (a.dir == 0) {           \
    RGFB_SEG(0, TR, P, Q)     \
  } else {                    \
    RGFB_SEG(1, TR, P, Q)     \
  }
  if (a.transpose) {
    if (pre) {
      if (post) { RGFB_SEG_D(true, true, true) } else { RGFB_SEG_D(true, true, false) }
    } else {
      if (post) { RGFB_SEG_D(true, false, true) } else { RGFB_SEG_D(true, false, false) }
    }
  } else {
    if (post) { RGFB_SEG_D(false, false, true) } else { RGFB_SEG_D(false, false, false) }
  }
#undef RGFB_SEG_D
#undef RGFB_SEG
  return true;
}

}  // namespace rgfb
