// Producer/consumer y-sweep (lines = columns) fed by bulk copies.
//
// One CTA owns a 32-column tile and up to NW planes of it (the planes share
// the tile's coefficients). Warp NW is the producer: it streams U-row stages
// of [planes x rows x 32 columns] field segments, the matching coefficient
// rows and (when needed) the inv_dc rows into an S-deep shared-memory ring
// with cp.async.bulk (TMA engine; completion counted in bytes on the
// stage's `full` mbarrier). Consumer warp w runs the 32 chains (lanes =
// columns) of plane w: it reads its field row and the shared coefficient row
// from shared memory, advances the recursion and stores the result with one
// coalesced 256 B st.global per row, then releases the stage on `empty`.
// Coefficients are loaded once per CTA for all its planes, and the ring
// keeps S*U rows of every plane in flight without spending registers.
//
// PD = false: pass A (ascending rows), TR selects FwdA / AdjA.
// PD = true:  pass D (descending rows) on the intermediate stored by pass A,
//             with the per-segment entry states of k_entries.
#pragma once
#include "async_copy.cuh"
#include "sweep_stream.cuh"
#include "tma.cuh"

namespace rgfb {

template <typename T, int NW, int U>
struct YStage {
  static constexpr size_t field = size_t(NW) * U * 32 * sizeof(T);
  static constexpr size_t coef = size_t(U) * 32 * sizeof(Coef3);
  static constexpr size_t idc = size_t(U) * 32 * sizeof(double);
  static constexpr size_t bytes = field + coef + idc;
};

template <typename T, bool TR, bool PD, int NW, int U, int S>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    k_ybulk(T* __restrict__ out, StreamArgs a, const __grid_constant__ CUtensorMap tm_field,
            const __grid_constant__ CUtensorMap tm_coef, const __grid_constant__ CUtensorMap tm_idc) {
  using L = YStage<T, NW, U>;
  extern __shared__ __align__(1024) unsigned char smem[];
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
  const bool need_idc = a.idc != nullptr && (PD ? !TR : TR);
  const int64_t nst = (ny + U - 1) / U;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwp);
    }
    mbar_fence_init();
  }
  __syncthreads();

  // stage i covers rows [lo, lo+U) (TMA zero-fills rows outside [0, ny))
  auto lo_of = [&](int64_t i) -> int64_t { return PD ? ny - (i + 1) * U : i * U; };

  if (warp == NW) {  // ------------------------------------------ producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_field);
      tma_prefetch_desc(&tm_coef);
      if (need_idc) tma_prefetch_desc(&tm_idc);
      const uint32_t total = static_cast<uint32_t>(L::field + L::coef + (need_idc ? L::idc : 0));
      for (int64_t i = 0; i < nst; ++i) {
        const int s = static_cast<int>(i % S);
        const int64_t n = i / S;
        if (n > 0) mbar_wait(&empty[s], static_cast<uint32_t>((n - 1) & 1));
        const int lo = static_cast<int>(lo_of(i));
        unsigned char* base = smem + s * L::bytes;
        mbar_arrive_expect_tx(&full[s], total);
        tma_load_3d(base, &tm_field, static_cast<int>(ix0), lo, static_cast<int>(p0), &full[s]);
        tma_load_2d(base + L::field, &tm_coef, static_cast<int>(4 * ix0), lo, &full[s]);
        if (need_idc) tma_load_2d(base + L::field + L::coef, &tm_idc, static_cast<int>(ix0), lo,
                                  &full[s]);
      }
    }
    return;
  }
  if (warp >= nwp) return;

  // -------------------------------------------------------------- consumer
  const int64_t p = p0 + warp;
  const int64_t var = p / a.nlev, lev = p - var * a.nlev;
  const bool act = lane < ncol;
  const int64_t ix = ix0 + (act ? lane : 0);
  T* dst = out + p * nh + ix;
  const uint64_t* W = a.bits + (lev * nx + ix) * a.words;
  const double* PRE = (!PD && TR && a.pre_scale) ? a.pre_scale + lev * nh + ix : nullptr;
  const double* POST = (PD && a.post_scale) ? a.post_scale + lev * nh + ix : nullptr;
  const double4* E = a.entry + var * a.nsegs;
  int64_t sidx = 0, sfirst = 0;
  double4 ent = make_double4(0, 0, 0, 0);
  if (PD) {
    sfirst = a.seg_off[lev * nx + ix];
    sidx = a.seg_off[lev * nx + ix + 1] - 1;
    if (sidx >= sfirst) ent = E[sidx];
  }
  typename std::conditional<PD, typename std::conditional<TR, AdjD, FwdD>::type,
                            typename std::conditional<TR, AdjA, FwdA>::type>::type st;
  int64_t widx = -1;
  uint64_t wc = 0;
  int nxt = 0;

  for (int64_t i = 0; i < nst; ++i) {
    const int s = static_cast<int>(i % S);
    mbar_wait(&full[s], static_cast<uint32_t>((i / S) & 1));
    const int64_t lo = lo_of(i);
    const unsigned char* base = smem + s * L::bytes;
    const T* fld = reinterpret_cast<const T*>(base) + warp * U * 32 + lane;
    const Coef3* cf = reinterpret_cast<const Coef3*>(base + L::field) + lane;
    const double* id = reinterpret_cast<const double*>(base + L::field + L::coef) + lane;
    if constexpr (!PD) {
      const int nr = static_cast<int>(ny - lo < U ? ny - lo : U);
      for (int r = 0; r < nr; ++r) {
        const int64_t k = lo + r;
        if ((k >> 6) != widx) {
          widx = k >> 6;
          wc = ldw(W, widx);
        }
        const bool sea = (wc >> (k & 63)) & 1ull;
        const Coef3 c = cf[r * 32];
        double w = static_cast<double>(fld[r * 32]);
        if (TR) {
          if (PRE) w *= __ldg(PRE + k * nx);
          if (need_idc) w *= id[r * 32];
        }
        const double res = st.step(c, w, sea);
        if (act) dst[k * nx] = static_cast<T>(res);
      }
    } else {
      const int rmin = static_cast<int>(lo < 0 ? -lo : 0);
      for (int r = U - 1; r >= rmin; --r) {
        const int64_t k = lo + r;
        if ((k >> 6) != widx) {
          widx = k >> 6;
          wc = ldw(W, widx);
        }
        const int sea = static_cast<int>((wc >> (k & 63)) & 1ull);
        const Coef3 c = cf[r * 32];
        if (sea && !nxt) {
          st.enter(ent, c);
          --sidx;
          if (sidx >= sfirst) ent = E[sidx];
        }
        double o = st.step(c, static_cast<double>(fld[r * 32]));
        if (!TR && need_idc) o *= id[r * 32];
        if (POST) o *= __ldg(POST + k * nx);
        if (act) dst[k * nx] = static_cast<T>(sea ? o : 0.0);
        nxt = sea;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

constexpr int kYbNW = 16, kYbU = 8, kYbS = 4;

// bulk copies need 16 B aligned row starts and sizes
template <typename T>
inline bool ybulk_supported(const T* in, const T* out, int64_t nx) {
  return (nx * static_cast<int64_t>(sizeof(T))) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(in) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0;
}

template <typename T, bool TR, bool PD>
void launch_ybulk(const T* in, T* out, const StreamArgs& a, cudaStream_t st) {
  constexpr int NW = kYbNW, U = kYbU, S = kYbS;
  const size_t smem = S * YStage<T, NW, U>::bytes + 2 * S * sizeof(uint64_t);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_ybulk<T, TR, PD, NW, U, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    attr = true;
  }
  const int64_t planes = a.nvar * a.nlev;
  const uint64_t sz = sizeof(T);
  const uint64_t fd[3] = {uint64_t(a.nx), uint64_t(a.ny), uint64_t(planes)};
  const uint64_t fs[2] = {uint64_t(a.nx) * sz, uint64_t(a.nx * a.ny) * sz};
  const uint32_t fb[3] = {32, U, NW};
  const CUtensorMap tf = make_tmap(PD ? static_cast<const void*>(out) : in, tma_dtype<T>(), 3, fd,
                                   fs, fb, CU_TENSOR_MAP_SWIZZLE_NONE);
  const uint64_t cd[2] = {uint64_t(4 * a.nx), uint64_t(a.ny)};
  const uint64_t cs[1] = {uint64_t(4 * a.nx) * 8};
  const uint32_t cb[2] = {128, U};
  const CUtensorMap tc = make_tmap(a.c3, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, cd, cs, cb,
                                   CU_TENSOR_MAP_SWIZZLE_NONE);
  const uint64_t id[2] = {uint64_t(a.nx), uint64_t(a.ny)};
  const uint64_t is[1] = {uint64_t(a.nx) * 8};
  const uint32_t ib[2] = {32, U};
  const CUtensorMap ti = a.idc ? make_tmap(a.idc, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, id, is, ib,
                                           CU_TENSOR_MAP_SWIZZLE_NONE)
                               : tc;
  const int64_t blocks = ((a.nx + 31) / 32) * ((planes + NW - 1) / NW);
  k_ybulk<T, TR, PD, NW, U, S><<<blocks, 32 * (NW + 1), smem, st>>>(out, a, tf, tc, ti);
}

}  // namespace rgfb

namespace rgfb {

// Producer/consumer x-sweep (lines = rows). The CTA owns 32*NW consecutive
// chains of the plane-fastest (row, plane) order, so each warp's lanes are
// mostly the same row of consecutive planes and share coefficient reads.
// Stage = U consecutive x positions of every chain: the producer bulk-copies
// each chain's U-element row segment into a padded tile (pitch XBP) and the
// coefficient/inv_dc segments of the CTA's (few) distinct rows. A consumer
// lane walks its own chain through the tile, writes results in place, and
// the warp returns its 32 segments to global memory with bulk stores
// (smem -> global), so every global access is a contiguous 16 B-aligned
// bulk transfer. Stage release is deferred one stage so the stores' smem
// reads overlap the next stage's recursion.
template <typename T, int NW, int U>
struct XStage {
  static constexpr int pitch = U + 16 / int(sizeof(T));  // 16 B pad, keeps bulk alignment
  static constexpr int rows = 9;                          // distinct rows per CTA (planes >= 16)
  static constexpr size_t field = size_t(NW) * 32 * pitch * sizeof(T);
  static constexpr size_t coef = size_t(rows) * U * sizeof(Coef3);
  static constexpr size_t idc = size_t(rows) * U * sizeof(double);
  static constexpr size_t bytes = field + coef + idc;
};

template <typename T, bool TR, bool PD, int NW, int U, int S>
__global__ void __launch_bounds__(32 * (NW + 1), 1)
    k_xbulk(const T* __restrict__ in, T* __restrict__ out, StreamArgs a) {
  using L = XStage<T, NW, U>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * L::bytes);
  uint64_t* empty = full + S;

  const int64_t n = a.nx, ny = a.ny, nh = n * ny;
  const int64_t planes = a.nvar * a.nlev;
  const int64_t chains = planes * ny;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32 * NW;
  const int nch = static_cast<int>(chains - c0 < 32 * NW ? chains - c0 : 32 * NW);
  const int nwp = (nch + 31) / 32;
  const int64_t row0 = c0 / planes;
  const int nrows = static_cast<int>((c0 + nch - 1) / planes - row0 + 1);
  const bool need_idc = a.idc != nullptr && (PD ? !TR : TR);
  const int64_t nst = (n + U - 1) / U;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwp);
    }
    mbar_fence_init();
  }
  __syncthreads();

  auto cols_of = [&](int64_t i, int64_t& k0, int& nk) {
    const int64_t b = PD ? nst - 1 - i : i;
    k0 = b * U;
    nk = static_cast<int>(n - k0 < U ? n - k0 : U);
  };

  if (warp == NW) {  // ------------------------------------------ producer
    const T* src = PD ? out : in;
    for (int64_t i = 0; i < nst; ++i) {
      const int s = static_cast<int>(i % S);
      const int64_t m = i / S;
      if (m > 0) mbar_wait(&empty[s], static_cast<uint32_t>((m - 1) & 1));
      int64_t k0;
      int nk;
      cols_of(i, k0, nk);
      const uint32_t fbytes = static_cast<uint32_t>(nk * sizeof(T));
      const uint32_t cbytes = static_cast<uint32_t>(nk * sizeof(Coef3));
      const uint32_t ibytes = static_cast<uint32_t>(nk * sizeof(double));
      const uint32_t total = static_cast<uint32_t>(nch) * fbytes + nrows * cbytes +
                             (need_idc ? nrows * ibytes : 0u);
      if (lane == 0) mbar_arrive_expect_tx(&full[s], total);
      __syncwarp();
      unsigned char* base = smem + s * L::bytes;
      T* fld = reinterpret_cast<T*>(base);
      Coef3* cf = reinterpret_cast<Coef3*>(base + L::field);
      double* id = reinterpret_cast<double*>(base + L::field + L::coef);
      for (int j = lane; j < nch; j += 32) {
        const int64_t c = c0 + j;
        const int64_t iy = c / planes, p = c - iy * planes;
        bulk_g2s(fld + j * L::pitch, src + p * nh + iy * n + k0, fbytes, &full[s]);
      }
      for (int r = lane; r < nrows; r += 32) {
        bulk_g2s(cf + r * U, a.c3 + (row0 + r) * n + k0, cbytes, &full[s]);
        if (need_idc) bulk_g2s(id + r * U, a.idc + (row0 + r) * n + k0, ibytes, &full[s]);
      }
    }
    return;
  }
  if (warp >= nwp) return;

  // -------------------------------------------------------------- consumer
  const int j = warp * 32 + lane;
  const bool act = j < nch;
  const int64_t c = c0 + (act ? j : 0);
  const int64_t iy = c / planes, p = c - iy * planes;
  const int64_t var = p / a.nlev, lev = p - var * a.nlev;
  const int rr = static_cast<int>(iy - row0);
  T* dst = out + p * nh + iy * n;
  const uint64_t* W = a.bits + (lev * ny + iy) * a.words;
  const double* PRE = (!PD && TR && a.pre_scale) ? a.pre_scale + lev * nh + iy * n : nullptr;
  const double* POST = (PD && a.post_scale) ? a.post_scale + lev * nh + iy * n : nullptr;
  const double4* E = a.entry + var * a.nsegs;
  int64_t sidx = 0, sfirst = 0;
  double4 ent = make_double4(0, 0, 0, 0);
  if (PD) {
    sfirst = a.seg_off[lev * ny + iy];
    sidx = a.seg_off[lev * ny + iy + 1] - 1;
    if (sidx >= sfirst) ent = E[sidx];
  }
  typename std::conditional<PD, typename std::conditional<TR, AdjD, FwdD>::type,
                            typename std::conditional<TR, AdjA, FwdA>::type>::type st;
  int nxt = 0;

  for (int64_t i = 0; i < nst; ++i) {
    const int s = static_cast<int>(i % S);
    mbar_wait(&full[s], static_cast<uint32_t>((i / S) & 1));
    int64_t k0;
    int nk;
    cols_of(i, k0, nk);
    unsigned char* base = smem + s * L::bytes;
    T* row = reinterpret_cast<T*>(base) + j * L::pitch;
    const Coef3* cf = reinterpret_cast<const Coef3*>(base + L::field) + rr * U;
    const double* id = reinterpret_cast<const double*>(base + L::field + L::coef) + rr * U;
    const uint64_t wc = ldw(W, k0 >> 6);
    if constexpr (!PD) {
      for (int u = 0; u < nk; ++u) {
        const int64_t k = k0 + u;
        const bool sea = (wc >> (k & 63)) & 1ull;
        double w = static_cast<double>(row[u]);
        if (TR) {
          if (PRE) w *= __ldg(PRE + k);
          if (need_idc) w *= id[u];
        }
        row[u] = static_cast<T>(st.step(cf[u], w, sea));
      }
    } else {
      for (int u = nk - 1; u >= 0; --u) {
        const int64_t k = k0 + u;
        const int sea = static_cast<int>((wc >> (k & 63)) & 1ull);
        const Coef3 cc = cf[u];
        if (sea && !nxt) {
          st.enter(ent, cc);
          --sidx;
          if (sidx >= sfirst) ent = E[sidx];
        }
        double o = st.step(cc, static_cast<double>(row[u]));
        if (!TR && need_idc) o *= id[u];
        if (POST) o *= __ldg(POST + k);
        row[u] = static_cast<T>(sea ? o : 0.0);
        nxt = sea;
      }
    }
    // results back to global with one bulk store per chain
    fence_proxy_async_smem();
    __syncwarp();
    if (act) bulk_s2g(dst + k0, row, static_cast<uint32_t>(nk * sizeof(T)));
    bulk_commit();
    // release the previous stage once its stores have read shared memory
    asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
    __syncwarp();
    if (i > 0 && lane == 0) mbar_arrive(&empty[(i - 1) % S]);
  }
  bulk_wait_all();
}

constexpr int kXbNW = 4, kXbU = 32, kXbS = 4;

template <typename T>
inline bool xbulk_supported(const T* in, const T* out, int64_t nx, int64_t planes) {
  return planes >= 16 && (nx * static_cast<int64_t>(sizeof(T))) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(in) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0;
}

template <typename T, bool TR, bool PD>
void launch_xbulk(const T* in, T* out, const StreamArgs& a, cudaStream_t st) {
  constexpr int NW = kXbNW, U = kXbU, S = kXbS;
  const size_t smem = S * XStage<T, NW, U>::bytes + 2 * S * sizeof(uint64_t);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_xbulk<T, TR, PD, NW, U, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    attr = true;
  }
  const int64_t chains = a.nvar * a.nlev * a.ny;
  const int64_t blocks = (chains + 32 * NW - 1) / (32 * NW);
  k_xbulk<T, TR, PD, NW, U, S><<<blocks, 32 * (NW + 1), smem, st>>>(in, out, a);
}

}  // namespace rgfb
