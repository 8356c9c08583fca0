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
    k_ybulk(const T* __restrict__ in, T* __restrict__ out, StreamArgs a) {
  using L = YStage<T, NW, U>;
  extern __shared__ __align__(128) unsigned char smem[];
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

  auto rows_of = [&](int64_t i, int64_t& lo, int& nr) {
    if (!PD) {
      lo = i * U;
      nr = static_cast<int>(ny - lo < U ? ny - lo : U);
    } else {
      const int64_t hi = ny - 1 - i * U;
      lo = hi - U + 1 < 0 ? 0 : hi - U + 1;
      nr = static_cast<int>(hi - lo + 1);
    }
  };

  if (warp == NW) {  // ------------------------------------------ producer
    const T* src = PD ? out : in;
    for (int64_t i = 0; i < nst; ++i) {
      const int s = static_cast<int>(i % S);
      const int64_t n = i / S;
      if (n > 0) mbar_wait(&empty[s], static_cast<uint32_t>((n - 1) & 1));
      int64_t lo;
      int nr;
      rows_of(i, lo, nr);
      const uint32_t fbytes = static_cast<uint32_t>(ncol * sizeof(T));
      const uint32_t cbytes = static_cast<uint32_t>(ncol * sizeof(Coef3));
      const uint32_t ibytes = static_cast<uint32_t>(ncol * sizeof(double));
      const uint32_t total = static_cast<uint32_t>(nwp * nr) * fbytes + nr * cbytes +
                             (need_idc ? nr * ibytes : 0u);
      if (lane == 0) mbar_arrive_expect_tx(&full[s], total);
      __syncwarp();
      unsigned char* base = smem + s * L::bytes;
      T* fld = reinterpret_cast<T*>(base);
      Coef3* cf = reinterpret_cast<Coef3*>(base + L::field);
      double* id = reinterpret_cast<double*>(base + L::field + L::coef);
      for (int j = lane; j < nwp * nr; j += 32) {
        const int w = j / nr, r = j - (j / nr) * nr;
        bulk_g2s(fld + (w * U + r) * 32, src + (p0 + w) * nh + (lo + r) * nx + ix0, fbytes,
                 &full[s]);
      }
      for (int r = lane; r < nr; r += 32) {
        bulk_g2s(cf + r * 32, a.c3 + (lo + r) * nx + ix0, cbytes, &full[s]);
        if (need_idc) bulk_g2s(id + r * 32, a.idc + (lo + r) * nx + ix0, ibytes, &full[s]);
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
    int64_t lo;
    int nr;
    rows_of(i, lo, nr);
    const unsigned char* base = smem + s * L::bytes;
    const T* fld = reinterpret_cast<const T*>(base) + warp * U * 32 + lane;
    const Coef3* cf = reinterpret_cast<const Coef3*>(base + L::field) + lane;
    const double* id = reinterpret_cast<const double*>(base + L::field + L::coef) + lane;
    if constexpr (!PD) {
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
      for (int r = nr - 1; r >= 0; --r) {
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
  const int64_t blocks = ((a.nx + 31) / 32) * ((planes + NW - 1) / NW);
  k_ybulk<T, TR, PD, NW, U, S><<<blocks, 32 * (NW + 1), smem, st>>>(in, out, a);
}

}  // namespace rgfb
