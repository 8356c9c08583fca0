// C ABI of the B200-native covariance operator (include/rgf_b200.h).
//
// Host side of the drop-in boundary: HorizontalCovarianceOp construction
// (covariance.cpp:155-220) becomes validation + coefficient precompute +
// segmentation kernels; the seven apply_* methods (covariance.cpp:362-398)
// become sequences of sweep kernels on one CUDA stream. No CPU arithmetic
// touches field values.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/rgf_b200.h"
#include "common.cuh"
#include "setup_kernels.cuh"
#include "sweep_generic.cuh"
#include "sweep_stream.cuh"
#include "sweep_tma.cuh"
#include "sweep_ckpt.cuh"
#include "sweep_few.cuh"
#include "rf1_stream.cuh"
#include "rf1_line.cuh"
#include "closures.cuh"
#include "solver_kernels.cuh"
#include "container_io.cuh"
#include "diag_kernels.cuh"

namespace {

thread_local std::string g_last_error;

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CUDA_OK(expr)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw CudaError(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " +   \
                      __FILE__ + ":" + std::to_string(__LINE__) + " (" #expr ")");   \
  } while (0)

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return RGF_OK;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return RGF_ECUDA;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return RGF_EINVAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return RGF_ERUNTIME;
  }
}

// RGF_B200_DEBUG_POISON=1: fill every new device buffer with 0xff bytes, so a
// read of memory nobody wrote shows up deterministically
bool debug_poison() {
  static const bool on = [] {
    const char* e = std::getenv("RGF_B200_DEBUG_POISON");
    return e && e[0] == '1';
  }();
  return on;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  // Buffers only grow; a growing apply-scratch buffer may still be read by
  // kernels in flight on a non-blocking stream (e.g. the checkpoint buffer of
  // a transposed x sweep while the y sweep re-sizes it), and cudaFree does
  // not wait for those: drain the device first (rare: growth only).
  bool owned = true;
  void release() {
    if (p && owned) {
      cudaDeviceSynchronize();
      cudaFree(p);
    }
    p = nullptr;
    n = 0;
    owned = true;
  }
  // a view of memory owned elsewhere (never freed here)
  void borrow(T* ptr, size_t count) {
    release();
    p = ptr;
    n = count;
    owned = false;
  }
  void alloc(size_t count) {
    if (count <= n && p) return;
    release();
    if (count == 0) return;
    CUDA_OK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
    if (debug_poison()) CUDA_OK(cudaMemset(p, 0xff, count * sizeof(T)));  // NaN / -1 patterns
  }
  void upload(const T* h, size_t count) {
    alloc(count);
    CUDA_OK(cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice));
  }
  size_t bytes() const { return n * sizeof(T); }
};

// RGF_B200_DEBUG_SYNC=1: synchronize and check after every launch group, so
// an asynchronous fault is reported at the launch that caused it
// (compute-sanitizer is not available on the GPU pool)
bool debug_sync() {
  static const bool on = [] {
    const char* e = std::getenv("RGF_B200_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  return on;
}
#define RGF_DEBUG_SYNC(st, what)                                                      \
  do {                                                                               \
    if (debug_sync()) {                                                              \
      const cudaError_t e2_ = cudaStreamSynchronize(st);                            \
      if (e2_ != cudaSuccess)                                                        \
        throw CudaError(std::string("debug sync after ") + (what) + ": " +           \
                        cudaGetErrorString(e2_));                                    \
    }                                                                                \
  } while (0)

int grid_for(int64_t work, int threads, int max_blocks = 148 * 16) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return static_cast<int>(b);
}

struct DirData {
  DevBuf<rgfb::Coef3> c3;
  DevBuf<double> c3s;  // SoA copy of c3 (y direction, checkpointed sweeps)
  DevBuf<double> idcp;  // inv_dc with even row pitch when nx is odd (TMA)
  DevBuf<double> zone[2];  // 1st-RF ghost-zone responses per segment [fwd, adjoint]
  DevBuf<double2> c1;
  DevBuf<double> idc;
  DevBuf<int64_t> seg_off;  // nlev*lines + 1
  std::vector<int64_t> seg_off_h;  // host copy (1st-RF level-chunk segment ranges)
  int segcap = 0;                   // most segments on one line (line-resident 1st-RF)
  DevBuf<int2> segs;
  DevBuf<int32_t> seg_line;  // per segment: lev*lines + line
  DevBuf<int64_t> close_order;  // segments sorted by (line, end, level)
  int64_t nsegs = 0;
  std::vector<char> uniform;        // per level
  std::vector<double> sigma_u;      // per level, uniform sigma value
};

}  // namespace

struct rgf_op {
  int device = 0;
  int64_t nx = 0, ny = 0, nlev = 0;
  int order = 3, k = 1, unit_dc = 1, calibration = 0;
  std::vector<uint8_t> mask0;  // level-0 mask on the host (observation stencils, obs.cpp:38-41)
  std::vector<int64_t> ghost;  // per level
  int64_t gmax = 0;
  DevBuf<int> ghost_d;
  DirData dx_, dy_;
  DevBuf<double> variance;
  bool has_variance = false;
  // apply-time buffers (grown on demand)
  DevBuf<char> in_d, out_d, tmp1, tmp2;
  DevBuf<double> scratch;
  int64_t scratch_threads = 0, scratch_slab = 0;
  cudaStream_t own_stream = nullptr;
  unsigned long long launches = 0;
  // streaming 3rd-RF path: bit-packed masks, closure classes and tables
  bool stream_ok = false;
  bool ckpt_ok = true;  // TMA-fed sweeps (checkpointed / single-pass) for this op's tables
  // few-plane x sweeps on the transposed field (lanes = rows instead of
  // planes): default on; RGF_B200_XT=0 at creation turns it off
  bool xt_mode = true;
  bool rf1_ok = false;  // streaming 1st-RF (ghost zones as per-segment convolutions)
  DevBuf<double> cg_aux;      // dot partials, observation-space temporaries, one field (Cg)
  DevBuf<double> cg_work;     // CG vectors of rgf_solve (b, chi, r, p, Ap, t, background, misfit)
  DevBuf<uint8_t> mask_same;  // per level: mask and ghost width equal the previous level's
  bool rf1_stream = true;  // streaming passes usable (every level has ghosts)
  bool rf1_line = true;  // line-resident 1st-RF sweeps (RGF_B200_RF1LINE=0 at creation: streaming)
  DevBuf<double> rf1_hist;  // [var][segment][2K] boundary states (apply scratch)
  DevBuf<double> rf1_ent;   // [var][segment] entry states of the current pass
  DevBuf<double> ckpt;  // per-block causal checkpoints (apply scratch)
  DevBuf<uint64_t> bits[2];
  DevBuf<uint64_t> bitsT[2];  // chain-minor copies (checkpointed sweeps)
  int64_t words[2] = {0, 0};
  DevBuf<int> cls_d;
  DevBuf<double> clos;  // [class][dir][nh][18]
  std::vector<int64_t> class_g;  // ghost width of each closure class
  // Few-plane x sweeps run as y sweeps on the transposed field (lanes = rows
  // instead of planes): the x tables in the transposed frame, built on first use
  bool xt_ok = false;
  DevBuf<rgfb::Coef3> xt_c3;
  DevBuf<double> xt_c3s, xt_idc, xt_clos;
  DevBuf<uint64_t> xt_bitsT;
  DevBuf<char> xt_in, xt_out;
  // single-level operators: chunked sweeps (sweep_few.cuh), tables per frame
  // (0: x lines through the transposed field, 1: y lines) and part
  bool few_mode = true;  // RGF_B200_FEW=0 at creation turns it off
  bool few_built[2][2] = {{false, false}, {false, false}};
  DevBuf<double> few_tab[2][2], few_chk[2][2], few_cta[2][2], few_scr;
  int few_cs[2] = {0, 0};  // CTAs per column tile, per frame
  DevBuf<double4> entry;  // [var][segments] anti-causal entry states (apply scratch)
  int nclass = 0;
  // host-apply pipeline: H2D / compute / D2H streams, per-slot chunk buffers
  cudaStream_t pipe_stream[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t pipe_ev[3][3] = {};
  cudaEvent_t pipe_ev_user = nullptr;
  DevBuf<char> pin[3], pout[3];
  DevBuf<char> pdin, pdout;  // pitched copies for device applies on unaligned rows
  void pipe_init() {
    if (pipe_stream[0]) return;
    for (auto& s : pipe_stream) CUDA_OK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (auto& row : pipe_ev)
      for (auto& e : row) CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_OK(cudaEventCreateWithFlags(&pipe_ev_user, cudaEventDisableTiming));
  }
  std::mutex mu;  // apply() is const in the reference; serialize buffer reuse
  // Apply scratch (tmp1/tmp2, ckpt, entry, rf1 histories, pitched and pipeline
  // slots) is shared by every apply of this op. The host lock only orders the
  // enqueueing, so each apply's first stream waits on this event and its last
  // stream records it: two applies on different streams (or a device apply
  // followed by a host one) never overlap on the scratch.
  cudaEvent_t scratch_free = nullptr;
  int64_t chunk_mb = 256;  // host-apply pipeline chunk (RGF_B200_CHUNK_MB at creation)

  ~rgf_op() {
    if (own_stream) cudaStreamDestroy(own_stream);
    for (auto s : pipe_stream)
      if (s) cudaStreamDestroy(s);
    for (auto& row : pipe_ev)
      for (auto e : row)
        if (e) cudaEventDestroy(e);
    if (pipe_ev_user) cudaEventDestroy(pipe_ev_user);
    if (scratch_free) cudaEventDestroy(scratch_free);
  }
};

namespace {

// ------------------------------------------------------------- sweeps
// One directional sweep over every (var, level, line): out = G_dir in (or
// its transpose), with optional fused per-point input/output scaling
// (the variance multiplies of apply_v / apply_v_transpose).
// Field row pitch (elements) the checkpointed kernels run on: nx, or nx
// rounded up to a 16 B multiple when the dense rows are not TMA-aligned
// (SURVEY §7 hard part 4: C2 fp64 nx=871, C4 fp32 nx=1442). Other kernels
// always use the dense layout.
template <typename T>
int64_t field_pitch(const rgf_op* op) {
  if (!op->stream_ok || !op->ckpt_ok) return op->nx;
  const int64_t q = 16 / static_cast<int64_t>(sizeof(T));
  return (op->nx + q - 1) / q * q;
}

// out[p][x][y] = in[p][y][x] (in rows `pin` apart, out rows `pout` apart)
template <typename T>
__global__ void k_transpose_planes(const T* __restrict__ in, T* __restrict__ out, int64_t nx,
                                   int64_t ny, int64_t pin, int64_t pout, int64_t planes) {
  __shared__ T tile[32][33];
  const int64_t tx = (nx + 31) / 32, ty = (ny + 31) / 32;
  for (int64_t t = blockIdx.x; t < planes * tx * ty; t += gridDim.x) {
    const int64_t p = t / (tx * ty), r = t - p * tx * ty;
    const int64_t by = r / tx, bx = r - by * tx;
    const T* src = in + p * ny * pin;
    T* dst = out + p * nx * pout;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
      const int64_t y = by * 32 + j, x = bx * 32 + threadIdx.x;
      if (y < ny && x < nx) tile[j][threadIdx.x] = src[y * pin + x];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
      const int64_t x = bx * 32 + j, y = by * 32 + threadIdx.x;
      if (y < ny && x < nx) dst[x * pout + y] = tile[threadIdx.x][j];
    }
    __syncthreads();
  }
}

template <typename T>
void transpose_planes(const T* in, T* out, int64_t nx, int64_t ny, int64_t pin, int64_t pout,
                      int64_t planes, cudaStream_t st) {
  const int64_t tiles = planes * ((nx + 31) / 32) * ((ny + 31) / 32);
  const int blocks = static_cast<int>(std::min<int64_t>(tiles, 148 * 16));
  k_transpose_planes<T><<<blocks, dim3(32, 8), 0, st>>>(in, out, nx, ny, pin, pout, planes);
  CUDA_OK(cudaGetLastError());
}

// x tables in the transposed frame (x runs down the rows of a [nx][ny] field)
void build_xt(rgf_op* op, cudaStream_t st) {
  const int64_t nx = op->nx, ny = op->ny, nh = nx * ny;
  op->xt_c3.alloc(static_cast<size_t>(nh));
  transpose_planes<rgfb::Coef3>(op->dx_.c3.p, op->xt_c3.p, nx, ny, nx, ny, 1, st);
  op->xt_c3s.alloc(static_cast<size_t>(4 * nh));
  rgfb::k_coef_soa<<<grid_for(nh, 256), 256, 0, st>>>(op->xt_c3.p, ny, nx, op->xt_c3s.p);
  CUDA_OK(cudaGetLastError());
  if (op->unit_dc) {  // rows padded to an even count (TMA: 16 B row pitch)
    const int64_t ip = (ny + 1) / 2 * 2;
    op->xt_idc.alloc(static_cast<size_t>(nx * ip));
    transpose_planes<double>(op->dx_.idc.p, op->xt_idc.p, nx, ny, nx, ip, 1, st);
  }
  // x bits [lev][iy][word] -> y-style chain-minor [lev][word][iy]
  const int64_t tot = op->nlev * ny * op->words[0];
  op->xt_bitsT.alloc(static_cast<size_t>(tot));
  rgfb::k_bits_transpose<<<grid_for(tot, 256), 256, 0, st>>>(op->bits[0].p, 1, ny, nx, op->nlev,
                                                             op->words[0], op->xt_bitsT.p);
  CUDA_OK(cudaGetLastError());
  op->xt_clos.alloc(static_cast<size_t>(op->nclass) * 2 * 2 * nh * 10);
  const int threads = 128;
  const int blocks = grid_for(nh, threads, 148 * 8);
  const int64_t slab = op->gmax + 1;
  DevBuf<double> scr;
  scr.alloc(static_cast<size_t>(blocks) * threads * slab);
  for (int c = 0; c < op->nclass; ++c) {
    rgfb::k_closures<<<blocks, threads, 0, st>>>(op->xt_c3.p, nh, static_cast<int>(op->class_g[c]),
                                                 op->xt_clos.p + rgfb::clos_off(c, 1, 0, nh, 0),
                                                 scr.p, slab);
    CUDA_OK(cudaGetLastError());
  }
  CUDA_OK(cudaStreamSynchronize(st));
  op->xt_ok = true;
}

// Frame arguments of the chunked few-plane sweep: frame 1 = y lines of the
// field, frame 0 = x lines as columns of the transposed field (xt tables).
rgfb::FewArgs few_args(const rgf_op* op, int frame, int part) {
  rgfb::FewArgs f{};
  if (frame == 1) {
    f.nx = op->nx;
    f.ny = op->ny;
    f.bits = op->bits[1].p;
    f.words = static_cast<int>(op->words[1]);
    f.c3 = op->dy_.c3.p;
    f.c3s = op->dy_.c3s.p;
    f.idc = op->unit_dc ? op->dy_.idc.p : nullptr;
    f.idc_pitch = op->nx;
    f.clos = op->clos.p;
  } else {
    f.nx = op->ny;
    f.ny = op->nx;
    f.bits = op->bits[0].p;
    f.words = static_cast<int>(op->words[0]);
    f.c3 = op->xt_c3.p;
    f.c3s = op->xt_c3s.p;
    f.idc = op->unit_dc ? op->xt_idc.p : nullptr;
    f.idc_pitch = (op->ny + 1) / 2 * 2;
    f.clos = op->xt_clos.p;
  }
  f.nh = op->nx * op->ny;
  f.part = part;
  f.ghost = op->ghost_d.p;
  f.cls = op->cls_d.p;
  // enough CTAs to cover the SMs: CS CTAs (a cluster, <= 8) per column tile
  if (!op->few_cs[frame]) {
    const int64_t tiles = (f.nx + 31) / 32;
    int cs = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, 148 / tiles)));
    while (cs > 1 && int64_t(cs) * rgfb::few::NW * 4 > f.ny) --cs;  // >= 4 rows per chunk
    const_cast<rgf_op*>(op)->few_cs[frame] = cs;
  }
  f.CS = op->few_cs[frame];
  f.R = static_cast<int>((f.ny + int64_t(f.CS) * rgfb::few::NW - 1) / (int64_t(f.CS) * rgfb::few::NW));
  f.tab = op->few_tab[frame][part].p;
  f.chk = op->few_chk[frame][part].p;
  f.chk_cta = op->few_cta[frame][part].p;
  return f;
}

// Few-plane (single-level operator) sweep in one frame: tables on first use.
template <typename T>
void few_sweep(rgf_op* op, int frame, bool transpose, const T* in, T* out, int64_t pitch,
               int64_t nvar, int64_t lev0, int64_t nlev, const double* pre, const double* post,
               cudaStream_t st) {
  const int part = transpose ? 1 : 0;
  if (!op->few_built[frame][part]) {
    rgfb::FewArgs f = few_args(op, frame, part);
    f.nlev = op->nlev;
    op->few_tab[frame][part].alloc(static_cast<size_t>(op->nlev * f.ny * 6 * f.nx));
    op->few_chk[frame][part].alloc(
        static_cast<size_t>(op->nlev * f.CS * rgfb::few::NW * rgfb::few::CHKW * f.nx));
    op->few_cta[frame][part].alloc(static_cast<size_t>(op->nlev * f.CS * 18 * f.nx));
    f.tab = op->few_tab[frame][part].p;
    f.chk = op->few_chk[frame][part].p;
    f.chk_cta = op->few_cta[frame][part].p;
    const int64_t work = op->nlev * f.nx * f.CS * rgfb::few::NW;
    if (transpose)
      rgfb::k_yfew_tables<true><<<grid_for(work, 128), 128, 0, st>>>(
          f, op->few_tab[frame][part].p, op->few_chk[frame][part].p);
    else
      rgfb::k_yfew_tables<false><<<grid_for(work, 128), 128, 0, st>>>(
          f, op->few_tab[frame][part].p, op->few_chk[frame][part].p);
    rgfb::k_yfew_cta<<<grid_for(op->nlev * f.nx * f.CS, 128), 128, 0, st>>>(
        f, op->few_chk[frame][part].p, op->few_cta[frame][part].p);
    CUDA_OK(cudaGetLastError());
    op->few_built[frame][part] = true;
  }
  rgfb::FewArgs f = few_args(op, frame, part);
  f.pitch = pitch;
  f.planes = nvar * nlev;
  f.nlev = nlev;
  f.lev0 = lev0;
  f.pre_scale = pre;
  f.post_scale = post;
  op->few_scr.alloc(static_cast<size_t>(f.planes * f.ny * f.nx));
  rgfb::launch_yfew<T>(in, out, op->few_scr.p, f, transpose, f.idc != nullptr, pre != nullptr,
                       post != nullptr, st);
  CUDA_OK(cudaGetLastError());
  op->launches += 1;
  RGF_DEBUG_SYNC(st, "few-plane sweep");
}

template <typename T>
void sweep(rgf_op* op, int dir, bool transpose, const T* in, T* out, int64_t nvar,
           int64_t lev0, int64_t nlev, const double* pre, const double* post, cudaStream_t st,
           int64_t pitch) {
  const DirData& d = dir == 0 ? op->dx_ : op->dy_;
  const int64_t lines = nvar * nlev * (dir == 0 ? op->ny : op->nx);

  if (op->stream_ok) {
    rgfb::StreamArgs a{};
    a.dir = dir;
    a.transpose = transpose;
    a.unit_dc = op->unit_dc;
    a.nx = op->nx;
    a.ny = op->ny;
    a.pitch = pitch;
    a.nlev = nlev;
    a.lev0 = lev0;
    a.nvar = nvar;
    a.c3 = d.c3.p;
    a.c3s = d.c3s.p;
    a.idc = op->unit_dc ? d.idc.p : nullptr;
    a.ipitch = (op->nx + 1) / 2 * 2;
    a.idcp = !op->unit_dc ? nullptr : (a.ipitch == op->nx ? d.idc.p : d.idcp.p);
    a.bits = op->bits[dir].p;
    a.bitsT = op->bitsT[dir].p;
    a.nlev_all = op->nlev;
    a.words = op->words[dir];
    a.ghost = op->ghost_d.p;
    a.cls = op->cls_d.p;
    a.nclass = op->nclass;
    a.clos = op->clos.p;
    a.seg_off = d.seg_off.p;
    a.segs = d.segs.p;
    a.seg_line = d.seg_line.p;
    a.close_order = d.close_order.p;
    a.nsegs = d.nsegs;
    op->entry.alloc(static_cast<size_t>(std::max<int64_t>(1, nvar * d.nsegs)));
    a.entry = op->entry.p;
    a.pre_scale = pre;
    a.post_scale = post;
    // few planes: the x sweep's lanes would be planes, mostly idle; run it as
    // a y sweep (lanes = rows) on the transposed field instead, with the
    // few-plane y shapes (launch_yck1 / launch_yck2). Default for <= 2 planes
    // (RGF_B200_XT=0 at creation turns it off); DESIGN §3.9. fp64 only: the
    // transposed sweep then has the x sweep's 16-point blocks, so results are
    // bit-identical to the direct x kernels (host pipeline chunks and level
    // shards of any size agree bit for bit); fp32 x blocks are 32 points.
    // single-level operators (the reference's own 2-D operator): chunked
    // sweeps, x lines through the transposed field
    if (op->few_mode && op->nlev == 1 && op->ckpt_ok) {
      if (dir == 1) {
        few_sweep<T>(op, 1, transpose, in, out, pitch, nvar, lev0, nlev, pre, post, st);
        return;
      }
      if (!op->xt_ok) build_xt(op, st);
      const int64_t q = 16 / static_cast<int64_t>(sizeof(T));
      const int64_t pt = (op->ny + q - 1) / q * q, planes = nvar * nlev;
      op->xt_in.alloc(static_cast<size_t>(planes * op->nx * pt) * sizeof(T));
      op->xt_out.alloc(static_cast<size_t>(planes * op->nx * pt) * sizeof(T));
      T* ti = reinterpret_cast<T*>(op->xt_in.p);
      T* to = reinterpret_cast<T*>(op->xt_out.p);
      transpose_planes<T>(in, ti, op->nx, op->ny, pitch, pt, planes, st);
      // the variance multiplies (pre/post) are [lev][iy][ix]: x sweeps never
      // carry them (V: post on y, V^T: pre on y)
      few_sweep<T>(op, 0, transpose, ti, to, pt, nvar, lev0, nlev, nullptr, nullptr, st);
      transpose_planes<T>(to, out, op->ny, op->nx, pt, pitch, planes, st);
      op->launches += 2;
      return;
    }
    if (op->xt_mode && sizeof(T) == 8 && dir == 0 && op->ckpt_ok && nvar * nlev <= 2 && !pre &&
        !post &&
        rgfb::tma_supported(in, out, pitch)) {
      if (!op->xt_ok) build_xt(op, st);
      // transposed rows (length ny) padded to a 16 B pitch for the TMA maps
      const int64_t q = 16 / static_cast<int64_t>(sizeof(T));
      const int64_t pt = (op->ny + q - 1) / q * q, planes = nvar * nlev;
      op->xt_in.alloc(static_cast<size_t>(planes * op->nx * pt) * sizeof(T));
      op->xt_out.alloc(static_cast<size_t>(planes * op->nx * pt) * sizeof(T));
      T* ti = reinterpret_cast<T*>(op->xt_in.p);
      T* to = reinterpret_cast<T*>(op->xt_out.p);
      transpose_planes<T>(in, ti, op->nx, op->ny, pitch, pt, planes, st);
      RGF_DEBUG_SYNC(st, "xt transpose in");
      rgfb::StreamArgs b = a;
      b.dir = 1;
      b.nx = op->ny;
      b.ny = op->nx;
      b.pitch = pt;
      b.c3 = op->xt_c3.p;
      b.c3s = op->xt_c3s.p;
      b.idc = op->unit_dc ? op->xt_idc.p : nullptr;
      b.idcp = b.idc;
      b.ipitch = (op->ny + 1) / 2 * 2;
      b.bitsT = op->xt_bitsT.p;
      b.words = op->words[0];
      b.clos = op->xt_clos.p;
      op->ckpt.alloc(static_cast<size_t>(std::max<int64_t>(1, rgfb::ckpt_doubles<T>(b))));
      op->launches +=
          static_cast<unsigned long long>(rgfb::launch_ckpt_sweep<T>(ti, to, b, op->ckpt.p, st));
      RGF_DEBUG_SYNC(st, "xt ckpt sweep");
      CUDA_OK(cudaGetLastError());
      transpose_planes<T>(to, out, op->ny, op->nx, pt, pitch, planes, st);
      RGF_DEBUG_SYNC(st, "xt transpose out");
      op->launches += 2;
      return;
    }
    if (op->ckpt_ok && rgfb::tma_supported(in, out, pitch)) {
      op->ckpt.alloc(static_cast<size_t>(std::max<int64_t>(1, rgfb::ckpt_doubles<T>(a))));
      op->launches +=
          static_cast<unsigned long long>(rgfb::launch_ckpt_sweep<T>(in, out, a, op->ckpt.p, st));
      CUDA_OK(cudaGetLastError());
      RGF_DEBUG_SYNC(st, dir == 0 ? "x ckpt sweep" : "y ckpt sweep");
      return;
    }
    if (pitch != op->nx) throw std::runtime_error("sweep: pitched field on a dense-only path");
    op->launches += static_cast<unsigned long long>(rgfb::launch_stream_sweep<T>(in, out, a, st));
    CUDA_OK(cudaGetLastError());
    return;
  }
  if (pitch != op->nx) throw std::runtime_error("sweep: pitched field on a dense-only path");
  if (op->rf1_ok) {
    rgfb::Rf1Args a{};
    a.dir = dir;
    a.transpose = transpose;
    a.k = op->k;
    a.nx = op->nx;
    a.ny = op->ny;
    a.nlev = nlev;
    a.nvar = nvar;
    a.lev0 = lev0;
    a.c1 = d.c1.p;
    a.bits = op->bits[dir].p;
    a.bitsT = op->bitsT[dir].p;
    a.nlev_all = op->nlev;
    a.seg_off = d.seg_off.p;
    a.segs = d.segs.p;
    a.nsegs = d.nsegs;
    {  // this launch's level range as a segment range (host copy of seg_off)
      const int64_t nl = dir == 0 ? op->ny : op->nx;
      a.seg_begin = d.seg_off_h[static_cast<size_t>(lev0 * nl)];
      a.seg_end = d.seg_off_h[static_cast<size_t>((lev0 + nlev) * nl)];
    }
    a.zone = d.zone[transpose ? 1 : 0].p;
    if (op->rf1_line) {  // all K iterations with the line resident: one field pass
      rgfb::Rf1LineArgs b{};
      b.dir = dir;
      b.transpose = transpose;
      b.k = op->k;
      b.nx = op->nx;
      b.ny = op->ny;
      b.nlev = nlev;
      b.nvar = nvar;
      b.lev0 = lev0;
      b.c1 = d.c1.p;
      b.bits = op->bits[dir].p;
      b.words = op->words[dir];
      b.seg_off = d.seg_off.p;
      b.segs = d.segs.p;
      b.nsegs = d.nsegs;
      b.zone = a.zone;
      b.ghost = op->ghost_d.p;
      b.same = op->mask_same.p;
      b.pre_scale = pre;
      b.post_scale = post;
      b.segcap = std::max(1, d.segcap);
      if (rgfb::launch_rf1_line<T>(in, out, b, st)) {
        op->launches += 1;
        CUDA_OK(cudaGetLastError());
        RGF_DEBUG_SYNC(st, "rf1 line sweep");
        return;
      }
    }
    if (op->rf1_stream) {
      op->rf1_hist.alloc(static_cast<size_t>(std::max<int64_t>(1, nvar * d.nsegs * 2 * op->k)));
      a.hist = op->rf1_hist.p;
      op->rf1_ent.alloc(static_cast<size_t>(std::max<int64_t>(1, nvar * d.nsegs)));
      a.ent = op->rf1_ent.p;
      a.pre_scale = pre;
      a.post_scale = post;
      op->launches += static_cast<unsigned long long>(rgfb::launch_rf1_sweep<T>(in, out, a, st));
      CUDA_OK(cudaGetLastError());
      RGF_DEBUG_SYNC(st, "rf1 sweep");
      return;
    }
  }

  const int64_t n = dir == 0 ? op->nx : op->ny;
  const int64_t slab = n + 2 * op->gmax + 4;
  const int threads = 128;
  int64_t want = std::min<int64_t>(lines, 148 * 4 * threads);
  if (op->scratch_threads < want || op->scratch_slab < slab) {
    op->scratch_threads = std::max(op->scratch_threads, want);
    op->scratch_slab = std::max(op->scratch_slab, slab);
    op->scratch.alloc(static_cast<size_t>(op->scratch_threads * op->scratch_slab));
  }
  rgfb::SweepArgs a{};
  a.dir = dir;
  a.transpose = transpose;
  a.order = op->order;
  a.k = op->k;
  a.unit_dc = op->unit_dc;
  a.nx = op->nx;
  a.ny = op->ny;
  a.nlev = nlev;
  a.lev0 = lev0;
  a.nvar = nvar;
  a.c3 = d.c3.p;
  a.c1 = d.c1.p;
  a.idc = d.idc.p;
  a.seg_off = d.seg_off.p;
  a.segs = d.segs.p;
  a.ghost = op->ghost_d.p;
  a.pre_scale = pre;
  a.post_scale = post;
  a.scratch = op->scratch.p;
  a.slab = op->scratch_slab;
  const int blocks = static_cast<int>((want + threads - 1) / threads);
  rgfb::k_sweep_generic<T><<<blocks, threads, 0, st>>>(in, out, a);
  CUDA_OK(cudaGetLastError());
  op->launches += 1;
}

template <typename T>
void apply_typed(rgf_op* op, int kind, const T* in, T* out, int64_t nvar, int64_t lev0,
                 int64_t nlev, cudaStream_t st, int64_t pitch) {
  const size_t count = static_cast<size_t>(nvar * nlev * pitch * op->ny);
  const double* var = op->has_variance ? op->variance.p : nullptr;
  auto tmp = [&](DevBuf<char>& b) {
    b.alloc(count * sizeof(T));
    return reinterpret_cast<T*>(b.p);
  };
  auto sw = [&](int dir, bool tr, const T* i, T* o, const double* pre, const double* post) {
    sweep<T>(op, dir, tr, i, o, nvar, lev0, nlev, pre, post, st, pitch);
  };
  switch (kind) {
    case RGF_GX: sw(0, false, in, out, nullptr, nullptr); break;
    case RGF_GY: sw(1, false, in, out, nullptr, nullptr); break;
    case RGF_GXT: sw(0, true, in, out, nullptr, nullptr); break;
    case RGF_GYT: sw(1, true, in, out, nullptr, nullptr); break;
    case RGF_GYGX: {
      T* t = tmp(op->tmp1);
      sw(0, false, in, t, nullptr, nullptr);
      sw(1, false, t, out, nullptr, nullptr);
      break;
    }
    case RGF_V: {  // covariance.cpp:382-387: diag(var) G_y G_x
      T* t = tmp(op->tmp1);
      sw(0, false, in, t, nullptr, nullptr);
      sw(1, false, t, out, nullptr, var);
      break;
    }
    case RGF_VT: {  // covariance.cpp:389-394: G_x^T G_y^T diag(var)
      T* t = tmp(op->tmp1);
      sw(1, true, in, t, var, nullptr);
      sw(0, true, t, out, nullptr, nullptr);
      break;
    }
    case RGF_B: {  // covariance.cpp:396-398: V V^T
      T* t = tmp(op->tmp1);
      T* u = tmp(op->tmp2);
      sw(1, true, in, t, var, nullptr);
      sw(0, true, t, u, nullptr, nullptr);
      sw(0, false, u, t, nullptr, nullptr);
      sw(1, false, t, out, nullptr, var);
      break;
    }
    default: throw InvalidArgument("apply: unknown operator kind");
  }
}

// Host-memory apply as a level-chunked pipeline: chunk c's H2D copy, its
// sweeps and its D2H copy run on three streams, so PCIe traffic in both
// directions overlaps the kernels of neighbouring chunks (levels are
// independent 2-D problems). Pinned host buffers give full overlap; pageable
// ones still work (the copies then serialise through staging).
template <typename T>
void apply_host_pipelined(rgf_op* op, int kind, const T* hin, T* hout, int64_t nvar,
                          cudaStream_t user) {
  const int64_t nh = op->nx * op->ny;
  const int64_t nlev = op->nlev;
  // ~256 MB per chunk, >= 1 level; at least 4 chunks per variable when possible
  const int64_t per_level = nh * static_cast<int64_t>(sizeof(T));
  const int64_t chunk_mb = op->chunk_mb;
  int64_t cl = std::max<int64_t>(1, (chunk_mb << 20) / per_level);
  cl = std::min(cl, std::max<int64_t>(1, (nlev + 3) / 4));
  // The x kernels give each lane a plane and walk a whole row per CTA, so a
  // sweep over a few planes costs nearly as much as over 128. The 3rd-RF's
  // four kernels per chunk hide under the PCIe copies; the 1st-RF's 2K passes
  // per sweep do not, so its chunks hold at least 32 levels.
  if (op->order == 1) cl = std::max<int64_t>(cl, 32);
  cl = std::min(cl, nlev);
  constexpr int kSlots = 3;
  op->pipe_init();
  // device slots use the kernels' row pitch; 2-D copies repack on the fly
  const int64_t pitch = field_pitch<T>(op);
  const size_t esz = sizeof(T);
  const size_t slot_bytes = static_cast<size_t>(cl * op->ny * pitch) * esz;
  for (int sl = 0; sl < kSlots; ++sl) {
    op->pin[sl].alloc(slot_bytes);
    op->pout[sl].alloc(slot_bytes);
  }
  cudaStream_t h2d = op->pipe_stream[0], cs = op->pipe_stream[1], d2h = op->pipe_stream[2];
  // order after the caller's prior work on its stream
  CUDA_OK(cudaEventRecord(op->pipe_ev_user, user));
  CUDA_OK(cudaStreamWaitEvent(h2d, op->pipe_ev_user, 0));
  CUDA_OK(cudaStreamWaitEvent(cs, op->pipe_ev_user, 0));
  // and after every earlier apply of this op (shared scratch), on any stream
  CUDA_OK(cudaStreamWaitEvent(h2d, op->scratch_free, 0));
  CUDA_OK(cudaStreamWaitEvent(cs, op->scratch_free, 0));
  int64_t c = 0;
  for (int64_t v = 0; v < nvar; ++v)
    for (int64_t l0 = 0; l0 < nlev; l0 += cl, ++c) {
      const int64_t nl = std::min(cl, nlev - l0);
      const int sl = static_cast<int>(c % kSlots);
      const size_t off = static_cast<size_t>((v * nlev + l0) * nh);
      const size_t rows = static_cast<size_t>(nl * op->ny);
      T* din = reinterpret_cast<T*>(op->pin[sl].p);
      T* dout = reinterpret_cast<T*>(op->pout[sl].p);
      cudaEvent_t* ev = op->pipe_ev[sl];  // 0: loaded, 1: computed, 2: drained
      // slot reuse: din is free once the chunk kSlots back was computed,
      // dout once it was drained
      if (c >= kSlots) CUDA_OK(cudaStreamWaitEvent(h2d, ev[1], 0));
      CUDA_OK(cudaMemcpy2DAsync(din, pitch * esz, hin + off, op->nx * esz, op->nx * esz, rows,
                                cudaMemcpyHostToDevice, h2d));
      CUDA_OK(cudaEventRecord(ev[0], h2d));
      CUDA_OK(cudaStreamWaitEvent(cs, ev[0], 0));
      if (c >= kSlots) CUDA_OK(cudaStreamWaitEvent(cs, ev[2], 0));
      apply_typed<T>(op, kind, din, dout, 1, l0, nl, cs, pitch);
      CUDA_OK(cudaEventRecord(ev[1], cs));
      CUDA_OK(cudaStreamWaitEvent(d2h, ev[1], 0));
      CUDA_OK(cudaMemcpy2DAsync(hout + off, op->nx * esz, dout, pitch * esz, op->nx * esz, rows,
                                cudaMemcpyDeviceToHost, d2h));
      CUDA_OK(cudaEventRecord(ev[2], d2h));
    }
  CUDA_OK(cudaEventRecord(op->scratch_free, d2h));  // d2h waited on every compute chunk
  CUDA_OK(cudaStreamSynchronize(d2h));
}

// Device-memory apply. Dense rows that are not 16 B aligned go through
// internal pitched buffers (one 2-D copy each way) so the checkpointed TMA
// kernels still run.
template <typename T>
void apply_device(rgf_op* op, int kind, const T* in, T* out, int64_t nvar, cudaStream_t st) {
  const int64_t pitch = field_pitch<T>(op);
  if (pitch == op->nx) {
    apply_typed<T>(op, kind, in, out, nvar, 0, op->nlev, st, pitch);
    return;
  }
  const size_t esz = sizeof(T);
  const size_t rows = static_cast<size_t>(nvar * op->nlev * op->ny);
  op->pdin.alloc(rows * pitch * esz);
  op->pdout.alloc(rows * pitch * esz);
  T* din = reinterpret_cast<T*>(op->pdin.p);
  T* dout = reinterpret_cast<T*>(op->pdout.p);
  CUDA_OK(cudaMemcpy2DAsync(din, pitch * esz, in, op->nx * esz, op->nx * esz, rows,
                            cudaMemcpyDeviceToDevice, st));
  apply_typed<T>(op, kind, din, dout, nvar, 0, op->nlev, st, pitch);
  CUDA_OK(cudaMemcpy2DAsync(out, op->nx * esz, dout, pitch * esz, op->nx * esz, rows,
                            cudaMemcpyDeviceToDevice, st));
}

unsigned long long read_u64(const unsigned long long* d) {
  unsigned long long h = 0;
  CUDA_OK(cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost));
  return h;
}

void build_segments(rgf_op* op, const uint8_t* mask_d, int dir, DirData& d) {
  const int64_t lines = op->nlev * (dir == 0 ? op->ny : op->nx);
  DevBuf<int64_t> counts;
  counts.alloc(lines);
  d.seg_off.alloc(lines + 1);
  rgfb::k_seg_count<<<grid_for(lines, 128), 128>>>(mask_d, dir, op->nx, op->ny, lines,
                                                   counts.p);
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaMemset(d.seg_off.p, 0, sizeof(int64_t)));
  size_t tmp_bytes = 0;
  CUDA_OK(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, counts.p, d.seg_off.p + 1, lines));
  DevBuf<char> tmp;
  tmp.alloc(tmp_bytes);
  CUDA_OK(cub::DeviceScan::InclusiveSum(tmp.p, tmp_bytes, counts.p, d.seg_off.p + 1, lines));
  d.seg_off_h.resize(static_cast<size_t>(lines + 1));
  CUDA_OK(cudaMemcpy(d.seg_off_h.data(), d.seg_off.p, (lines + 1) * sizeof(int64_t),
                     cudaMemcpyDeviceToHost));
  const int64_t total = d.seg_off_h[static_cast<size_t>(lines)];
  d.nsegs = total;
  d.segs.alloc(std::max<int64_t>(total, 1));
  d.seg_line.alloc(std::max<int64_t>(total, 1));
  rgfb::k_seg_fill<<<grid_for(lines, 128), 128>>>(mask_d, dir, op->nx, op->ny, lines,
                                                  d.seg_off.p, d.segs.p, d.seg_line.p);
  CUDA_OK(cudaGetLastError());
  if (total > 0) {  // closure-pass order: (line, end, level)
    const int64_t nl = dir == 0 ? op->ny : op->nx;
    const int64_t n = dir == 0 ? op->nx : op->ny;
    DevBuf<uint64_t> keys, keys2;
    DevBuf<int64_t> idx;
    keys.alloc(total);
    keys2.alloc(total);
    idx.alloc(total);
    d.close_order.alloc(total);
    rgfb::k_seg_keys<<<grid_for(total, 256), 256>>>(d.segs.p, d.seg_line.p, total, nl, n,
                                                    op->nlev, keys.p, idx.p);
    CUDA_OK(cudaGetLastError());
    size_t sb = 0;
    CUDA_OK(cub::DeviceRadixSort::SortPairs(nullptr, sb, keys.p, keys2.p, idx.p, d.close_order.p,
                                            total));
    DevBuf<char> st;
    st.alloc(sb);
    CUDA_OK(cub::DeviceRadixSort::SortPairs(st.p, sb, keys.p, keys2.p, idx.p, d.close_order.p,
                                            total));
  }
  CUDA_OK(cudaDeviceSynchronize());
}

}  // namespace

// ---------------------------------------------------------- observations + CG
// the observation operator (obs.cpp) and the
// control-variable CG analysis (solver.cpp) kept on the device. Stencils are
// validated and built on the host with the reference's formulas; the
// per-iteration work (V, V^T sweeps, H, H^T, dots, updates) runs on the GPU.
struct rgf_obs {
  int device = 0;
  int64_t n = 0, nx = 0, ny = 0;
  std::mutex mu;
  std::vector<double> values_h, rvar_h;
  DevBuf<int64_t> cell;
  DevBuf<double4> w;
  DevBuf<double> values, rvar;
  // H^T gather lists: touched cells, CSR offsets, (obs*4 + corner) entries
  int64_t ncell = 0;
  DevBuf<int64_t> tcells, tptr;
  DevBuf<int32_t> tent;
  DevBuf<char> arena;  // one allocation and one upload for all of the above
};

namespace {

int blocks_for(int64_t n) { return grid_for(std::max<int64_t>(n, 1), 256, 148 * 8); }

// obs.cpp:18-44 (mask: level 0 of the grid, host)
void obs_stencil(const rgf_grid_desc* g, double x, double y, int64_t row, int64_t& i0, int64_t& j0,
                 double4& w) {
  const auto fail = [row](const std::string& why) {
    throw InvalidArgument("observation " + std::to_string(row) + ": " + why);
  };
  if (!std::isfinite(x) || !std::isfinite(y) || x < 0 || y < 0 || x > double(g->nx - 1) ||
      y > double(g->ny - 1))
    fail("position (" + std::to_string(x) + "," + std::to_string(y) + ") is outside the grid");
  i0 = std::min<int64_t>(static_cast<int64_t>(std::floor(x)), g->nx - 2);
  j0 = std::min<int64_t>(static_cast<int64_t>(std::floor(y)), g->ny - 2);
  const double fx = x - double(i0), fy = y - double(j0);
  w = make_double4((1 - fx) * (1 - fy), fx * (1 - fy), (1 - fx) * fy, fx * fy);
  const auto sea = [&](int64_t i, int64_t j) { return g->mask[j * g->nx + i] != 0; };
  if (!(sea(i0, j0) || sea(i0 + 1, j0) || sea(i0, j0 + 1) || sea(i0 + 1, j0 + 1)))
    fail("all four stencil corners are land");
}

struct Cg {
  rgf_op* op;
  rgf_obs* o;
  cudaStream_t st;
  int64_t nh;
  DevBuf<double> partial, scal, tmp_obs, tmp_obs2, tmp_f;
  void init() {
    const size_t nobs = static_cast<size_t>(std::max<int64_t>(o->n, 1));
    if (op) {  // the operator keeps these between calls (no cudaMalloc/cudaFree per solve)
      op->cg_aux.alloc(rgfb::kDotBlocks + 1 + 2 * nobs + static_cast<size_t>(nh));
      double* q = op->cg_aux.p;
      partial.borrow(q, rgfb::kDotBlocks);
      scal.borrow(q + rgfb::kDotBlocks, 1);
      tmp_obs.borrow(q + rgfb::kDotBlocks + 1, nobs);
      tmp_obs2.borrow(q + rgfb::kDotBlocks + 1 + nobs, nobs);
      tmp_f.borrow(q + rgfb::kDotBlocks + 1 + 2 * nobs, static_cast<size_t>(nh));
      return;
    }
    partial.alloc(rgfb::kDotBlocks);
    scal.alloc(1);
    tmp_obs.alloc(nobs);
    tmp_obs2.alloc(nobs);
    tmp_f.alloc(nh);
  }
  // a.b, or sum a^2 / r (r != nullptr)
  double dot(const double* a, const double* b, int64_t n, const double* r = nullptr) {
    rgfb::k_dot1<<<rgfb::kDotBlocks, rgfb::kDotThreads, 0, st>>>(a, b, r, n, partial.p);
    rgfb::k_dot2<<<1, rgfb::kDotThreads, 0, st>>>(partial.p, rgfb::kDotBlocks, scal.p);
    CUDA_OK(cudaGetLastError());
    double h = 0.0;
    CUDA_OK(cudaMemcpyAsync(&h, scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    if (op) op->launches += 2;
    return h;
  }
  void h(const double* f, double* out) {
    if (o->n == 0) return;
    rgfb::k_obs_h<<<blocks_for(o->n), 256, 0, st>>>(f, o->n, o->nx, o->cell.p, o->w.p, out);
    CUDA_OK(cudaGetLastError());
    if (op) op->launches += 1;
  }
  void ht(const double* v, const double* rvar, double* out) {
    CUDA_OK(cudaMemsetAsync(out, 0, static_cast<size_t>(nh) * sizeof(double), st));
    if (o->ncell == 0) return;
    rgfb::k_obs_ht<<<blocks_for(o->ncell), 256, 0, st>>>(
        v, rvar, o->ncell, o->tcells.p, o->tptr.p, o->tent.p,
        reinterpret_cast<const double*>(o->w.p), out);
    CUDA_OK(cudaGetLastError());
    if (op) op->launches += 1;
  }
  void v(const double* in, double* out) { apply_device<double>(op, RGF_V, in, out, 1, st); }
  // solver.cpp:26-31: V^T H^T (v ./ r_var)
  void adjoint_rhs(const double* vobs, double* out) {
    ht(vobs, o->rvar.p, tmp_f.p);
    apply_device<double>(op, RGF_VT, tmp_f.p, out, 1, st);
  }
  // solver.cpp:18-22: d = y (no background) or y - H x_b
  void misfit(const double* bg_dev, double* d) {
    if (o->n == 0) return;
    if (!bg_dev) {
      CUDA_OK(cudaMemcpyAsync(d, o->values.p, o->n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      return;
    }
    h(bg_dev, tmp_obs2.p);
    rgfb::k_obs_residual<<<blocks_for(o->n), 256, 0, st>>>(o->values.p, tmp_obs2.p, o->n, d);
    CUDA_OK(cudaGetLastError());
    op->launches += 1;
  }
};

void check_cg_op(const rgf_op* op, const rgf_obs* o) {
  if (op->nlev != 1) throw InvalidArgument("solve: the operator must have one level");
  if (o->nx != op->nx || o->ny != op->ny || o->device != op->device)
    throw InvalidArgument("solve: observations are not on the operator's grid");
}
void validate_rvar(const rgf_obs* o) {  // obs.cpp:48-57 (positions checked at creation)
  for (int64_t k = 0; k < o->n; ++k)
    if (!(o->rvar_h[static_cast<size_t>(k)] > 0))
      throw InvalidArgument("observation " + std::to_string(k) +
                            ": error variance must be positive");
}

}  // namespace

namespace {

__global__ void k_f64_to_f32(const double* in, float* out, int64_t n) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    out[p] = static_cast<float>(in[p]);
}
__global__ void k_f32_to_f64(const float* in, double* out, int64_t n) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    out[p] = static_cast<double>(in[p]);
}

// two pinned host slots + events for the streamed field loads/saves
struct PinnedPair {
  static constexpr size_t kChunk = size_t(32) << 20;  // bytes per slot
  void* h[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  bool used[2] = {false, false};
  PinnedPair() {
    for (int b = 0; b < 2; ++b) {
      CUDA_OK(cudaMallocHost(&h[b], kChunk));
      CUDA_OK(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
    }
  }
  ~PinnedPair() {
    for (int b = 0; b < 2; ++b) {
      if (ev[b]) cudaEventSynchronize(ev[b]);
      if (h[b]) cudaFreeHost(h[b]);
      if (ev[b]) cudaEventDestroy(ev[b]);
    }
  }
  void acquire(int b) {  // slot b's previous copy has finished
    if (used[b]) CUDA_OK(cudaEventSynchronize(ev[b]));
    used[b] = true;
  }
};

void check_dims(int64_t nx, int64_t ny, int64_t nlev) {
  if (nx < 1 || ny < 1 || nlev < 1) throw InvalidArgument("container: bad dimensions");
}

}  // namespace

extern "C" {

const char* rgf_last_error(void) { return g_last_error.c_str(); }

// --------------------------------------------------------- diagnostics
// diagnostics.cpp:69-96 impulse_response, batched over n studies (host arrays)
int rgf_impulse_responses(const double* sigma, int64_t n, int order, int k, int64_t length,
                          int calibration, double* h, double* sum_h, double* err_h_l2,
                          double* err_h_max) {
  return guarded([&] {
    if (length < 4) throw InvalidArgument("impulse_response: length must be >= 4");
    if (n < 1) throw InvalidArgument("impulse_response: no studies");
    if (!sigma || !h || !sum_h || !err_h_l2 || !err_h_max)
      throw InvalidArgument("impulse_response: null argument");
    for (int64_t s = 0; s < n; ++s)
      if (!(sigma[s] > 0)) throw InvalidArgument("impulse_response: sigma must be positive");
    if (order != RGF_ORDER_FIRST && order != RGF_ORDER_THIRD)
      throw InvalidArgument("covariance: order must be 1 or 3");
    if (order == RGF_ORDER_THIRD && k != 1)
      throw InvalidArgument("the third-order filter is single-iteration by construction");
    if (order == RGF_ORDER_FIRST && k < 1) throw InvalidArgument("rf1_coefficients: k must be >= 1");
    DevBuf<double> sg, dh, o3;
    sg.upload(sigma, static_cast<size_t>(n));
    dh.alloc(static_cast<size_t>(n * length));
    o3.alloc(static_cast<size_t>(3 * n));
    rgfb::k_impulse<<<grid_for(n, 64), 64>>>(sg.p, n, order, k, length, calibration, dh.p, o3.p,
                                             o3.p + n, o3.p + 2 * n);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaMemcpy(h, dh.p, static_cast<size_t>(n * length) * 8, cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(sum_h, o3.p, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(err_h_l2, o3.p + n, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(err_h_max, o3.p + 2 * n, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
  });
}

// diagnostics.cpp:102-135 remark1_bound_check, batched: s0 is n x m, one
// sigma per study; out4[s] = {lhs, rhs, err_h_l2, holds}
int rgf_remark1_checks(const double* s0, const double* sigma, int64_t n, int64_t m, int order,
                       int k, int calibration, double* out4) {
  return guarded([&] {
    if (m < 4) throw InvalidArgument("remark1_bound_check: input too short");
    if (n < 1 || !s0 || !sigma || !out4) throw InvalidArgument("remark1_bound_check: null argument");
    for (int64_t p = 0; p < n * m; ++p)
      if (!std::isfinite(s0[p])) throw InvalidArgument("remark1_bound_check: input must be finite");
    for (int64_t s = 0; s < n; ++s)
      if (!(sigma[s] > 0)) throw InvalidArgument("remark1_bound_check: sigma must be positive");
    if (order == RGF_ORDER_THIRD && k != 1)
      throw InvalidArgument("the third-order filter is single-iteration by construction");
    DevBuf<double> x, sg, scr, o;
    x.upload(s0, static_cast<size_t>(n * m));
    sg.upload(sigma, static_cast<size_t>(n));
    scr.alloc(static_cast<size_t>(3 * n * m));
    o.alloc(static_cast<size_t>(4 * n));
    rgfb::k_remark1<<<grid_for(n, 64), 64>>>(x.p, sg.p, n, m, order, k, calibration, scr.p, o.p);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaMemcpy(out4, o.p, static_cast<size_t>(4 * n) * 8, cudaMemcpyDeviceToHost));
  });
}

// --------------------------------------------------------- container I/O
int rgf_container_info(const char* path, char* format, int64_t* nx, int64_t* ny,
                       int64_t* ghost_width, int64_t* nlev) {
  return guarded([&] {
    if (!path) throw InvalidArgument("container: null path");
    rgfio::File in(path, "rb");
    std::string line;
    int c;
    while ((c = std::fgetc(in.f)) != EOF && c != '\n') line.push_back(static_cast<char>(c));
    if (line.empty()) throw std::runtime_error("missing container header");
    const rgfio::Header h = rgfio::parse_header(line);
    const auto f = h.scalars.find("format");
    if (format) {
      const std::string fs = f == h.scalars.end() ? "" : f->second;
      std::snprintf(format, 32, "%s", fs.c_str());
    }
    if (nx) *nx = rgfio::get_int(h, "nx", -1);
    if (ny) *ny = rgfio::get_int(h, "ny", -1);
    if (ghost_width) *ghost_width = rgfio::get_int(h, "ghost_width", 0);
    if (nlev) *nlev = rgfio::get_int(h, "nlev", 1);
  });
}

// io.cpp:133-181 load_grid (binary containers) + grid.cpp:27-39 validate
int rgf_grid_load(const char* path, int64_t nx, int64_t ny, double* dx, double* dy,
                  uint8_t* mask, int64_t* ghost_width) {
  return guarded([&] {
    if (!path || !dx || !dy || !mask) throw InvalidArgument("load_grid: null argument");
    check_dims(nx, ny, 1);
    rgfio::File in(path, "rb");
    const rgfio::Header h = rgfio::read_header(in, "rgf-grid");
    if (rgfio::get_int(h, "nx", -1) != nx || rgfio::get_int(h, "ny", -1) != ny)
      throw InvalidArgument("load_grid: buffers do not match the container's nx/ny");
    const int64_t g = rgfio::get_int(h, "ghost_width", 0);
    const size_t n = static_cast<size_t>(nx * ny);
    bool has_dx = false, has_dy = false, has_mask = false;
    std::vector<uint8_t> raw;
    for (const std::string& sec : h.sections) {
      if (sec == "dx") {
        rgfio::read_exact(in, dx, n * 8, "payload section \"dx\" is truncated (dimension mismatch?)");
        has_dx = true;
      } else if (sec == "dy") {
        rgfio::read_exact(in, dy, n * 8, "payload section \"dy\" is truncated (dimension mismatch?)");
        has_dy = true;
      } else if (sec == "mask") {
        raw.resize(n);
        rgfio::read_exact(in, raw.data(), n, "mask section is truncated");
        for (size_t p = 0; p < n; ++p) mask[p] = raw[p] != 0 ? 1 : 0;
        has_mask = true;
      } else {
        throw std::runtime_error("unknown grid section \"" + sec + "\"");
      }
    }
    if (!has_dx || !has_dy) throw std::runtime_error("grid container is missing dx/dy sections");
    if (!has_mask) std::memset(mask, 1, n);
    rgfio::expect_eof(in, "trailing bytes after grid payload");
    if (nx < 4 || ny < 4) throw InvalidArgument("Grid2D: nx and ny must both be >= 4");
    for (size_t p = 0; p < n; ++p)
      if (!(dx[p] > 0) || !(dy[p] > 0))
        throw InvalidArgument("Grid2D: grid spacing must be strictly positive");
    if (g < 0) throw InvalidArgument("Grid2D: ghost_width must be >= 0");
    if (ghost_width) *ghost_width = g;
  });
}

// io.cpp:183-202 save_grid (level 0 of the mask)
int rgf_grid_save(const char* path, const rgf_grid_desc* g) {
  return guarded([&] {
    if (!path || !g || !g->dx || !g->dy || !g->mask) throw InvalidArgument("save_grid: null argument");
    check_dims(g->nx, g->ny, 1);
    const size_t n = static_cast<size_t>(g->nx * g->ny);
    rgfio::File out(path, "wb");
    const int64_t gw = g->ghost_width;
    const std::string hd = rgfio::dump_header("rgf-grid", g->nx, g->ny, &gw, 1, {"dx", "dy", "mask"});
    rgfio::write_exact(out, hd.data(), hd.size());
    rgfio::write_exact(out, g->dx, n * 8);
    rgfio::write_exact(out, g->dy, n * 8);
    std::vector<uint8_t> raw(n);
    for (size_t p = 0; p < n; ++p) raw[p] = g->mask[p] ? 1 : 0;
    rgfio::write_exact(out, raw.data(), n);
  });
}

// io.cpp:204-235 load_scale_field (binary) + grid.cpp:40-55 validate
int rgf_scale_load(const char* path, const rgf_grid_desc* g, double* rx, double* ry) {
  return guarded([&] {
    if (!path || !g || !rx || !ry || !g->dx || !g->dy || !g->mask)
      throw InvalidArgument("load_scale_field: null argument");
    check_dims(g->nx, g->ny, 1);
    rgfio::File in(path, "rb");
    const rgfio::Header h = rgfio::read_header(in, "rgf-scale");
    if (rgfio::get_int(h, "nx", -1) != g->nx || rgfio::get_int(h, "ny", -1) != g->ny)
      throw std::runtime_error("scale file dimensions do not match the grid");
    const size_t n = static_cast<size_t>(g->nx * g->ny);
    bool has_rx = false, has_ry = false;
    for (const std::string& sec : h.sections) {
      if (sec == "rx") {
        rgfio::read_exact(in, rx, n * 8, "payload section \"rx\" is truncated (dimension mismatch?)");
        has_rx = true;
      } else if (sec == "ry") {
        rgfio::read_exact(in, ry, n * 8, "payload section \"ry\" is truncated (dimension mismatch?)");
        has_ry = true;
      } else {
        throw std::runtime_error("unknown scale section \"" + sec + "\"");
      }
    }
    if (!has_rx) throw std::runtime_error("scale file is missing the zonal (rx) component");
    if (!has_ry) throw std::runtime_error("scale file is missing the meridional (ry) component");
    for (int64_t j = 0; j < g->ny; ++j)
      for (int64_t i = 0; i < g->nx; ++i) {
        const size_t p = static_cast<size_t>(j * g->nx + i);
        if (!g->mask[p]) continue;
        const double sx = rx[p] / g->dx[p], sy = ry[p] / g->dy[p];
        if (!(rx[p] > 0) || !(ry[p] > 0) || !std::isfinite(sx) || !std::isfinite(sy))
          throw InvalidArgument("ScaleField: non-positive or non-finite radius at sea point (" +
                                std::to_string(i) + "," + std::to_string(j) + ")");
      }
  });
}

// io.cpp:237-249 save_scale_field
int rgf_scale_save(const char* path, int64_t nx, int64_t ny, const double* rx, const double* ry) {
  return guarded([&] {
    if (!path || !rx || !ry) throw InvalidArgument("save_scale_field: null argument");
    check_dims(nx, ny, 1);
    const size_t n = static_cast<size_t>(nx * ny);
    rgfio::File out(path, "wb");
    const std::string hd = rgfio::dump_header("rgf-scale", nx, ny, nullptr, 1, {"rx", "ry"});
    rgfio::write_exact(out, hd.data(), hd.size());
    rgfio::write_exact(out, rx, n * 8);
    rgfio::write_exact(out, ry, n * 8);
  });
}

// io.cpp:251-269 load_state_field, streamed into host or device memory
int rgf_field_load(const char* path, int64_t nx, int64_t ny, int64_t nlev, int dtype, void* dst,
                   int memory, void* stream) {
  return guarded([&] {
    if (!path || !dst) throw InvalidArgument("load_state_field: null argument");
    if (dtype != RGF_F64 && dtype != RGF_F32) throw InvalidArgument("load_state_field: unknown dtype");
    if (memory != RGF_HOST && memory != RGF_DEVICE)
      throw InvalidArgument("load_state_field: unknown memory kind");
    check_dims(nx, ny, nlev);
    rgfio::File in(path, "rb");
    const rgfio::Header h = rgfio::read_header(in, "rgf-field");
    if (rgfio::get_int(h, "nx", -1) != nx || rgfio::get_int(h, "ny", -1) != ny)
      throw std::runtime_error("field file dimensions do not match the grid");
    if (rgfio::get_int(h, "nlev", 1) != nlev)
      throw std::runtime_error("field file level count does not match");
    const std::string trunc = "payload section \"values\" is truncated (dimension mismatch?)";
    const size_t total = static_cast<size_t>(nx * ny * nlev);
    if (memory == RGF_HOST) {
      if (dtype == RGF_F64) {
        rgfio::read_exact(in, dst, total * 8, trunc);
      } else {
        std::vector<double> buf(std::min<size_t>(total, size_t(1) << 20));
        float* d = static_cast<float*>(dst);
        for (size_t off = 0; off < total; off += buf.size()) {
          const size_t n = std::min(buf.size(), total - off);
          rgfio::read_exact(in, buf.data(), n * 8, trunc);
          for (size_t p = 0; p < n; ++p) d[off + p] = static_cast<float>(buf[p]);
        }
      }
      return;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PinnedPair pp;
    const size_t per = PinnedPair::kChunk / 8;  // doubles per slot
    DevBuf<double> stage;
    if (dtype == RGF_F32) stage.alloc(std::min(per, total));
    int b = 0;
    for (size_t off = 0; off < total; off += per, b ^= 1) {
      const size_t n = std::min(per, total - off);
      pp.acquire(b);  // the copy out of slot b two chunks ago is done
      rgfio::read_exact(in, pp.h[b], n * 8, trunc);  // overlaps the previous slot's H2D
      if (dtype == RGF_F64) {
        CUDA_OK(cudaMemcpyAsync(static_cast<double*>(dst) + off, pp.h[b], n * 8,
                                cudaMemcpyHostToDevice, st));
      } else {
        CUDA_OK(cudaMemcpyAsync(stage.p, pp.h[b], n * 8, cudaMemcpyHostToDevice, st));
        k_f64_to_f32<<<grid_for(static_cast<int64_t>(n), 256), 256, 0, st>>>(
            stage.p, static_cast<float*>(dst) + off, static_cast<int64_t>(n));
        CUDA_OK(cudaGetLastError());
      }
      CUDA_OK(cudaEventRecord(pp.ev[b], st));
    }
    CUDA_OK(cudaStreamSynchronize(st));
  });
}

// io.cpp:271-281 save_state_field, streamed out of host or device memory
int rgf_field_save(const char* path, int64_t nx, int64_t ny, int64_t nlev, int dtype,
                   const void* src, int memory, void* stream) {
  return guarded([&] {
    if (!path || !src) throw InvalidArgument("save_state_field: null argument");
    if (dtype != RGF_F64 && dtype != RGF_F32) throw InvalidArgument("save_state_field: unknown dtype");
    if (memory != RGF_HOST && memory != RGF_DEVICE)
      throw InvalidArgument("save_state_field: unknown memory kind");
    check_dims(nx, ny, nlev);
    const size_t total = static_cast<size_t>(nx * ny * nlev);
    rgfio::File out(path, "wb");
    const std::string hd = rgfio::dump_header("rgf-field", nx, ny, nullptr, nlev, {"values"});
    rgfio::write_exact(out, hd.data(), hd.size());
    if (memory == RGF_HOST) {
      if (dtype == RGF_F64) {
        rgfio::write_exact(out, src, total * 8);
      } else {
        std::vector<double> buf(std::min<size_t>(total, size_t(1) << 20));
        const float* s = static_cast<const float*>(src);
        for (size_t off = 0; off < total; off += buf.size()) {
          const size_t n = std::min(buf.size(), total - off);
          for (size_t p = 0; p < n; ++p) buf[p] = static_cast<double>(s[off + p]);
          rgfio::write_exact(out, buf.data(), n * 8);
        }
      }
      return;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    PinnedPair pp;
    const size_t per = PinnedPair::kChunk / 8;
    DevBuf<double> stage;
    if (dtype == RGF_F32) stage.alloc(std::min(per, total));
    auto issue = [&](size_t off, int b) {  // D2H of the chunk at `off` into slot b
      const size_t n = std::min(per, total - off);
      if (dtype == RGF_F64) {
        CUDA_OK(cudaMemcpyAsync(pp.h[b], static_cast<const double*>(src) + off, n * 8,
                                cudaMemcpyDeviceToHost, st));
      } else {
        k_f32_to_f64<<<grid_for(static_cast<int64_t>(n), 256), 256, 0, st>>>(
            static_cast<const float*>(src) + off, stage.p, static_cast<int64_t>(n));
        CUDA_OK(cudaGetLastError());
        CUDA_OK(cudaMemcpyAsync(pp.h[b], stage.p, n * 8, cudaMemcpyDeviceToHost, st));
      }
      CUDA_OK(cudaEventRecord(pp.ev[b], st));
      pp.used[b] = true;
    };
    if (total > 0) issue(0, 0);
    int b = 0;
    for (size_t off = 0; off < total; off += per, b ^= 1) {
      if (off + per < total) issue(off + per, b ^ 1);  // next chunk's D2H overlaps this write
      CUDA_OK(cudaEventSynchronize(pp.ev[b]));
      rgfio::write_exact(out, pp.h[b], std::min(per, total - off) * 8);
    }
  });
}

#ifdef RGF_RING_PROF
// development build only: per-section cycle totals of the ring sweeps
int rgf_debug_ring_prof(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, rgfb::g_ring_prof, 8 * sizeof(unsigned long long)) != cudaSuccess) return 1;
  if (reset) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (cudaMemcpyToSymbol(rgfb::g_ring_prof, z, sizeof(z)) != cudaSuccess) return 1;
  }
  return 0;
}
#endif

void rgf_options_default(rgf_options* o) {
  o->order = RGF_ORDER_THIRD;
  o->k_iterations = 1;
  o->unit_dc = 1;
  o->calibration = RGF_CAL_YVV95;
  o->ghost_width = -1;
  o->variance = nullptr;
  o->threads = 0;
  o->device = 0;
}

int rgf_op_create(const rgf_grid_desc* g, const double* rx, const double* ry,
                  const rgf_options* opt, rgf_op** out) {
  if (out) *out = nullptr;
  return guarded([&] {
    if (!g || !rx || !ry || !opt || !out) throw InvalidArgument("rgf_op_create: null argument");
    // grid.cpp:27-39 Grid2D::validate
    if (g->nx < 4 || g->ny < 4) throw InvalidArgument("Grid2D: nx and ny must both be >= 4");
    if (g->nlev < 1) throw InvalidArgument("Grid2D: nlev must be >= 1");
    if (!g->dx || !g->dy || !g->mask) throw InvalidArgument("Grid2D: spacing field shape mismatch");
    if (g->ghost_width < 0) throw InvalidArgument("Grid2D: ghost_width must be >= 0");
    // covariance.cpp:159-166 option checks (after the grid/scale checks below
    // in the reference; both orders raise invalid_argument)
    if (opt->order != RGF_ORDER_FIRST && opt->order != RGF_ORDER_THIRD)
      throw InvalidArgument("covariance: order must be 1 or 3");

    auto op = std::make_unique<rgf_op>();
    op->device = opt->device;
    CUDA_OK(cudaSetDevice(op->device));
    op->nx = g->nx;
    op->ny = g->ny;
    op->nlev = g->nlev;
    const int64_t nh = g->nx * g->ny;

    DevBuf<double> dx, dy, rxd, ryd;
    DevBuf<uint8_t> mask, any_sea;
    DevBuf<unsigned long long> flag;
    dx.upload(g->dx, nh);
    dy.upload(g->dy, nh);
    rxd.upload(rx, nh);
    ryd.upload(ry, nh);
    mask.upload(g->mask, static_cast<size_t>(nh * g->nlev));
    op->mask0.assign(g->mask, g->mask + nh);
    any_sea.alloc(nh);
    flag.alloc(1);

    // grid.cpp:33-34
    CUDA_OK(cudaMemset(flag.p, 0xff, sizeof(unsigned long long)));
    rgfb::k_check_spacing<<<grid_for(nh, 256), 256>>>(dx.p, dy.p, nh, flag.p);
    CUDA_OK(cudaGetLastError());
    if (read_u64(flag.p) != ~0ull)
      throw InvalidArgument("Grid2D: grid spacing must be strictly positive");
    // grid.cpp:41-55
    CUDA_OK(cudaMemset(flag.p, 0xff, sizeof(unsigned long long)));
    rgfb::k_check_scales<<<grid_for(nh, 256), 256>>>(rxd.p, ryd.p, dx.p, dy.p, mask.p, nh,
                                                     g->nlev, flag.p, any_sea.p);
    CUDA_OK(cudaGetLastError());
    const unsigned long long bad = read_u64(flag.p);
    if (bad != ~0ull) {
      const int64_t p = static_cast<int64_t>(bad % nh);
      throw InvalidArgument("ScaleField: non-positive or non-finite radius at sea point (" +
                            std::to_string(p % g->nx) + "," + std::to_string(p / g->nx) + ")");
    }
    // covariance.cpp:159-166
    if (opt->order == RGF_ORDER_FIRST && opt->k_iterations < 1)
      throw InvalidArgument("covariance: k_iterations must be >= 1");
    if (opt->order == RGF_ORDER_THIRD && opt->k_iterations != 1)
      throw InvalidArgument("covariance: the third-order filter is single-iteration by construction");
    if (opt->calibration < 0 || opt->calibration > 2)
      throw InvalidArgument("covariance: unknown calibration");
    op->order = opt->order;
    op->k = opt->k_iterations;
    op->unit_dc = opt->unit_dc ? 1 : 0;
    op->calibration = opt->calibration;

    // per-level sigma statistics: uniform test and max sigma
    DevBuf<unsigned long long> stats;
    stats.alloc(4 * g->nlev);
    std::vector<unsigned long long> init(4 * g->nlev);
    for (int64_t l = 0; l < g->nlev; ++l) {
      init[4 * l + 0] = ~0ull;
      init[4 * l + 1] = 0;
      init[4 * l + 2] = ~0ull;
      init[4 * l + 3] = 0;
    }
    CUDA_OK(cudaMemcpy(stats.p, init.data(), init.size() * 8, cudaMemcpyHostToDevice));
    {
      dim3 grid(grid_for(nh, 256, 256), static_cast<unsigned>(g->nlev));
      rgfb::k_level_stats<<<grid, 256>>>(rxd.p, ryd.p, dx.p, dy.p, mask.p, nh, stats.p);
      CUDA_OK(cudaGetLastError());
    }
    std::vector<unsigned long long> st(4 * g->nlev);
    CUDA_OK(cudaMemcpy(st.data(), stats.p, st.size() * 8, cudaMemcpyDeviceToHost));
    auto as_d = [](unsigned long long b) {
      double v;
      std::memcpy(&v, &b, 8);
      return v;
    };
    op->ghost.resize(g->nlev);
    op->dx_.uniform.resize(g->nlev);
    op->dy_.uniform.resize(g->nlev);
    op->dx_.sigma_u.resize(g->nlev);
    op->dy_.sigma_u.resize(g->nlev);
    for (int64_t l = 0; l < g->nlev; ++l) {
      const double mnx = as_d(st[4 * l]), mxx = as_d(st[4 * l + 1]);
      const double mny = as_d(st[4 * l + 2]), mxy = as_d(st[4 * l + 3]);
      op->dx_.uniform[l] = mnx == mxx;
      op->dy_.uniform[l] = mny == mxy;
      op->dx_.sigma_u[l] = mnx;
      op->dy_.sigma_u[l] = mny;
      // covariance.cpp:173-180 ghost width resolution
      if (opt->ghost_width >= 0) {
        op->ghost[l] = opt->ghost_width;
      } else if (g->ghost_width > 0) {
        op->ghost[l] = g->ghost_width;
      } else {
        op->ghost[l] = static_cast<int64_t>(std::ceil(9.0 * std::max(mxx, mxy)));
      }
    }
    op->gmax = *std::max_element(op->ghost.begin(), op->ghost.end());
    std::vector<int> gi(op->ghost.begin(), op->ghost.end());
    op->ghost_d.upload(gi.data(), gi.size());

    // coefficient precompute (covariance.cpp:182-219)
    for (int dir = 0; dir < 2; ++dir) {
      DirData& d = dir == 0 ? op->dx_ : op->dy_;
      const double* r = dir == 0 ? rxd.p : ryd.p;
      const double* s = dir == 0 ? dx.p : dy.p;
      if (op->order == 3) {
        d.c3.alloc(nh);
        if (op->unit_dc) d.idc.alloc(nh);
      } else {
        d.c1.alloc(nh);
      }
      const int threads = 128;
      rgfb::k_coefficients<<<grid_for(nh, threads, 148 * 64), threads>>>(
          r, s, any_sea.p, nh, op->order, op->k, op->calibration, op->unit_dc, d.c3.p, d.c1.p,
          d.idc.p);
      CUDA_OK(cudaGetLastError());
      build_segments(op.get(), mask.p, dir, d);
    }
    // Streaming 3rd-RF path (sweep_stream.cuh). Needs every level's ghost
    // width >= 3 (then no segment can fall under the pass-through length,
    // covariance.cpp:260-269) and is skipped when RGF_B200_EXACT=1 selects
    // the bit-exact segment-serial kernel.
    {
      const char* ex = std::getenv("RGF_B200_EXACT");
      const bool exact = ex && ex[0] == '1';
      const int64_t gmin = *std::min_element(op->ghost.begin(), op->ghost.end());
      if (op->order == 3 && !exact && gmin >= 3) {
        std::vector<int64_t> classes;
        std::vector<int> cls(g->nlev);
        for (int64_t l = 0; l < g->nlev; ++l) {
          auto it = std::find(classes.begin(), classes.end(), op->ghost[l]);
          if (it == classes.end()) {
            classes.push_back(op->ghost[l]);
            it = classes.end() - 1;
          }
          cls[l] = static_cast<int>(it - classes.begin());
        }
        op->nclass = static_cast<int>(classes.size());
        op->class_g = classes;
        op->cls_d.upload(cls.data(), cls.size());
        op->clos.alloc(static_cast<size_t>(op->nclass) * 2 * 2 * nh * 10);
        const int threads = 128;
        const int blocks = grid_for(nh, threads, 148 * 8);
        const int64_t slab = op->gmax + 1;
        DevBuf<double> scr;
        scr.alloc(static_cast<size_t>(blocks) * threads * slab);
        for (int c = 0; c < op->nclass; ++c)
          for (int dir = 0; dir < 2; ++dir) {
            const DirData& d = dir == 0 ? op->dx_ : op->dy_;
            rgfb::k_closures<<<blocks, threads>>>(d.c3.p, nh, static_cast<int>(classes[c]),
                                                  op->clos.p + rgfb::clos_off(c, dir, 0, nh, 0),
                                                  scr.p, slab);
            CUDA_OK(cudaGetLastError());
          }
        for (int dir = 0; dir < 2; ++dir) {
          const int64_t n = dir == 0 ? g->nx : g->ny;
          const int64_t nl = dir == 0 ? g->ny : g->nx;
          op->words[dir] = (n + 63) / 64;
          const int64_t tot = g->nlev * nl * op->words[dir];
          op->bits[dir].alloc(tot);
          rgfb::k_pack_bits<<<grid_for(tot, 256), 256>>>(mask.p, dir, g->nx, g->ny, g->nlev,
                                                         op->words[dir], op->bits[dir].p);
          CUDA_OK(cudaGetLastError());
        }
        CUDA_OK(cudaDeviceSynchronize());
        op->stream_ok = true;
        if (const char* fe = std::getenv("RGF_B200_FEW")) op->few_mode = fe[0] != '0';
        const char* xte = std::getenv("RGF_B200_XT");
        op->xt_mode = !(xte && xte[0] == '0');
        if (op->ckpt_ok) {
          for (int dir = 0; dir < 2; ++dir) {
            const int64_t tot = g->nlev * (dir == 0 ? g->ny : g->nx) * op->words[dir];
            op->bitsT[dir].alloc(tot);
            rgfb::k_bits_transpose<<<grid_for(tot, 256), 256>>>(
                op->bits[dir].p, dir, g->nx, g->ny, g->nlev, op->words[dir], op->bitsT[dir].p);
            CUDA_OK(cudaGetLastError());
          }
          if (op->unit_dc && (g->nx & 1)) {  // even-pitch inv_dc copies for the TMA maps
            const int64_t ip = g->nx + 1;
            for (DirData* dd : {&op->dx_, &op->dy_}) {
              dd->idcp.alloc(static_cast<size_t>(ip * g->ny));
              CUDA_OK(cudaMemcpy2D(dd->idcp.p, ip * 8, dd->idc.p, g->nx * 8, g->nx * 8, g->ny,
                                   cudaMemcpyDeviceToDevice));
            }
          }
          op->dy_.c3s.alloc(static_cast<size_t>(4 * nh));
          rgfb::k_coef_soa<<<grid_for(nh, 256), 256>>>(op->dy_.c3.p, g->nx, g->ny, op->dy_.c3s.p);
          CUDA_OK(cudaGetLastError());
        }
      }
    }
    if (op->order == 1 && g->nx > 1 && g->ny > 1) {
      const char* ex = std::getenv("RGF_B200_EXACT");
      if (!(ex && ex[0] == '1')) {
        // streaming 1st-RF: level-major mask bits + per-segment ghost-zone
        // responses (forward and adjoint dynamics)
        for (int dir = 0; dir < 2; ++dir) {
          const int64_t n = dir == 0 ? g->nx : g->ny;
          const int64_t nl = dir == 0 ? g->ny : g->nx;
          op->words[dir] = (n + 63) / 64;
          const int64_t tot = g->nlev * nl * op->words[dir];
          op->bits[dir].alloc(tot);
          rgfb::k_pack_bits<<<grid_for(tot, 256), 256>>>(mask.p, dir, g->nx, g->ny, g->nlev,
                                                         op->words[dir], op->bits[dir].p);
          CUDA_OK(cudaGetLastError());
          op->bitsT[dir].alloc(tot);  // chain-minor words for the TMA x pass
          rgfb::k_bits_transpose<<<grid_for(tot, 256), 256>>>(
              op->bits[dir].p, dir, g->nx, g->ny, g->nlev, op->words[dir], op->bitsT[dir].p);
          CUDA_OK(cudaGetLastError());
        }
        const int threads = 128, blocks = 148 * 4;
        const int64_t slab = std::max<int64_t>(1, op->gmax);
        DevBuf<double> scr;
        scr.alloc(static_cast<size_t>(threads) * blocks * 2 * slab);
        for (int dir = 0; dir < 2; ++dir) {
          DirData& d = dir == 0 ? op->dx_ : op->dy_;
          for (int tr = 0; tr < 2; ++tr) {
            d.zone[tr].alloc(static_cast<size_t>(std::max<int64_t>(1, d.nsegs) * 2 * op->k));
            if (d.nsegs > 0)
              rgfb::k_rf1_zones<<<blocks, threads>>>(d.segs.p, d.seg_line.p, d.nsegs, dir, g->nx,
                                                     g->ny, d.c1.p, op->ghost_d.p, op->k, tr == 1,
                                                     d.zone[tr].p, scr.p, slab);
            CUDA_OK(cudaGetLastError());
          }
        }
        CUDA_OK(cudaDeviceSynchronize());
        op->rf1_ok = true;
        if (const char* le = std::getenv("RGF_B200_RF1LINE")) op->rf1_line = le[0] != '0';
        // the streaming passes assume ghost zones on every side that meets
        // land; without ghosts (ghost_width = 0) lines that do not fit the
        // resident kernel take the segment-serial kernel
        op->rf1_stream = *std::min_element(op->ghost.begin(), op->ghost.end()) > 0;
        {
          std::vector<uint8_t> same(static_cast<size_t>(g->nlev), 1);
          same[0] = 0;
          op->mask_same.upload(same.data(), same.size());
          if (g->nlev > 1) {
            rgfb::k_mask_same<<<grid_for(nh * (g->nlev - 1), 256, 148 * 32), 256>>>(
                mask.p, nh, g->nlev, op->mask_same.p);
            CUDA_OK(cudaGetLastError());
            CUDA_OK(cudaMemcpy(same.data(), op->mask_same.p, same.size(), cudaMemcpyDeviceToHost));
            for (int64_t l = 1; l < g->nlev; ++l)
              if (op->ghost[l] != op->ghost[l - 1]) same[static_cast<size_t>(l)] = 0;
            op->mask_same.upload(same.data(), same.size());
          }
        }
        for (int dir = 0; dir < 2; ++dir) {
          DirData& d = dir == 0 ? op->dx_ : op->dy_;
          int64_t cap = 0;
          for (size_t i = 0; i + 1 < d.seg_off_h.size(); ++i)
            cap = std::max(cap, d.seg_off_h[i + 1] - d.seg_off_h[i]);
          d.segcap = static_cast<int>(cap);
        }
      }
    }
    if (opt->variance) {
      op->variance.upload(opt->variance, static_cast<size_t>(nh * g->nlev));
      op->has_variance = true;
    }
    CUDA_OK(cudaStreamCreateWithFlags(&op->own_stream, cudaStreamNonBlocking));
    CUDA_OK(cudaEventCreateWithFlags(&op->scratch_free, cudaEventDisableTiming));
    if (const char* e = std::getenv("RGF_B200_CHUNK_MB"))
      op->chunk_mb = std::max<int64_t>(1, std::atol(e));
    CUDA_OK(cudaDeviceSynchronize());
    *out = op.release();
  });
}

int rgf_op_destroy(rgf_op* op) {
  return guarded([&] {
    if (!op) return;
    cudaSetDevice(op->device);
    delete op;
  });
}

int rgf_op_apply(rgf_op* op, int kind, int dtype, const void* in, void* out, int64_t nvar,
                 int memory, void* stream) {
  return guarded([&] {
    if (!op) throw InvalidArgument("apply: null operator");
    if (!in || !out) throw InvalidArgument("apply: null field");
    if (nvar < 1) throw InvalidArgument("apply: nvar must be >= 1");
    if (dtype != RGF_F64 && dtype != RGF_F32) throw InvalidArgument("apply: unknown dtype");
    if (kind < RGF_GX || kind > RGF_GYGX) throw InvalidArgument("apply: unknown operator kind");
    std::lock_guard<std::mutex> lock(op->mu);
    CUDA_OK(cudaSetDevice(op->device));
    // NULL = the legacy default stream (torch's default stream hands us 0)
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (memory == RGF_HOST) {
      if (dtype == RGF_F64)
        apply_host_pipelined<double>(op, kind, static_cast<const double*>(in),
                                     static_cast<double*>(out), nvar, st);
      else
        apply_host_pipelined<float>(op, kind, static_cast<const float*>(in),
                                    static_cast<float*>(out), nvar, st);
      return;
    }
    if (memory != RGF_DEVICE) throw InvalidArgument("apply: unknown memory kind");
    CUDA_OK(cudaStreamWaitEvent(st, op->scratch_free, 0));
    if (dtype == RGF_F64)
      apply_device<double>(op, kind, static_cast<const double*>(in), static_cast<double*>(out),
                           nvar, st);
    else
      apply_device<float>(op, kind, static_cast<const float*>(in), static_cast<float*>(out), nvar,
                          st);
    CUDA_OK(cudaEventRecord(op->scratch_free, st));
  });
}

int rgf_op_ghost_width(const rgf_op* op, int64_t level, int64_t* out) {
  return guarded([&] {
    if (!op || !out) throw InvalidArgument("ghost_width: null argument");
    if (level < 0 || level >= op->nlev) throw InvalidArgument("ghost_width: level out of range");
    *out = op->ghost[level];
  });
}

int rgf_op_coefficient_bytes(const rgf_op* op, uint64_t* out) {
  return guarded([&] {
    if (!op || !out) throw InvalidArgument("coefficient_bytes: null argument");
    const uint64_t per_point = op->order == RGF_ORDER_FIRST ? 2 : 4;
    *out = 2 * per_point * sizeof(double) * static_cast<uint64_t>(op->nx * op->ny);
  });
}

int rgf_op_device_bytes(const rgf_op* op, uint64_t* out) {
  return guarded([&] {
    if (!op || !out) throw InvalidArgument("device_bytes: null argument");
    uint64_t b = op->ghost_d.bytes() + op->variance.bytes() + op->in_d.bytes() +
                 op->pin[0].bytes() + op->pin[1].bytes() + op->pin[2].bytes() +
                 op->pdin.bytes() + op->pdout.bytes() +
                 op->pout[0].bytes() + op->pout[1].bytes() + op->pout[2].bytes() +
                 op->bits[0].bytes() + op->bits[1].bytes() + op->bitsT[0].bytes() +
                 op->bitsT[1].bytes() + op->clos.bytes() + op->cls_d.bytes() + op->entry.bytes() +
                 op->out_d.bytes() + op->tmp1.bytes() + op->tmp2.bytes() + op->scratch.bytes();
    for (const DirData* d : {&op->dx_, &op->dy_})
      b += d->c3.bytes() + d->c3s.bytes() + d->idcp.bytes() + d->zone[0].bytes() +
           d->zone[1].bytes() + d->c1.bytes() + d->idc.bytes() + d->seg_off.bytes() + d->segs.bytes() +
           d->seg_line.bytes() + d->close_order.bytes();
    *out = b;
  });
}

int rgf_op_launch_count(const rgf_op* op, uint64_t* out) {
  return guarded([&] {
    if (!op || !out) throw InvalidArgument("launch_count: null argument");
    *out = op->launches;
  });
}

int rgf_op_segments(const rgf_op* op, int dir, int64_t* nlines, int64_t* nsegs,
                    int64_t* offsets, int32_t* segs) {
  return guarded([&] {
    if (!op) throw InvalidArgument("segments: null operator");
    if (dir != 0 && dir != 1) throw InvalidArgument("segments: dir must be 0 or 1");
    CUDA_OK(cudaSetDevice(op->device));
    const DirData& d = dir == 0 ? op->dx_ : op->dy_;
    const int64_t lines = op->nlev * (dir == 0 ? op->ny : op->nx);
    if (nlines) *nlines = lines;
    if (nsegs) *nsegs = d.nsegs;
    if (offsets)
      CUDA_OK(cudaMemcpy(offsets, d.seg_off.p, (lines + 1) * sizeof(int64_t),
                         cudaMemcpyDeviceToHost));
    if (segs && d.nsegs)
      CUDA_OK(cudaMemcpy(segs, d.segs.p, d.nsegs * sizeof(int2), cudaMemcpyDeviceToHost));
  });
}

int rgf_op_coefficients(const rgf_op* op, int dir, double* alpha1, double* alpha2,
                        double* alpha3, double* beta, double* inv_dc) {
  return guarded([&] {
    if (!op) throw InvalidArgument("coefficients: null operator");
    CUDA_OK(cudaSetDevice(op->device));
    const DirData& d = dir == 0 ? op->dx_ : op->dy_;
    const int64_t nh = op->nx * op->ny;
    if (op->order == 3) {
      std::vector<rgfb::Coef3> h(nh);
      CUDA_OK(cudaMemcpy(h.data(), d.c3.p, nh * sizeof(rgfb::Coef3), cudaMemcpyDeviceToHost));
      for (int64_t p = 0; p < nh; ++p) {
        if (alpha1) alpha1[p] = h[p].a1;
        if (alpha2) alpha2[p] = h[p].a2;
        if (alpha3) alpha3[p] = h[p].a3;
        if (beta) beta[p] = h[p].b;
      }
      if (inv_dc && op->unit_dc)
        CUDA_OK(cudaMemcpy(inv_dc, d.idc.p, nh * sizeof(double), cudaMemcpyDeviceToHost));
    } else {
      std::vector<double2> h(nh);
      CUDA_OK(cudaMemcpy(h.data(), d.c1.p, nh * sizeof(double2), cudaMemcpyDeviceToHost));
      for (int64_t p = 0; p < nh; ++p) {
        if (alpha1) alpha1[p] = h[p].x;
        if (beta) beta[p] = h[p].y;
      }
    }
  });
}

static void scalar_coefficients(double sigma, int calibration, int k, double* out15) {
  DevBuf<double> d;
  d.alloc(15);
  CUDA_OK(cudaMemset(d.p, 0, 15 * sizeof(double)));
  rgfb::k_scalar_coefficients<<<1, 32>>>(sigma, calibration, k, d.p);
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaMemcpy(out15, d.p, 15 * sizeof(double), cudaMemcpyDeviceToHost));
}

int rgf_rf3_coefficients(double sigma, double out[8]) {
  return guarded([&] {
    if (!(sigma > 0)) throw InvalidArgument("rf3_coefficients: sigma must be positive");
    double r[15];
    scalar_coefficients(sigma, RGF_CAL_YVV95, 0, r);
    std::memcpy(out, r, 8 * sizeof(double));
  });
}

int rgf_rf3_filter_scalars(double sigma, int calibration, double out[5]) {
  return guarded([&] {
    if (!(sigma > 0)) throw InvalidArgument("rf3_filter_scalars: sigma must be positive");
    if (calibration < 0 || calibration > 2) throw InvalidArgument("unknown calibration");
    double r[15];
    scalar_coefficients(sigma, calibration, 0, r);
    std::memcpy(out, r + 8, 5 * sizeof(double));
  });
}

int rgf_rf1_coefficients(double sigma, int k, double out[2]) {
  return guarded([&] {
    if (!(sigma > 0)) throw InvalidArgument("rf1_coefficients: sigma must be positive");
    if (k < 1) throw InvalidArgument("rf1_coefficients: k must be >= 1");
    double r[15];
    scalar_coefficients(sigma, RGF_CAL_YVV95, k, r);
    out[0] = r[13];
    out[1] = r[14];
  });
}

static void apply_1d(const double* in, const double* sigma, int64_t m, int64_t nlines,
                     int order, int k, int calibration, int transpose, double* out) {
  DevBuf<double> sig, din, dout, scr;
  DevBuf<rgfb::Coef3> c3;
  DevBuf<double2> c1;
  sig.upload(sigma, m);
  din.upload(in, static_cast<size_t>(m * nlines));
  dout.alloc(static_cast<size_t>(m * nlines));
  scr.alloc(static_cast<size_t>(m * nlines));
  if (order == 3)
    c3.alloc(m);
  else
    c1.alloc(m);
  rgfb::k_coefficients_1d<<<grid_for(m, 128), 128>>>(sig.p, m, order, k, calibration, c3.p,
                                                    c1.p);
  CUDA_OK(cudaGetLastError());
  rgfb::k_apply_1d<<<grid_for(nlines, 64, 1 << 20), 64>>>(din.p, dout.p, c3.p, c1.p, m, nlines,
                                                          order, k, transpose, scr.p);
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaMemcpy(out, dout.p, static_cast<size_t>(m * nlines) * sizeof(double),
                     cudaMemcpyDeviceToHost));
}

static double scalar_helper(double x, int calibration, int mode) {
  DevBuf<double> d;
  d.alloc(1);
  rgfb::k_scalar_helper<<<1, 32>>>(x, calibration, mode, d.p);
  CUDA_OK(cudaGetLastError());
  double h = 0.0;
  CUDA_OK(cudaMemcpy(&h, d.p, sizeof(double), cudaMemcpyDeviceToHost));
  return h;
}

int rgf_rf3_cascade_variance(double q, double* out) {
  return guarded([&] {
    if (!out) throw InvalidArgument("rf3_cascade_variance: null argument");
    *out = scalar_helper(q, RGF_CAL_YVV95, 0);
  });
}

int rgf_rf3_length_scale_argument(double sigma, int calibration, double* out) {
  return guarded([&] {
    if (!out) throw InvalidArgument("rf3_length_scale_argument: null argument");
    if (calibration < 0 || calibration > 2) throw InvalidArgument("unknown calibration");
    *out = scalar_helper(sigma, calibration, 1);
  });
}

// rf3.hpp:191-210 / rf1.hpp:96-110: per-point tables on the device
static void tables_1d(const double* sigma, int64_t m, int order, int k, int calibration,
                      double* a1, double* a2, double* a3, double* b) {
  DevBuf<double> sig, t1, t2, t3, t4;
  DevBuf<rgfb::Coef3> c3;
  DevBuf<double2> c1;
  sig.upload(sigma, static_cast<size_t>(m));
  if (order == 3)
    c3.alloc(static_cast<size_t>(m));
  else
    c1.alloc(static_cast<size_t>(m));
  for (DevBuf<double>* t : {&t1, &t2, &t3, &t4}) t->alloc(static_cast<size_t>(m));
  rgfb::k_coefficients_1d<<<grid_for(m, 128), 128>>>(sig.p, m, order, k, calibration, c3.p, c1.p);
  rgfb::k_unpack_tables_1d<<<grid_for(m, 128), 128>>>(c3.p, c1.p, m, t1.p, t2.p, t3.p, t4.p);
  CUDA_OK(cudaGetLastError());
  const size_t bytes = static_cast<size_t>(m) * sizeof(double);
  CUDA_OK(cudaMemcpy(a1, t1.p, bytes, cudaMemcpyDeviceToHost));
  if (order == 3) {
    CUDA_OK(cudaMemcpy(a2, t2.p, bytes, cudaMemcpyDeviceToHost));
    CUDA_OK(cudaMemcpy(a3, t3.p, bytes, cudaMemcpyDeviceToHost));
  }
  CUDA_OK(cudaMemcpy(b, t4.p, bytes, cudaMemcpyDeviceToHost));
}

int rgf_rf3_filter_coefficients(const double* sigma, int64_t m, int calibration, double* alpha1,
                                double* alpha2, double* alpha3, double* beta) {
  return guarded([&] {
    if (m < 0) throw InvalidArgument("rf3_filter_coefficients: negative length");
    if (m > 0 && (!sigma || !alpha1 || !alpha2 || !alpha3 || !beta))
      throw InvalidArgument("rf3_filter_coefficients: null argument");
    if (calibration < 0 || calibration > 2) throw InvalidArgument("unknown calibration");
    for (int64_t i = 0; i < m; ++i)  // rf3.hpp:170 (rf3_filter_scalars)
      if (!(sigma[i] > 0)) throw InvalidArgument("rf3_filter_scalars: sigma must be positive");
    if (m > 0) tables_1d(sigma, m, 3, 1, calibration, alpha1, alpha2, alpha3, beta);
  });
}

int rgf_rf1_coefficients_table(const double* sigma, int64_t m, int k, double* alpha,
                               double* beta) {
  return guarded([&] {
    if (m < 0) throw InvalidArgument("rf1_coefficients: negative length");
    if (m > 0 && (!sigma || !alpha || !beta))
      throw InvalidArgument("rf1_coefficients: null argument");
    for (int64_t i = 0; i < m; ++i)  // rf1.hpp:79-80
      if (!(sigma[i] > 0)) throw InvalidArgument("rf1_coefficients: sigma must be positive");
    if (k < 1) throw InvalidArgument("rf1_coefficients: k must be >= 1");
    if (m > 0) tables_1d(sigma, m, 1, k, RGF_CAL_YVV95, alpha, nullptr, nullptr, beta);
  });
}

// rf3.hpp:292-334 / rf1.hpp:113-155 with caller tables, one thread per vector
static void filter_tables_1d(const double* in, const double* a1, const double* a2,
                             const double* a3, const double* b, int64_t m, int64_t nlines,
                             int order, int k, int transpose, double* out) {
  DevBuf<double> t1, t2, t3, t4, din, dout, scr;
  DevBuf<rgfb::Coef3> c3;
  DevBuf<double2> c1;
  t1.upload(a1, static_cast<size_t>(m));
  t4.upload(b, static_cast<size_t>(m));
  if (order == 3) {
    t2.upload(a2, static_cast<size_t>(m));
    t3.upload(a3, static_cast<size_t>(m));
    c3.alloc(static_cast<size_t>(m));
  } else {
    c1.alloc(static_cast<size_t>(m));
  }
  din.upload(in, static_cast<size_t>(m * nlines));
  dout.alloc(static_cast<size_t>(m * nlines));
  scr.alloc(static_cast<size_t>(m * nlines));
  rgfb::k_pack_tables_1d<<<grid_for(m, 128), 128>>>(t1.p, t2.p, t3.p, t4.p, m, c3.p, c1.p);
  rgfb::k_apply_1d<<<grid_for(nlines, 64, 1 << 20), 64>>>(din.p, dout.p, c3.p, c1.p, m, nlines,
                                                          order, k, transpose, scr.p);
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaMemcpy(out, dout.p, static_cast<size_t>(m * nlines) * sizeof(double),
                     cudaMemcpyDeviceToHost));
}

int rgf_rf3_filter(const double* in, const double* alpha1, const double* alpha2,
                   const double* alpha3, const double* beta, int64_t m, int64_t nlines,
                   int transpose, double* out) {
  return guarded([&] {
    if (m < 4) throw InvalidArgument("rf3 filter: segment length must be >= 4");  // rf3.hpp:296
    if (nlines < 1) throw InvalidArgument("rf3 filter: nlines must be >= 1");
    if (!in || !alpha1 || !alpha2 || !alpha3 || !beta || !out)
      throw InvalidArgument("rf3 filter: null argument");
    filter_tables_1d(in, alpha1, alpha2, alpha3, beta, m, nlines, 3, 1, transpose, out);
  });
}

int rgf_rf1_filter(const double* in, const double* alpha, const double* beta, int64_t m,
                   int64_t nlines, int k, int transpose, double* out) {
  return guarded([&] {
    if (m < 2) throw InvalidArgument("rf1 filter: segment length must be >= 2");  // rf1.hpp:117
    if (nlines < 1) throw InvalidArgument("rf1 filter: nlines must be >= 1");
    if (k < 1) throw InvalidArgument("rf1_coefficients: k must be >= 1");
    if (!in || !alpha || !beta || !out) throw InvalidArgument("rf1 filter: null argument");
    filter_tables_1d(in, alpha, nullptr, nullptr, beta, m, nlines, 1, k, transpose, out);
  });
}

int rgf_rf3_apply_1d(const double* in, const double* sigma, int64_t m, int64_t nlines,
                     int calibration, int transpose, double* out) {
  return guarded([&] {
    for (int64_t i = 0; i < m; ++i)
      if (!(sigma[i] > 0)) throw InvalidArgument("rf3_filter_scalars: sigma must be positive");
    if (m < 4) throw InvalidArgument("rf3 filter: segment length must be >= 4");
    if (nlines < 1) throw InvalidArgument("rf3 filter: nlines must be >= 1");
    apply_1d(in, sigma, m, nlines, 3, 1, calibration, transpose, out);
  });
}

int rgf_rf1_apply_1d(const double* in, const double* sigma, int64_t m, int64_t nlines, int k,
                     int transpose, double* out) {
  return guarded([&] {
    for (int64_t i = 0; i < m; ++i)
      if (!(sigma[i] > 0)) throw InvalidArgument("rf1_coefficients: sigma must be positive");
    if (k < 1) throw InvalidArgument("rf1_coefficients: k must be >= 1");
    if (m < 2) throw InvalidArgument("rf1 filter: segment length must be >= 2");
    if (nlines < 1) throw InvalidArgument("rf1 filter: nlines must be >= 1");
    apply_1d(in, sigma, m, nlines, 1, k, RGF_CAL_YVV95, transpose, out);
  });
}


// ------------------------------------------------------------ observations
int rgf_obs_create(const rgf_grid_desc* grid, int32_t device, int64_t n, const double* x,
                   const double* y, const double* values, const double* r_var, rgf_obs** out) {
  return guarded([&] {
    if (!grid || !grid->mask || !out) throw InvalidArgument("obs: null argument");
    if (grid->nx < 2 || grid->ny < 2) throw InvalidArgument("obs: grid too small");
    if (n < 0) throw InvalidArgument("ObsSet: inconsistent column lengths");
    if (n > 0 && (!x || !y || !values || !r_var)) throw InvalidArgument("obs: null argument");
    if (n >= (int64_t(1) << 29)) throw InvalidArgument("obs: too many observations");
    CUDA_OK(cudaSetDevice(device));
    auto o = std::make_unique<rgf_obs>();
    o->device = device;
    o->n = n;
    o->nx = grid->nx;
    o->ny = grid->ny;
    std::vector<int64_t> cell(static_cast<size_t>(n));
    std::vector<double4> w(static_cast<size_t>(n));
    for (int64_t k = 0; k < n; ++k) {
      int64_t i0, j0;
      obs_stencil(grid, x[k], y[k], k, i0, j0, w[static_cast<size_t>(k)]);
      cell[static_cast<size_t>(k)] = j0 * grid->nx + i0;
    }
    o->values_h.assign(values, values + n);
    o->rvar_h.assign(r_var, r_var + n);
    // H^T gather lists: the touched cells in ascending order, each with its
    // (observation, corner) entries in observation order. A stable sort of the
    // 4n entries by cell (O(n log n); a counting sort over the nx*ny cells
    // cost 10 ms per handle on a 1442x1021 grid).
    auto corner = [&](int64_t k, int q) {
      const int64_t c = cell[static_cast<size_t>(k)];
      return c + (q & 1) + (q >> 1) * grid->nx;
    };
    // keys (cell, entry), sorted by cell with the entries of a cell in observation order
    // (n < 2^29 entries fit 31 bits; cells < 2^33)
    std::vector<uint64_t> ent(static_cast<size_t>(4 * n));
    for (int64_t k = 0; k < n; ++k)
      for (int q = 0; q < 4; ++q)
        ent[static_cast<size_t>(4 * k + q)] =
            (static_cast<uint64_t>(corner(k, q)) << 31) | static_cast<uint64_t>(4 * k + q);
    {  // LSD radix sort on the cell bits (stable; entries were generated in order)
      const int64_t nh = grid->nx * grid->ny;
      int bits = 1;
      while ((int64_t(1) << bits) < nh) ++bits;
      std::vector<uint64_t> tmp(ent.size());
      for (int sh = 0; sh < bits; sh += 11) {
        size_t cnt[2049] = {0};
        for (uint64_t e : ent) ++cnt[((e >> (31 + sh)) & 2047u) + 1];
        for (int b = 0; b < 2048; ++b) cnt[b + 1] += cnt[b];
        for (uint64_t e : ent) tmp[cnt[(e >> (31 + sh)) & 2047u]++] = e;
        ent.swap(tmp);
      }
    }
    std::vector<int64_t> tcells, tptr{0};
    std::vector<int32_t> tent(static_cast<size_t>(4 * n));
    for (size_t e = 0; e < ent.size(); ++e) {
      const int64_t c = static_cast<int64_t>(ent[e] >> 31);
      if (e == 0 || c != static_cast<int64_t>(ent[e - 1] >> 31)) {
        if (e > 0) tptr.push_back(static_cast<int64_t>(e));
        tcells.push_back(c);
      }
      tent[e] = static_cast<int32_t>(ent[e] & 0x7fffffffu);
    }
    if (!ent.empty()) tptr.push_back(static_cast<int64_t>(ent.size()));
    o->ncell = static_cast<int64_t>(tcells.size());
    if (n > 0) {  // one device allocation and one copy (seven cudaMallocs cost milliseconds)
      const size_t sizes[7] = {cell.size() * sizeof(int64_t), w.size() * sizeof(double4),
                               static_cast<size_t>(n) * sizeof(double),
                               static_cast<size_t>(n) * sizeof(double),
                               tcells.size() * sizeof(int64_t), tptr.size() * sizeof(int64_t),
                               tent.size() * sizeof(int32_t)};
      const void* srcs[7] = {cell.data(), w.data(), values, r_var, tcells.data(), tptr.data(),
                             tent.data()};
      size_t off[8] = {0};
      for (int q = 0; q < 7; ++q) off[q + 1] = (off[q] + sizes[q] + 255) / 256 * 256;
      std::vector<char> host(off[7]);
      for (int q = 0; q < 7; ++q) std::memcpy(host.data() + off[q], srcs[q], sizes[q]);
      o->arena.upload(host.data(), host.size());
      char* base = o->arena.p;
      o->cell.borrow(reinterpret_cast<int64_t*>(base + off[0]), cell.size());
      o->w.borrow(reinterpret_cast<double4*>(base + off[1]), w.size());
      o->values.borrow(reinterpret_cast<double*>(base + off[2]), static_cast<size_t>(n));
      o->rvar.borrow(reinterpret_cast<double*>(base + off[3]), static_cast<size_t>(n));
      o->tcells.borrow(reinterpret_cast<int64_t*>(base + off[4]), tcells.size());
      o->tptr.borrow(reinterpret_cast<int64_t*>(base + off[5]), tptr.size());
      o->tent.borrow(reinterpret_cast<int32_t*>(base + off[6]), tent.size());
    }
    *out = o.release();
  });
}

int rgf_obs_destroy(rgf_obs* o) {
  return guarded([&] {
    if (o) {
      cudaSetDevice(o->device);
      delete o;
    }
  });
}

// transpose 0: out (n) = H in (ny*nx field); 1: out (field) = H^T in (n)
int rgf_obs_apply(rgf_obs* o, int transpose, const double* in, double* out, int memory,
                  void* stream) {
  return guarded([&] {
    if (!o || !in || !out) throw InvalidArgument("obs: null argument");
    std::lock_guard<std::mutex> lock(o->mu);
    CUDA_OK(cudaSetDevice(o->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Cg cg{nullptr, o, st, o->nx * o->ny, {}, {}, {}, {}, {}};
    const int64_t nin = transpose ? o->n : cg.nh, nout = transpose ? cg.nh : o->n;
    DevBuf<double> di, dout;
    const double* src = in;
    double* dst = out;
    if (memory == RGF_HOST) {
      di.alloc(std::max<int64_t>(nin, 1));
      dout.alloc(std::max<int64_t>(nout, 1));
      if (nin > 0)
        CUDA_OK(cudaMemcpyAsync(di.p, in, nin * sizeof(double), cudaMemcpyHostToDevice, st));
      src = di.p;
      dst = dout.p;
    } else if (memory != RGF_DEVICE) {
      throw InvalidArgument("obs: unknown memory kind");
    }
    if (transpose)
      cg.ht(src, nullptr, dst);
    else
      cg.h(src, dst);
    if (memory == RGF_HOST && nout > 0)
      CUDA_OK(cudaMemcpyAsync(out, dst, nout * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
  });
}

// solver.cpp:35-50 (host arrays): j3 = {j_total, j_background, j_obs}
int rgf_cost(rgf_op* op, rgf_obs* o, const double* chi, const double* background, double* j3,
             double* gradient) {
  return guarded([&] {
    if (!op || !o || !chi || !j3 || !gradient) throw InvalidArgument("cost: null argument");
    check_cg_op(op, o);
    validate_rvar(o);
    std::lock_guard<std::mutex> lock(op->mu);
    CUDA_OK(cudaSetDevice(op->device));
    cudaStream_t st = nullptr;
    CUDA_OK(cudaStreamWaitEvent(st, op->scratch_free, 0));
    struct Rec {
      rgf_op* op;
      ~Rec() { cudaEventRecord(op->scratch_free, nullptr); }
    } rec{op};
    Cg cg{op, o, st, op->nx * op->ny, {}, {}, {}, {}, {}};
    cg.init();
    const int64_t nh = cg.nh, n = o->n;
    DevBuf<double> c, bg, d, vc, res, g;
    c.upload(chi, static_cast<size_t>(nh));
    if (background) bg.upload(background, static_cast<size_t>(nh));
    d.alloc(std::max<int64_t>(n, 1));
    res.alloc(std::max<int64_t>(n, 1));
    vc.alloc(nh);
    g.alloc(nh);
    cg.misfit(background ? bg.p : nullptr, d.p);
    cg.v(c.p, vc.p);  // solver.cpp:41
    cg.h(vc.p, cg.tmp_obs.p);
    if (n > 0) {
      rgfb::k_obs_residual<<<blocks_for(n), 256, 0, st>>>(d.p, cg.tmp_obs.p, n, res.p);
      CUDA_OK(cudaGetLastError());
    }
    const double jb = 0.5 * cg.dot(c.p, c.p, nh);
    const double jo = n > 0 ? 0.5 * cg.dot(res.p, nullptr, n, o->rvar.p) : 0.0;
    cg.adjoint_rhs(res.p, g.p);
    rgfb::k_axmy<<<blocks_for(nh), 256, 0, st>>>(g.p, c.p, g.p, 1.0, nh);  // chi - V^T H^T R^-1 r
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaMemcpy(gradient, g.p, nh * sizeof(double), cudaMemcpyDeviceToHost));
    j3[0] = jb + jo;
    j3[1] = jb;
    j3[2] = jo;
  });
}

// solver.cpp:52-114 (host arrays). gnorms: max_iter + 1 slots.
int rgf_solve(rgf_op* op, rgf_obs* o, double tol, int32_t max_iter, const double* background,
              double* increment, double* misfit, double* gnorms, rgf_analysis* out) {
  return guarded([&] {
    if (!(tol > 0)) throw InvalidArgument("solve: tol must be positive");
    if (max_iter < 0) throw InvalidArgument("solve: max_iter must be >= 0");
    if (!op || !o || !increment || !out || !gnorms) throw InvalidArgument("solve: null argument");
    check_cg_op(op, o);
    validate_rvar(o);
    std::lock_guard<std::mutex> lock(op->mu);
    CUDA_OK(cudaSetDevice(op->device));
    cudaStream_t st = nullptr;
    CUDA_OK(cudaStreamWaitEvent(st, op->scratch_free, 0));
    struct Rec {
      rgf_op* op;
      ~Rec() { cudaEventRecord(op->scratch_free, nullptr); }
    } rec{op};
    Cg cg{op, o, st, op->nx * op->ny, {}, {}, {}, {}, {}};
    cg.init();
    const int64_t nh = cg.nh, n = o->n;
    *out = rgf_analysis{};
    std::fill(increment, increment + nh, 0.0);
    // CG work vectors live in the operator (grown on demand, reused by every
    // solve: cudaMalloc/cudaFree of seven fields cost more than the iterations)
    op->cg_work.alloc(static_cast<size_t>(7 * nh + std::max<int64_t>(n, 1)));
    struct View {
      double* p;
    };
    double* const w0 = op->cg_work.p;
    View bg{w0}, b{w0 + nh}, chi{w0 + 2 * nh}, r{w0 + 3 * nh}, p{w0 + 4 * nh}, ap{w0 + 5 * nh},
        t{w0 + 6 * nh}, d{w0 + 7 * nh};
    if (background)
      CUDA_OK(cudaMemcpy(bg.p, background, nh * sizeof(double), cudaMemcpyHostToDevice));
    cg.misfit(background ? bg.p : nullptr, d.p);
    if (n > 0 && misfit)
      CUDA_OK(cudaMemcpy(misfit, d.p, n * sizeof(double), cudaMemcpyDeviceToHost));
    if (n == 0) {
      out->converged = 1;
      return;
    }
    const int blk = blocks_for(nh);
    cg.adjoint_rhs(d.p, b.p);
    const double bnorm = std::sqrt(cg.dot(b.p, b.p, nh));
    if (bnorm == 0) {
      out->converged = 1;
      return;
    }
    CUDA_OK(cudaMemsetAsync(chi.p, 0, nh * sizeof(double), st));
    CUDA_OK(cudaMemcpyAsync(r.p, b.p, nh * sizeof(double), cudaMemcpyDeviceToDevice, st));
    CUDA_OK(cudaMemcpyAsync(p.p, r.p, nh * sizeof(double), cudaMemcpyDeviceToDevice, st));
    double rs = cg.dot(r.p, r.p, nh);
    std::vector<double> gn{std::sqrt(rs)};
    int iters = 0;
    for (int it = 0; it < max_iter; ++it) {
      cg.v(p.p, t.p);  // apply_hessian, solver.cpp:81-85
      cg.h(t.p, cg.tmp_obs.p);
      cg.adjoint_rhs(cg.tmp_obs.p, ap.p);
      rgfb::k_add<<<blk, 256, 0, st>>>(ap.p, p.p, ap.p, nh);
      const double denom = cg.dot(p.p, ap.p, nh);
      if (denom <= 0) break;
      const double alpha = rs / denom;
      rgfb::k_axpy<<<blk, 256, 0, st>>>(chi.p, chi.p, p.p, alpha, nh);
      rgfb::k_axmy<<<blk, 256, 0, st>>>(r.p, r.p, ap.p, alpha, nh);
      CUDA_OK(cudaGetLastError());
      op->launches += 3;
      const double rs_next = cg.dot(r.p, r.p, nh);
      iters = it + 1;
      gn.push_back(std::sqrt(rs_next));
      if (std::sqrt(rs_next) <= tol * bnorm) {
        rs = rs_next;
        break;
      }
      rgfb::k_axpy<<<blk, 256, 0, st>>>(p.p, r.p, p.p, rs_next / rs, nh);
      CUDA_OK(cudaGetLastError());
      op->launches += 1;
      rs = rs_next;
    }
    const double rel = gn.back() / bnorm;
    cg.v(chi.p, t.p);  // increment = V chi
    cg.h(t.p, cg.tmp_obs.p);
    rgfb::k_obs_residual<<<blocks_for(n), 256, 0, st>>>(d.p, cg.tmp_obs.p, n, cg.tmp_obs2.p);
    CUDA_OK(cudaGetLastError());
    const double jb = 0.5 * cg.dot(chi.p, chi.p, nh);
    const double jo = 0.5 * cg.dot(cg.tmp_obs2.p, nullptr, n, o->rvar.p);
    CUDA_OK(cudaMemcpy(increment, t.p, nh * sizeof(double), cudaMemcpyDeviceToHost));
    std::copy(gn.begin(), gn.end(), gnorms);
    out->cg_iterations = iters;
    out->converged = rel <= tol ? 1 : 0;
    out->n_gradient_norms = static_cast<int64_t>(gn.size());
    out->final_relative_residual = rel;
    out->j_background = jb;
    out->j_obs = jo;
  });
}

}  // extern "C"
