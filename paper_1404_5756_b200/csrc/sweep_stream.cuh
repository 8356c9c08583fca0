// Streaming 3rd-RF sweep kernels (placeholder).
#pragma once
#include "common.cuh"
namespace rgfb {
struct StreamArgs {
  int dir, transpose, unit_dc;
  int64_t nx, ny, nlev, nvar;
  const Coef3* c3;
  const double* idc;
  const int64_t* seg_off;
  const int2* segs;
  const int* ghost;
  const double* pre_scale;
  const double* post_scale;
};
inline bool stream_supported(int64_t, int64_t) { return false; }
template <typename T>
int launch_stream_sweep(const T*, T*, const StreamArgs&, cudaStream_t) { return 0; }
}  // namespace rgfb
