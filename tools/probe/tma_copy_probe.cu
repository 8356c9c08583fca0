// Diagnostic: how fast can the checkpointed sweeps' TMA access pattern move
// data with no arithmetic? A CTA walks a line of blocks (descending, like
// the x C2 kernel) and copies each [W points x P planes x R rows] box from
// `in` to `out` through shared memory (TMA load -> TMA store), 3 buffers.
// Varying W (contiguous bytes per (plane,row) run) at fixed box bytes tests
// whether DRAM row locality caps the C2 kernels at ~5 TB/s.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tma_copy_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  static PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
  if (!f) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    f = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return f;
}
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S>
__global__ void __launch_bounds__(128) k_copy(const __grid_constant__ CUtensorMap tin,
                                              const __grid_constant__ CUtensorMap tout, int nblk,
                                              int W, int P, int R, int planes, int ny, int box_bytes) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = sm_raw + ((1024u - (su(sm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + S * box_bytes);
  const int PB = planes / P;
  const int rg = blockIdx.x / PB, pg = blockIdx.x % PB;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  auto load = [&](int b) {
    const int s = b % S;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])),
                 "r"(box_bytes));
    const int x0 = (nblk - 1 - b) * W;
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            su(sm + s * box_bytes)),
        "l"(&tin), "r"(x0), "r"(pg * P), "r"(rg * R), "r"(su(&full[s]))
        : "memory");
  };
  for (int b = 0; b < S && b < nblk; ++b) load(b);
  for (int b = 0; b < nblk; ++b) {
    const int s = b % S;
    const uint32_t par = (b / S) & 1;
    asm volatile(
        "{\n .reg .pred P1;\nW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra W;\n}" ::"r"(
            su(&full[s])),
        "r"(par)
        : "memory");
    const int x0 = (nblk - 1 - b) * W;
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     &tout),
                 "r"(x0), "r"(pg * P), "r"(rg * R), "r"(su(sm + s * box_bytes))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (b + S < nblk) load(b + S);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const int nx = 4320, ny = 2160, planes = 128;  // 128 planes so boxes tile exactly
  const size_t n = (size_t)nx * ny * planes;
  double *a, *b;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMemset(a, 0, n * 8);
  struct Shape { int W, P, R, S, ctas_per_sm; };
  const Shape shapes[] = {{16, 128, 4, 3, 1}, {16, 128, 4, 3, 2}, {32, 64, 4, 3, 1}, {32, 64, 4, 3, 2},
                          {64, 32, 4, 3, 2}, {16, 64, 4, 3, 2}, {32, 32, 4, 6, 2}, {128, 16, 4, 3, 2}};
  for (const Shape& sh : shapes) {
    CUtensorMap tin, tout;
    const uint64_t dims[3] = {(uint64_t)nx, (uint64_t)planes, (uint64_t)ny};
    const uint64_t str[2] = {(uint64_t)nx * ny * 8, (uint64_t)nx * 8};
    const uint32_t box[3] = {(uint32_t)sh.W, (uint32_t)sh.P, (uint32_t)sh.R};
    const uint32_t es[3] = {1, 1, 1};
    const CUtensorMapSwizzle sw = sh.W * 8 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r1 = enc()(&tin, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, a, dims, str, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult r2 = enc()(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, b, dims, str, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r1 || r2) { printf("W=%d box encode failed %d %d\n", sh.W, r1, r2); continue; }
    const int box_bytes = sh.W * sh.P * sh.R * 8;
    const int smem = sh.S * box_bytes + 64 + 1024;
    auto kern = sh.S == 3 ? k_copy<3> : k_copy<6>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int nblk = nx / sh.W;
    const int grid = (ny / sh.R) * (planes / sh.P);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) kern<<<grid, 128, smem>>>(tin, tout, nblk, sh.W, sh.P, sh.R, planes, ny, box_bytes);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int rep = 0; rep < reps; ++rep) kern<<<grid, 128, smem>>>(tin, tout, nblk, sh.W, sh.P, sh.R, planes, ny, box_bytes);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, smem);
    printf("box W=%3d pts (%4d B runs) P=%3d R=%d S=%d smem=%6d B occ=%d CTA/SM: %.3f ms, %.0f GB/s (read+write) err=%s\n",
           sh.W, sh.W * 8, sh.P, sh.R, sh.S, smem, occ, ms, 2.0 * n * 8 / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
