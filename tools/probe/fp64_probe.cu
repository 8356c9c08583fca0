// Microbenchmark: FP64 pipe latency/throughput, HBM copy bandwidth, L2 read
// bandwidth on the target B200. Informs the recursive-filter kernel design
// (DESIGN.md "measured machine constants"). Not part of the product.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void dfma_lat(double* out, int iters, double a, double b) {
  double x = threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
  out[1 + threadIdx.x] = x;
}

__global__ void dadd_lat(double* out, int iters, double b) {
  double x = threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __dadd_rn(x, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
  out[1 + threadIdx.x] = x;
}

// rf3 step in the reference's left-to-right unfused order: 4 mul + 3 add
__global__ void rf3_chain_exact(double* out, int iters, double a1, double a2, double a3, double b) {
  double p1 = 1e-3 * threadIdx.x, p2 = 0, p3 = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double s = 1.0;
    double t = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(b, s), __dmul_rn(a1, p1)), __dmul_rn(a2, p2)), __dmul_rn(a3, p3));
    p3 = p2; p2 = p1; p1 = t;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
  out[1 + threadIdx.x] = p1;
}

// rf3 step reassociated so only one DFMA sits on the p1 critical path
__global__ void rf3_chain_fast(double* out, int iters, double a1, double a2, double a3, double b) {
  double p1 = 1e-3 * threadIdx.x, p2 = 0, p3 = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double s = 1.0;
    double t = fma(a1, p1, fma(a2, p2, fma(a3, p3, b * s)));
    p3 = p2; p2 = p1; p1 = t;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
  out[1 + threadIdx.x] = p1;
}

template <int ILP>
__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ in, double2* __restrict__ out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = in[i];
}

__global__ void read_kernel(const double2* __restrict__ in, double* out, size_t n, int reps) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      double2 v = in[i];
      acc += v.x + v.y;
    }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs %d clock %d kHz L2 %d MB persistL2max %d MB smemOptin %zu\n", prop.name,
         prop.multiProcessorCount, prop.clockRate, prop.l2CacheSize >> 20,
         prop.persistingL2CacheMaxSize >> 20, prop.sharedMemPerBlockOptin);
  double* d;
  CK(cudaMalloc(&d, 1 << 26));
  const int iters = 1 << 16;
  double* h = (double*)malloc(8);
  dfma_lat<<<1, 32>>>(d, iters, 0.999, 1e-3); CK(cudaDeviceSynchronize());
  dfma_lat<<<1, 32>>>(d, iters, 0.999, 1e-3); CK(cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost));
  printf("DFMA latency %.2f cyc\n", h[0]);
  dadd_lat<<<1, 32>>>(d, iters, 1e-3); CK(cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost));
  printf("DADD latency %.2f cyc\n", h[0]);
  rf3_chain_exact<<<1, 32>>>(d, iters, 1.7, -1.0, 0.2, 0.2); CK(cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost));
  printf("rf3 step exact-order latency %.2f cyc/step\n", h[0]);
  rf3_chain_fast<<<1, 32>>>(d, iters, 1.7, -1.0, 0.2, 0.2); CK(cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost));
  printf("rf3 step fma-reassoc latency %.2f cyc/step\n", h[0]);

  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  for (int threads : {128, 256, 512, 1024}) {
    const int blocks = prop.multiProcessorCount * (2048 / threads);
    const int it = 4096;
    dfma_tput<8><<<blocks, threads>>>(d, it, 0.999, 1e-3);
    CK(cudaEventRecord(e0));
    dfma_tput<8><<<blocks, threads>>>(d, it, 0.999, 1e-3);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    double fmas = double(blocks) * threads * it * 8;
    printf("DFMA tput (threads/blk %d): %.2f TFMA/s = %.1f TFLOP/s\n", threads, fmas / ms / 1e9, 2 * fmas / ms / 1e9);
  }
  // HBM copy
  size_t bytes = size_t(4) << 30;
  double2 *a, *b;
  CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  CK(cudaMemset(a, 0, bytes));
  size_t n = bytes / 16;
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaEventRecord(e0));
    copy_kernel<<<prop.multiProcessorCount * 8, 256>>>(a, b, n);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("copy 4GiB: %.1f GB/s (r+w)\n", 2.0 * bytes / ms / 1e6);
  }
  // L2 read bandwidth: 32 MB resident buffer read 50 times
  size_t l2n = (size_t(32) << 20) / 16;
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaEventRecord(e0));
    read_kernel<<<prop.multiProcessorCount * 8, 256>>>(a, d, l2n, 50);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("L2 read 32MB x50: %.1f GB/s\n", 50.0 * 32 * (1 << 20) / ms / 1e6);
  }
  // HBM read-only
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaEventRecord(e0));
    read_kernel<<<prop.multiProcessorCount * 8, 256>>>(a, d, n, 1);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("HBM read 4GiB: %.1f GB/s\n", 1.0 * bytes / ms / 1e6);
  }
  printf("done\n");
  return 0;
}
