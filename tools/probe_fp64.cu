// Microbenchmark: FP64 FMA throughput and clocks on this B200 (used to derive the "alu" roofline peak).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void copy_k(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("name=%s sms=%d smem_optin=%zu l2=%d clock_khz=%d\n", p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin, p.l2CacheSize, p.clockRate);
  double* out; cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bpsm = 1; bpsm <= 8; bpsm *= 2) {
    int blocks = p.multiProcessorCount * bpsm, threads = 256, iters = 4000;
    dfma_loop<<<blocks, threads>>>(out, 10, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("dfma blocks/sm=%d warps/sm=%d: %.2f TFLOP/s (%.3f ms)\n", bpsm, bpsm * 8, flops / ms / 1e9, ms);
  }
  size_t n = (size_t)1 << 28; double4 *a, *b; cudaMalloc(&a, n * 32); cudaMalloc(&b, n * 32);
  cudaMemset(a, 0, n * 32);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); copy_k<<<148 * 8, 512>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.1f GB/s\n", 2.0 * n * 32 / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
