// Microbenchmark: DMMA (mma.sync m8n8k4 f64) throughput vs warps per SM and independent chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void dmma_chains(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  double c[C][2];
  for (int t = 0; t < C; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < C; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int t = 0; t < C; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int C>
void run(double* out, int wps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4000;
  dmma_chains<C><<<148, 32 * wps>>>(out, 10);
  cudaEventRecord(e0); dmma_chains<C><<<148, 32 * wps>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = (double)C * iters * 148 * wps;  // DMMAs
  printf("warps/sm=%2d chains=%d: %.2f TFLOP/s, %.1f cycles per DMMA per warp (1965 MHz)\n", wps, C,
         n * 512 / ms / 1e9, ms * 1e-3 * 1.965e9 / ((double)C * iters));
}
int main() {
  double* out; cudaMalloc(&out, 148 * 64 * 1024 * sizeof(double));
  for (int w : {1, 4, 8}) { run<1>(out, w); run<2>(out, w); run<4>(out, w); run<6>(out, w); run<8>(out, w); }
}
