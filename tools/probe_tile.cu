// Microbenchmark: the pass-B tile (8 fibers x 24 columns, K = 8) with operands in shared memory:
// 2 A-fragment LDS + 1 label LDS + 6 DMMA + 3 F_V row read-modify-writes (random rows), W warps per
// SM (one CTA per SM, 104 KB F_V slice as in pass B at Scale). Reports cycles per tile per SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int MODE>  // 0: full tile, 1: no RMW, 2: RMW only, 3: full with loads-first RMW, 4: 3 + 2-tile batches
__global__ void tile_loop(double* out, int iters, int rows) {
  extern __shared__ double sm[];
  double* Fs = sm;                       // rows x 20
  double* val = sm + rows * 20;          // 256 x 7
  int* col = (int*)(val + 256 * 7);      // 256
  for (int x = threadIdx.x; x < rows * 20; x += blockDim.x) Fs[x] = 0;
  for (int x = threadIdx.x; x < 256 * 7; x += blockDim.x) val[x] = 1e-3 * x;
  unsigned s = 12345u + threadIdx.x;
  for (int x = threadIdx.x; x < 256; x += blockDim.x) { s = s * 1664525u + 1013904223u; col[x] = (s >> 8) % (rows / (blockDim.x >> 5)); }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int nw = blockDim.x >> 5;
  const int rb = w * (rows / nw);  // warp-owned row range
  double b[2][3];
  for (int ks = 0; ks < 2; ++ks) for (int nt = 0; nt < 3; ++nt) b[ks][nt] = 0.5 + ks + nt;
  for (int it = 0; it < iters; it += (MODE == 4 ? 2 : 1)) {
    constexpr int NB = MODE == 4 ? 2 : 1;
    int c[NB];
    double av[NB][2];
    double cc[NB][3][2] = {};
#pragma unroll
    for (int bb = 0; bb < NB; ++bb) {
      const int f = (((it + bb) * 8) & 255) + g;
      c[bb] = col[f] + rb;
      for (int ks = 0; ks < 2; ++ks) { const int a = 4 * ks + t; av[bb][ks] = a < 7 ? val[f * 7 + a] : 0.0; }
    }
    if (MODE != 2) {
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int bb = 0; bb < NB; ++bb)
#pragma unroll
          for (int nt = 0; nt < 3; ++nt) dmma(cc[bb][nt][0], cc[bb][nt][1], av[bb][ks], b[ks][nt]);
    } else {
      for (int nt = 0; nt < 3; ++nt) { cc[0][nt][0] = av[0][0]; cc[0][nt][1] = av[0][1]; }
    }
    if (MODE == 1) {
      for (int nt = 0; nt < 3; ++nt) b[0][nt] += cc[0][nt][0] * 1e-30 + cc[0][nt][1] * 1e-30;
    } else if (MODE == 0 || MODE == 2) {
      double* row = Fs + c[0] * 20;
#pragma unroll
      for (int nt = 0; nt < 3; ++nt)
        if (8 * nt + 2 * t < 20) {
          double2 v = *reinterpret_cast<double2*>(row + 8 * nt + 2 * t);
          v.x += cc[0][nt][0]; v.y += cc[0][nt][1];
          *reinterpret_cast<double2*>(row + 8 * nt + 2 * t) = v;
        }
    } else {
      double2 v[NB][3];
#pragma unroll
      for (int bb = 0; bb < NB; ++bb)
#pragma unroll
        for (int nt = 0; nt < 3; ++nt)
          if (8 * nt + 2 * t < 20) v[bb][nt] = *reinterpret_cast<double2*>(Fs + c[bb] * 20 + 8 * nt + 2 * t);
#pragma unroll
      for (int bb = 0; bb < NB; ++bb)
#pragma unroll
        for (int nt = 0; nt < 3; ++nt)
          if (8 * nt + 2 * t < 20) {
            v[bb][nt].x += cc[bb][nt][0]; v[bb][nt].y += cc[bb][nt][1];
            *reinterpret_cast<double2*>(Fs + c[bb] * 20 + 8 * nt + 2 * t) = v[bb][nt];
          }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = Fs[5] + b[0][0];
}
template <int MODE>
void run(double* out, int warps, const char* name) {
  const int rows = 652, iters = 20000;
  size_t smem = (rows * 20 + 256 * 7) * 8 + 256 * 4;
  cudaFuncSetAttribute(tile_loop<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  tile_loop<MODE><<<148, 32 * warps, smem>>>(out, 100, rows);
  cudaEventRecord(e0); tile_loop<MODE><<<148, 32 * warps, smem>>>(out, iters, rows); cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double cyc = ms * 1e-3 * 1.965e9;
  printf("%-10s warps=%d: %.1f cycles per tile per warp, %.1f cycles per tile per SM\n", name, warps, cyc / iters,
         cyc / iters / warps);
}
int main() {
  double* out; cudaMalloc(&out, 148 * 8);
  for (int w : {4, 8}) {
    run<0>(out, w, "full"); run<1>(out, w, "no-rmw"); run<2>(out, w, "rmw-only");
    run<3>(out, w, "full-ldfirst"); run<4>(out, w, "full-2tile");
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
