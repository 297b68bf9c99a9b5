// Verifies the mma.sync.m8n8k4 f64 fragment layout assumed by the kernels:
//   A (8x4 row): lane holds A[g][t]   (g = lane>>2, t = lane&3)
//   B (4x8 col): lane holds B[t][g]
//   C (8x8):     lane holds C[g][2t+i], i = 0,1
#include <cstdio>
__global__ void k(double* out) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a = 1.0 + g * 10 + t;          // A[g][t] = 1 + 10 g + t
  double b = (t == 0 ? 1.0 : 0.0) * (g + 1) + (t == 1 ? 100.0 : 0.0);  // B[t][n]: row0 = n+1, row1 = 100
  double c0 = 0, c1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  out[g * 8 + 2 * t] = c0;
  out[g * 8 + 2 * t + 1] = c1;
}
int main() {
  double* d; cudaMalloc(&d, 64 * 8); k<<<1, 32>>>(d); double h[64]; cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 8; ++m) for (int n = 0; n < 8; ++n) {
    // C[m][n] = sum_k A[m][k] B[k][n] = A[m][0]*(n+1) + A[m][1]*100
    double ref = (1.0 + 10 * m) * (n + 1) + (1.0 + 10 * m + 1) * 100.0;
    if (h[m * 8 + n] != ref) { ++bad; if (bad < 5) printf("mismatch m=%d n=%d got %f ref %f\n", m, n, h[m*8+n], ref); }
  }
  printf("layout %s\n", bad ? "WRONG" : "OK");
}
