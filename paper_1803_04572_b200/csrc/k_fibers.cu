// k_fibers.cu — the two streaming passes over the projected fibers X'_k (smooth path), FP64 on
// the tensor cores (mma.sync m8n8k4 f64 = SASS DMMA; 36.9 TFLOP/s measured).
//
// Fiber (k, j): the l-vector x'_kj = X'_k(:, j) = C_k^T X_k(:, j). Fibers of a patient are
// contiguous and sorted by feature j.
//
// Pass A  P'_k = X'_k V(cols_k, :)          (m_k x R)   — per patient, warp per patient,
//         dynamic scheduling over patients sorted by fiber count, V staged in shared memory.
//         GEMM shape per 4 fibers: M = basis index a (8/tile), N = r (8/tile), K = fibers (4).
// Pass B  F_V(j, :) += x'_kj^T N_k              (J x R)   — each CTA owns a private F_V in shared
//         memory and a balanced contiguous patient range; warp w of the CTA owns the feature range
//         [jlo_w, jlo_{w+1}) so no two warps ever update the same row: no atomics, deterministic.
//         GEMM shape per 8 fibers: M = fibers (8), N = r (8/tile), K = a (4/step).
//         The per-CTA F_V copies are summed in a fixed order (deterministic).
#include <cub/cub.cuh>

#include "copa_internal.cuh"

namespace copa {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------------ pass A
template <int MT, int NT, bool VSMEM>
__global__ void __launch_bounds__(512) k_spmm_mma(const int64_t* __restrict__ fiber_ptr,
                                                  const int32_t* __restrict__ fiber_col,
                                                  const double* __restrict__ fiber_val, const int32_t* __restrict__ m,
                                                  const int64_t* __restrict__ srow, const int32_t* __restrict__ order,
                                                  int64_t K, int l, int R, int64_t J, const double* __restrict__ Vg,
                                                  double* __restrict__ Pp, int* counter) {
  extern __shared__ double smem_v[];
  const double* V = Vg;
  if (VSMEM) {
    const int64_t n = J * R;
    for (int64_t x = threadIdx.x; x < n; x += blockDim.x) smem_v[x] = Vg[x];
    __syncthreads();
    V = smem_v;
  }
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  for (;;) {
    int idx = 0;
    if (lane == 0) idx = atomicAdd(counter, 1);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= K) break;
    const int64_t k = order[idx];
    const int64_t f0 = fiber_ptr[k], f1 = fiber_ptr[k + 1];
    double acc[MT][NT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    for (int64_t fb = f0; fb < f1; fb += 8) {
      // two k-steps (8 fibers) per trip: loads first, then the MMAs
      double afr[2][MT], bfr[2][NT];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int64_t f = fb + 4 * s + t;
        const bool ok = f < f1;
        const int64_t j = ok ? (int64_t)fiber_col[f] : 0;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int a = mt * 8 + g;
          afr[s][mt] = (ok && a < l) ? fiber_val[f * l + a] : 0.0;
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int r = nt * 8 + g;
          bfr[s][nt] = (ok && r < R) ? V[j * R + r] : 0.0;
        }
      }
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], afr[s][mt], bfr[s][nt]);
    }
    const int mk = m[k];
    double* out = Pp + srow[k] * R;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int a = mt * 8 + g;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r = nt * 8 + 2 * t + i;
          if (a < mk && r < R) out[a * R + r] = acc[mt][nt][i];
        }
    }
  }
}

template <int MT, int NT, bool VS>
static void spmm_inst(Handle& h, int smem_bytes) {
  auto fn = k_spmm_mma<MT, NT, VS>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 512, smem_bytes);
  if (per_sm < 1) per_sm = 1;
  cudaMemsetAsync(h.counter, 0, sizeof(int), h.stream);
  fn<<<148 * per_sm, 512, smem_bytes, h.stream>>>(h.fiber_ptr, h.fiber_col, h.fiber_val, h.m, h.srow, h.order, h.K,
                                                   h.l, h.R, h.J, h.V, h.Pp, h.counter);
}

template <int MT, int NT>
static void spmm_dispatch_v(Handle& h) {
  size_t vbytes = sizeof(double) * (size_t)(h.J * h.R);
  if (vbytes <= 200 * 1024) spmm_inst<MT, NT, true>(h, (int)vbytes);
  else spmm_inst<MT, NT, false>(h, 0);
}

template <int MT>
static void spmm_dispatch_n(Handle& h) {
  switch ((h.R + 7) / 8) {
    case 1: spmm_dispatch_v<MT, 1>(h); break;
    case 2: spmm_dispatch_v<MT, 2>(h); break;
    case 3: spmm_dispatch_v<MT, 3>(h); break;
    case 4: spmm_dispatch_v<MT, 4>(h); break;
    case 5: spmm_dispatch_v<MT, 5>(h); break;
    case 6: spmm_dispatch_v<MT, 6>(h); break;
    case 7: spmm_dispatch_v<MT, 7>(h); break;
    default: spmm_dispatch_v<MT, 8>(h); break;
  }
}

void launch_spmm_fibers(Handle& h) {
  if (h.l <= 8) spmm_dispatch_n<1>(h);
  else spmm_dispatch_n<2>(h);
}

// ------------------------------------------------------------------ pass B
// Warp w of each CTA: features [jlo[w], jlo[w+1]); for patient k its fibers are
// [f0 + woff[k*(W+1)+w], f0 + woff[k*(W+1)+w+1]).
template <int KS, int NT>
__global__ void __launch_bounds__(512) k_scatter_mma(const int64_t* __restrict__ fiber_ptr,
                                                     const int32_t* __restrict__ fiber_col,
                                                     const double* __restrict__ fiber_val,
                                                     const int32_t* __restrict__ m, const int64_t* __restrict__ srow,
                                                     const uint16_t* __restrict__ woff,
                                                     const int64_t* __restrict__ block_k, int l, int R, int64_t J,
                                                     const double* __restrict__ Nst, double* __restrict__ FVpart) {
  extern __shared__ double Fs[];
  const int64_t JR = J * R;
  for (int64_t x = threadIdx.x; x < JR; x += blockDim.x) Fs[x] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t k0 = block_k[blockIdx.x], k1 = block_k[blockIdx.x + 1];
  for (int64_t k = k0; k < k1; ++k) {
    const uint16_t* wo = woff + k * (W + 1);
    const int64_t f0 = fiber_ptr[k];
    const int64_t fa = f0 + wo[w], fz = f0 + wo[w + 1];
    if (fa >= fz) continue;
    const int mk = m[k];
    const double* N = Nst + srow[k] * R;
    double bfr[KS][NT];  // B[t][g] = N(a = 4 ks + t, r = 8 nt + g)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int a = 4 * ks + t, r = 8 * nt + g;
        bfr[ks][nt] = (a < mk && r < R) ? N[a * R + r] : 0.0;
      }
    for (int64_t fb = fa; fb < fz; fb += 8) {
      const int64_t f = fb + g;  // A[g][t] = X'(a = 4 ks + t, fiber fb + g)
      const bool ok = f < fz;
      double afr[KS];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int a = 4 * ks + t;
        afr[ks] = (ok && a < l) ? fiber_val[f * l + a] : 0.0;
      }
      double c[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        c[nt][0] = c[nt][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) dmma(c[nt][0], c[nt][1], afr[ks], bfr[ks][nt]);
      }
      // C[g][2t+i] = contribution of fiber fb+g to column 8 nt + 2t + i
      if (ok) {
        const int64_t j = fiber_col[f];
        double* row = Fs + j * R;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int r = 8 * nt + 2 * t + i;
            if (r < R) row[r] += c[nt][i];
          }
      }
    }
  }
  __syncthreads();
  double* out = FVpart + (int64_t)blockIdx.x * JR;
  for (int64_t x = threadIdx.x; x < JR; x += blockDim.x) out[x] = Fs[x];
}

__global__ void k_sum_blocks(const double* __restrict__ part, int nb, int64_t n, double* __restrict__ out) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= n) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += part[(int64_t)b * n + x];
  out[x] = s;
}

template <int KS, int NT>
static void scatter_inst(Handle& h) {
  auto fn = k_scatter_mma<KS, NT>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  size_t smem = sizeof(double) * (size_t)(h.J * h.R);
  fn<<<h.sc_blocks, 32 * h.sc_warps, smem, h.stream>>>(h.fiber_ptr, h.fiber_col, h.fiber_val, h.m, h.srow, h.woff,
                                                       h.block_k, h.l, h.R, h.J, h.Nst, h.fv_part);
  int64_t n = h.J * h.R;
  k_sum_blocks<<<(unsigned)((n + 255) / 256), 256, 0, h.stream>>>(h.fv_part, h.sc_blocks, n, h.FV);
}

template <int KS>
static void scatter_dispatch_n(Handle& h) {
  switch ((h.R + 7) / 8) {
    case 1: scatter_inst<KS, 1>(h); break;
    case 2: scatter_inst<KS, 2>(h); break;
    case 3: scatter_inst<KS, 3>(h); break;
    case 4: scatter_inst<KS, 4>(h); break;
    case 5: scatter_inst<KS, 5>(h); break;
    case 6: scatter_inst<KS, 6>(h); break;
    case 7: scatter_inst<KS, 7>(h); break;
    default: scatter_inst<KS, 8>(h); break;
  }
}

int launch_scatter_fibers(Handle& h) {
  switch ((h.l + 3) / 4) {
    case 1: scatter_dispatch_n<1>(h); break;
    case 2: scatter_dispatch_n<2>(h); break;
    case 3: scatter_dispatch_n<3>(h); break;
    default: scatter_dispatch_n<4>(h); break;
  }
  return 2;
}

bool scatter_smem_ok(const Handle& h) { return sizeof(double) * (size_t)(h.J * h.R) <= 220 * 1024; }

// ------------------------------------------------------------------ init-time layout for the passes
// order: patients sorted by fiber count (descending) for pass A's dynamic scheduler.
__global__ void k_fiber_counts(const int64_t* fiber_ptr, int64_t K, int32_t* cnt, int32_t* idx) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  cnt[k] = (int32_t)(fiber_ptr[k + 1] - fiber_ptr[k]);
  idx[k] = (int32_t)k;
}

// feature histogram of fibers
__global__ void k_feature_hist(const int32_t* fiber_col, int64_t F, unsigned long long* hist) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < F; f += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[fiber_col[f]], 1ull);
}

// woff[k][w] = lower_bound(jlo[w]) within the patient's (sorted) fiber columns, relative to f0.
__global__ void k_warp_offsets(const int64_t* fiber_ptr, const int32_t* fiber_col, int64_t K, int W, const int32_t* jlo,
                               uint16_t* woff) {
  int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (x >= K * (W + 1)) return;
  int64_t k = x / (W + 1);
  int w = (int)(x - k * (W + 1));
  int64_t f0 = fiber_ptr[k], f1 = fiber_ptr[k + 1];
  int32_t key = jlo[w];
  int64_t lo = f0, hi = f1;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (fiber_col[mid] < key) lo = mid + 1; else hi = mid;
  }
  woff[x] = (uint16_t)(lo - f0);
}

// block_k[b] = first patient whose cumulative fiber start >= b * F / nb (balanced patient ranges)
__global__ void k_block_ranges(const int64_t* fiber_ptr, int64_t K, int nb, int64_t* block_k) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nb) return;
  if (b == nb) { block_k[nb] = K; return; }
  int64_t F = fiber_ptr[K];
  int64_t target = (F * b) / nb;
  int64_t lo = 0, hi = K;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (fiber_ptr[mid] < target) lo = mid + 1; else hi = mid;
  }
  block_k[b] = lo;
}

size_t fiber_layout_temp_bytes(int64_t K) {
  size_t a = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, a, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                            (int32_t*)nullptr, (int)K);
  return a + 256;
}

// Builds order, woff, jlo, block_k. tmp: >= fiber_layout_temp_bytes(K) + 16 K bytes + 8 (J+1) bytes.
void build_fiber_layout(Handle& h, void* tmp, size_t tmp_bytes) {
  cudaStream_t s = h.stream;
  char* p = (char*)tmp;
  auto take = [&](size_t n) { char* r = p; p += (n + 255) & ~(size_t)255; return (void*)r; };
  int32_t* cnt = (int32_t*)take(sizeof(int32_t) * (size_t)h.K);
  int32_t* cnt_sorted = (int32_t*)take(sizeof(int32_t) * (size_t)h.K);
  int32_t* idx = (int32_t*)take(sizeof(int32_t) * (size_t)h.K);
  unsigned long long* hist = (unsigned long long*)take(sizeof(unsigned long long) * (size_t)h.J);
  size_t sort_bytes = fiber_layout_temp_bytes(h.K);
  void* sort_tmp = take(sort_bytes);
  if (h.K > 0) {
    k_fiber_counts<<<(unsigned)((h.K + 255) / 256), 256, 0, s>>>(h.fiber_ptr, h.K, cnt, idx);
    cub::DeviceRadixSort::SortPairsDescending(sort_tmp, sort_bytes, cnt, cnt_sorted, idx, h.order, (int)h.K, 0, 32, s);
  }
  // feature ranges of the scatter warps, balanced by fiber mass (host computes the cut points)
  cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * (size_t)h.J, s);
  if (h.F > 0) k_feature_hist<<<148 * 8, 256, 0, s>>>(h.fiber_col, h.F, hist);
  std::vector<unsigned long long> hh((size_t)h.J);
  cudaMemcpyAsync(hh.data(), hist, sizeof(unsigned long long) * (size_t)h.J, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  const int W = h.sc_warps;
  std::vector<int32_t> jlo((size_t)W + 1);
  unsigned long long tot = 0;
  for (auto v : hh) tot += v;
  jlo[0] = 0;
  jlo[W] = (int32_t)h.J;
  {
    unsigned long long acc = 0;
    int w = 1;
    for (int64_t j = 0; j < h.J && w < W; ++j) {
      acc += hh[(size_t)j];
      while (w < W && acc * (unsigned long long)W >= tot * (unsigned long long)w) jlo[(size_t)w++] = (int32_t)(j + 1);
    }
    for (; w < W; ++w) jlo[(size_t)w] = (int32_t)h.J;
  }
  cudaMemcpyAsync(h.jlo, jlo.data(), sizeof(int32_t) * (size_t)(W + 1), cudaMemcpyHostToDevice, s);
  if (h.K > 0) {
    int64_t n = h.K * (W + 1);
    k_warp_offsets<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(h.fiber_ptr, h.fiber_col, h.K, W, h.jlo, h.woff);
  }
  k_block_ranges<<<(h.sc_blocks + 1 + 255) / 256, 256, 0, s>>>(h.fiber_ptr, h.K, h.sc_blocks, h.block_k);
  cudaStreamSynchronize(s);  // jlo host vector goes out of scope
}

}  // namespace copa
