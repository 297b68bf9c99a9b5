// k_init.cu — one-off layout kernels run by copa_init (not part of the timed outer iteration).
//   validate     : CSR / times / finiteness checks (copa.h contract)
//   count_fibers : distinct (patient, feature) pairs per patient (warp per patient, smem bitmap)
//   basis        : per-patient orthonormal spline basis C_k = M_k B_k
//   build_fibers : projected slices X'_k = C_k^T X_k, one l-vector per fiber
//   sumsq        : normX = sum of x^2 (FIT denominator)
#include <cub/cub.cuh>

#include "copa_internal.cuh"

namespace copa {

// ------------------------------------------------------------------ validation
__global__ void k_validate_patients(const int64_t* prp, int64_t K, int64_t rows, const double* times, int* err) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  int64_t a = prp[k], b = prp[k + 1];
  if (b <= a || a < 0 || b > rows) { set_err(err, ERR_SHAPE); return; }
  if (times) {
    for (int64_t i = a; i < b; ++i) {
      double t = times[i];
      if (!isfinite(t)) { set_err(err, ERR_INPUT_NONFINITE); return; }
      if (i > a && !(t > times[i - 1])) { set_err(err, ERR_SHAPE); return; }
    }
  }
}

__global__ void k_validate_rows(const int64_t* rp, const int32_t* col, const double* val, int64_t rows, int64_t nnz,
                                int64_t J, int* err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  int64_t a = rp[i], b = rp[i + 1];
  if (a < 0 || b < a || b > nnz) { set_err(err, ERR_SHAPE); return; }
  for (int64_t e = a; e < b; ++e) {
    int32_t j = col[e];
    if (j < 0 || j >= J) { set_err(err, ERR_SHAPE); return; }
    if (!isfinite(val[e])) { set_err(err, ERR_INPUT_NONFINITE); return; }
    for (int64_t f = a; f < e; ++f)
      if (col[f] == j) { set_err(err, ERR_SHAPE); return; }
  }
}

void launch_validate(Handle& h) {
  if (h.K > 0)
    k_validate_patients<<<(unsigned)((h.K + 255) / 256), 256, 0, h.stream>>>(h.p.patient_row_ptr, h.K, h.rows,
                                                                               h.smooth ? h.p.visit_time : nullptr, h.err);
  if (h.rows > 0)
    k_validate_rows<<<(unsigned)((h.rows + 255) / 256), 256, 0, h.stream>>>(h.p.row_ptr, h.p.col, h.p.val, h.rows,
                                                                            h.nnz, h.J, h.err);
}

// ------------------------------------------------------------------ fibers: count
// Warp per patient; each warp owns a J-bit bitmap in shared memory. Also accumulates the number of
// fibers per feature (hist, optional) used to relabel features into balanced ranges.
__global__ void k_count_fibers(const int64_t* prp, const int64_t* rp, const int32_t* col, int64_t K, int words,
                               int64_t* counts, unsigned long long* hist, int64_t J) {
  extern __shared__ unsigned smem_bits[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned* bits = smem_bits + wib * words;
  unsigned* bh = smem_bits + nw * words;  // block histogram [J]
  if (hist)
    for (int64_t j = threadIdx.x; j < J; j += blockDim.x) bh[j] = 0u;
  __syncthreads();
  const int64_t nwarps = (int64_t)gridDim.x * nw;
  for (int64_t k = blockIdx.x * (int64_t)nw + wib; k < K; k += nwarps) {
    for (int w = lane; w < words; w += 32) bits[w] = 0u;
    __syncwarp();
    int64_t e0 = rp[prp[k]], e1 = rp[prp[k + 1]];
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      int32_t j = col[e];
      atomicOr(&bits[j >> 5], 1u << (j & 31));
    }
    __syncwarp();
    int c = 0;
    for (int w = lane; w < words; w += 32) {
      unsigned b = bits[w];
      c += __popc(b);
      if (hist)
        while (b) {
          int bit = __ffs(b) - 1;
          b &= b - 1;
          atomicAdd(&bh[w * 32 + bit], 1u);
        }
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) counts[k + 1] = c;
    __syncwarp();
  }
  if (hist) {
    __syncthreads();
    for (int64_t j = threadIdx.x; j < J; j += blockDim.x)
      if (bh[j]) atomicAdd(&hist[j], (unsigned long long)bh[j]);
  }
}

void launch_count_fibers(Handle& h, int64_t* counts, unsigned long long* hist) {
  int words = (int)((h.J + 31) / 32);
  int warps = 8;
  size_t smem = (size_t)warps * words * sizeof(unsigned) + (hist ? sizeof(unsigned) * (size_t)h.J : 0);
  cudaMemsetAsync(counts, 0, sizeof(int64_t), h.stream);
  if (hist) cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * (size_t)h.J, h.stream);
  if (h.K == 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_count_fibers, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  int64_t blocks = (h.K + warps - 1) / warps;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_count_fibers<<<(unsigned)blocks, warps * 32, smem, h.stream>>>(h.p.patient_row_ptr, h.p.row_ptr, h.p.col, h.K,
                                                                    words, counts, hist, h.J);
}

// ------------------------------------------------------------------ basis (thread per patient)
// M_k rows by the de Boor triangle; Givens-QR of M_k into Rm (l x l); one-sided Jacobi on the
// rows of Rm gives sigma_j v_j; B_k column c (kept j) = v_j / sigma_j, so C_k = M_k B_k are the
// left singular vectors of M_k with sigma_j > tau * sigma_max (reading R-spline-4).
__global__ void k_basis(const int64_t* prp, const double* times, int64_t K, int l, int d, double tau, double* Bk,
                        int32_t* m) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  double Rm[kMaxL * kMaxL];
  double a[kMaxL];
  double N[kMaxDeg + 1];
  for (int i = 0; i < l * kMaxL; ++i) Rm[i] = 0.0;
  int64_t r0 = prp[k], r1 = prp[k + 1];
  double t1 = times[r0], tn = times[r1 - 1];
  double* B = Bk + k * (int64_t)l * l;
  if (!(tn > t1)) {  // single visit: all knots coincide, M_k = 0 (same as the recursion's 0/0 := 0)
    for (int i = 0; i < l * l; ++i) B[i] = 0.0;
    m[k] = 0;
    return;
  }
  for (int64_t i = r0; i < r1; ++i) {
    int mu = spline_eval(times[i], t1, tn, l, d, N);
    for (int b = 0; b < l; ++b) a[b] = 0.0;
    for (int r = 0; r <= d; ++r) a[mu - d + r] = N[r];
    givens_insert(Rm, kMaxL, a, l);
  }
  jacobi_rows(Rm, kMaxL, l);
  double sig[kMaxL], smax = 0.0;
  for (int j = 0; j < l; ++j) {
    double s = 0.0;
    for (int i = 0; i < l; ++i) s = fma(Rm[j * kMaxL + i], Rm[j * kMaxL + i], s);
    sig[j] = sqrt(s);
    smax = fmax(smax, sig[j]);
  }
  // keep in descending sigma order (stable): selection by repeated max
  int used[kMaxL];
  for (int j = 0; j < l; ++j) used[j] = 0;
  int c = 0;
  for (int it = 0; it < l; ++it) {
    int best = -1;
    for (int j = 0; j < l; ++j)
      if (!used[j] && (best < 0 || sig[j] > sig[best])) best = j;
    used[best] = 1;
    if (!(smax > 0.0) || !(sig[best] > tau * smax)) break;
    double inv2 = 1.0 / (sig[best] * sig[best]);
    for (int i = 0; i < l; ++i) B[i * l + c] = Rm[best * kMaxL + i] * inv2;
    ++c;
  }
  for (int cc = c; cc < l; ++cc)
    for (int i = 0; i < l; ++i) B[i * l + cc] = 0.0;
  m[k] = c;
}

void launch_basis(Handle& h) {
  if (h.K == 0) return;
  k_basis<<<(unsigned)((h.K + 63) / 64), 64, 0, h.stream>>>(h.p.patient_row_ptr, h.p.visit_time, h.K, h.l, h.d,
                                                          h.o.basis_tol, h.Bk, h.m);
}

// ------------------------------------------------------------------ fibers: per-group counts
// Patient bitmap over the relabeled feature ids (labels); the fibers of group g are the distinct
// labels in [g Jg, (g+1) Jg). rank(x) = number of the patient's labels below x.
__device__ __forceinline__ void patient_label_bitmap(const int64_t* prp, const int64_t* rp, const int32_t* col,
                                                     const int32_t* perm, int64_t k, int words, unsigned* bits,
                                                     int* pref) {
  const int lane = threadIdx.x & 31;
  for (int w = lane; w < words; w += 32) bits[w] = 0u;
  __syncwarp();
  const int64_t e0 = rp[prp[k]], e1 = rp[prp[k + 1]];
  for (int64_t e = e0 + lane; e < e1; e += 32) {
    const int32_t j = perm[col[e]];
    atomicOr(&bits[j >> 5], 1u << (j & 31));
  }
  __syncwarp();
  // exclusive prefix of popcounts over words (warp-strided chunks)
  int carry = 0;
  for (int w0 = 0; w0 < words; w0 += 32) {
    const int w = w0 + lane;
    const int c = w < words ? __popc(bits[w]) : 0;
    int inc = c;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (w < words) pref[w] = carry + inc - c;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  __syncwarp();
}

__device__ __forceinline__ int label_rank(const unsigned* bits, const int* pref, int words, int64_t x) {
  const int64_t w = x >> 5;
  if (w >= words) return pref[words - 1] + __popc(bits[words - 1]);
  return pref[w] + __popc(bits[w] & ((1u << (x & 31)) - 1u));
}

// Also writes, per (group, patient), the offsets of the W label sub-runs inside the run:
// woff[(g K + k) kWoS + w] = rank(g Jg + w Js) - rank(g Jg), w = 0..W (W < kWoS).
__global__ void k_count_groups(const int64_t* prp, const int64_t* rp, const int32_t* col, const int32_t* perm,
                               int64_t K, int words, int G, int64_t Jg, int W, int64_t Js, int32_t* gcnt /*[G][K]*/,
                               uint16_t* woff /*[G][K][8]*/) {
  extern __shared__ unsigned smem_g[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned* bits = smem_g + wib * words;
  int* pref = (int*)(smem_g + nw * words) + wib * words;
  const int64_t nwarps = (int64_t)gridDim.x * nw;
  for (int64_t k = blockIdx.x * (int64_t)nw + wib; k < K; k += nwarps) {
    patient_label_bitmap(prp, rp, col, perm, k, words, bits, pref);
    if (lane < G) {
      const int a = label_rank(bits, pref, words, lane * Jg);
      const int b = label_rank(bits, pref, words, (lane + 1) * Jg);
      gcnt[(int64_t)lane * K + k] = b - a;
    }
    for (int x = lane; x < G * kWoS; x += 32) {
      const int g = x / kWoS, w = x % kWoS;
      const int a = label_rank(bits, pref, words, g * Jg);
      const int v = w <= W ? label_rank(bits, pref, words, g * Jg + (int64_t)w * Js) - a : 0;
      woff[((int64_t)g * K + k) * kWoS + w] = (uint16_t)v;
    }
    __syncwarp();
  }
}

void launch_count_groups(Handle& h, int32_t* gcnt) {
  if (h.K == 0) return;
  const int words = (int)((h.Jl + 31) / 32);
  const int warps = 8;
  const size_t smem = (size_t)warps * words * (sizeof(unsigned) + sizeof(int));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_count_groups, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  int64_t blocks = (h.K + warps - 1) / warps;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_count_groups<<<(unsigned)blocks, warps * 32, smem, h.stream>>>(h.p.patient_row_ptr, h.p.row_ptr, h.p.col, h.perm,
                                                                    h.K, words, h.sc_G, h.sc_Jg, h.sc_W, h.sc_Js, gcnt,
                                                                    h.woff);
}

// ------------------------------------------------------------------ fibers: build X'_k = C_k^T X_k
// Warp per patient. The fibers of a patient are its distinct labels; the fiber with label j goes to
// stream g = j / Jg at gptr[g][k] + (rank(j) - rank(g Jg)), so every stream is sorted by label within
// each patient. Rows are processed in order; within a row the lanes own distinct nonzeros (distinct
// columns => distinct fibers), so the accumulation is race-free and its order (ascending row)
// deterministic.
__global__ void k_build_fibers(const int64_t* prp, const int64_t* rp, const int32_t* col, const double* val,
                               const double* times, int64_t K, int words, int l, int d, const double* Bk,
                               const int32_t* m, const int64_t* gptr, int G, int64_t Jg, const int32_t* perm,
                               int32_t* fiber_col, double* fiber_val) {
  extern __shared__ unsigned smem_b[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  unsigned* bits = smem_b + wib * words;
  int* pref = (int*)(smem_b + nw * words) + wib * words;
  const int64_t nwarps = (int64_t)gridDim.x * nw;
  const int64_t K1 = K + 1;
  for (int64_t k = blockIdx.x * (int64_t)nw + wib; k < K; k += nwarps) {
    patient_label_bitmap(prp, rp, col, perm, k, words, bits, pref);
    // per-group destination offset: dst(j) = gptr[g][k] - rank(g Jg) + rank(j)
    int64_t gdst[kMaxGroups];
#pragma unroll
    for (int g = 0; g < kMaxGroups; ++g)
      gdst[g] = g < G ? gptr[g * K1 + k] - label_rank(bits, pref, words, g * Jg) : 0;
    for (int w = lane; w < words; w += 32) {
      unsigned b = bits[w];
      int rk = pref[w];
      while (b) {
        const int bit = __ffs(b) - 1;
        b &= b - 1;
        const int64_t j = (int64_t)w * 32 + bit;
        const int g = (int)(j / Jg);
        const int64_t dst = gdst[g] + rk;
        fiber_col[dst] = (int32_t)j;
        for (int a = 0; a < l; ++a) fiber_val[dst * l + a] = 0.0;
        ++rk;
      }
    }
    __syncwarp();
    const int mk = m[k];
    const double* B = Bk + k * (int64_t)l * l;
    const int64_t r0 = prp[k], r1 = prp[k + 1];
    const double t1 = times[r0], tn = times[r1 - 1];
    if (mk > 0) {
      for (int64_t i = r0; i < r1; ++i) {
        double N[kMaxDeg + 1];
        const int mu = spline_eval(times[i], t1, tn, l, d, N);
        double c[kMaxL];  // C_k(i, :) = M_k(i, :) B_k
        for (int a = 0; a < mk; ++a) {
          double s = 0.0;
          for (int r = 0; r <= d; ++r) s = fma(N[r], B[(mu - d + r) * l + a], s);
          c[a] = s;
        }
        for (int64_t e = rp[i] + lane; e < rp[i + 1]; e += 32) {
          const int32_t j = perm[col[e]];
          const double x = val[e];
          const int g = (int)(j / Jg);
          double* dst = fiber_val + (gdst[g] + label_rank(bits, pref, words, j)) * l;
          for (int a = 0; a < mk; ++a) dst[a] = fma(x, c[a], dst[a]);
        }
        __syncwarp();
      }
    }
    __syncwarp();
  }
}

void launch_build_fibers(Handle& h) {
  if (h.K == 0) return;
  const int words = (int)((h.Jl + 31) / 32);  // bitmap over relabeled feature ids
  const int warps = 8;
  const size_t smem = (size_t)warps * words * (sizeof(unsigned) + sizeof(int));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_build_fibers, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  int64_t blocks = (h.K + warps - 1) / warps;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_build_fibers<<<(unsigned)blocks, warps * 32, smem, h.stream>>>(
      h.p.patient_row_ptr, h.p.row_ptr, h.p.col, h.p.val, h.p.visit_time, h.K, words, h.l, h.d, h.Bk, h.m, h.gptr,
      h.sc_G, h.sc_Jg, h.perm, h.fiber_col, h.fiber_val);
}

// ------------------------------------------------------------------ non-smooth helpers
__global__ void k_row_patient(const int64_t* prp, int64_t K, int32_t* row_patient, int32_t* m, int64_t* srow) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  int64_t a = prp[k], b = prp[k + 1];
  for (int64_t i = a; i < b; ++i) row_patient[i] = (int32_t)k;
  m[k] = (int32_t)(b - a);
  srow[k] = a;
  if (k == K - 1) srow[K] = b;
}

void launch_row_patient(Handle& h) {
  if (h.K == 0) return;
  k_row_patient<<<(unsigned)((h.K + 255) / 256), 256, 0, h.stream>>>(h.p.patient_row_ptr, h.K, h.row_patient, h.m,
                                                                     h.srow);
}

// ------------------------------------------------------------------ normX
__global__ void k_sumsq(const double* val, int64_t n, double* partial) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    s = fma(val[e], val[e], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}
__global__ void k_sum_partials(const double* partial, int n, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partial[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

void launch_sumsq(Handle& h, double* out) {
  k_sumsq<<<kPartBlocks, 256, 0, h.stream>>>(h.p.val, h.nnz, h.partial);
  k_sum_partials<<<1, 256, 0, h.stream>>>(h.partial, kPartBlocks, out);
}

}  // namespace copa
