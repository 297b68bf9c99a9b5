// k_init.cu — one-off layout kernels run by copa_init (not part of the timed outer iteration).
//   validate     : CSR / times / finiteness checks (copa.h contract)
//   count_fibers : distinct (patient, feature) pairs per patient (warp per patient, smem bitmap)
//   basis        : per-patient orthonormal spline basis C_k = M_k B_k
//   build_fibers : projected slices X'_k = C_k^T X_k, one l-vector per fiber
//   sumsq        : normX = sum of x^2 (FIT denominator)
#include <cub/cub.cuh>

#include "copa_internal.cuh"
#include "k_dense.cuh"  // register Givens / Jacobi helpers (givens_insert_reg, jacobi_rows_reg)

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

// val may be null: the structure and columns only (copa_fit validates the values once their copy,
// overlapped with the first init stages, has landed: launch_validate_vals)
__global__ void k_validate_rows(const int64_t* rp, const int32_t* col, const double* val, int64_t rows, int64_t nnz,
                                int64_t J, int* err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  int64_t a = rp[i], b = rp[i + 1];
  if (a < 0 || b < a || b > nnz) { set_err(err, ERR_SHAPE); return; }
  for (int64_t e = a; e < b; ++e) {
    int32_t j = col[e];
    if (j < 0 || j >= J) { set_err(err, ERR_SHAPE); return; }
    if (val && !isfinite(val[e])) { set_err(err, ERR_INPUT_NONFINITE); return; }
    for (int64_t f = a; f < e; ++f)
      if (col[f] == j) { set_err(err, ERR_SHAPE); return; }
  }
}

__global__ void k_validate_vals(const double* val, int64_t nnz, int* err) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(val[e])) { set_err(err, ERR_INPUT_NONFINITE); return; }
}

void launch_validate(Handle& h, bool vals) {
  if (h.K > 0)
    k_validate_patients<<<(unsigned)((h.K + 255) / 256), 256, 0, h.stream>>>(h.p.patient_row_ptr, h.K, h.rows,
                                                                               h.smooth ? h.p.visit_time : nullptr, h.err);
  if (h.rows > 0)
    k_validate_rows<<<(unsigned)((h.rows + 255) / 256), 256, 0, h.stream>>>(h.p.row_ptr, h.p.col,
                                                                            vals ? h.p.val : nullptr, h.rows, h.nnz,
                                                                            h.J, h.err);
}

void launch_validate_vals(Handle& h, int64_t e0, int64_t e1) {
  if (e1 < 0) e1 = h.nnz;
  if (e1 > e0) k_validate_vals<<<(unsigned)(h.sms * 8), 256, 0, h.stream>>>(h.p.val + e0, e1 - e0, h.err);
}

// ------------------------------------------------------------------ fibers: count
// Warp per patient; each warp owns a J-bit bitmap in shared memory. Also accumulates the number of
// fibers per feature (hist, optional) used to relabel features into balanced ranges.
// Runs before validation (copa_workspace_size sizes the workspace from it): every index is
// bounds-checked so malformed input yields some count (rejected later by k_validate_*), never an
// out-of-range access.
__global__ void k_count_fibers(const int64_t* prp, const int64_t* rp, const int32_t* col, int64_t K, int words,
                               int64_t* counts, unsigned long long* hist, int64_t J, int64_t rows, int64_t nnz) {
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
    const int64_t a = prp[k], b = prp[k + 1];
    int64_t e0 = 0, e1 = 0;
    if (a >= 0 && b >= a && b <= rows) {
      e0 = rp[a];
      e1 = rp[b];
      if (e0 < 0 || e1 < e0 || e1 > nnz) e0 = e1 = 0;
    }
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      int32_t j = col[e];
      if (j >= 0 && j < J) atomicOr(&bits[j >> 5], 1u << (j & 31));
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
  max_smem_attr<k_count_fibers>(h, 200 * 1024);
  int64_t blocks = (h.K + warps - 1) / warps;
  if (blocks > h.sms * 16) blocks = h.sms * 16;
  k_count_fibers<<<(unsigned)blocks, warps * 32, smem, h.stream>>>(h.p.patient_row_ptr, h.p.row_ptr, h.p.col, h.K,
                                                                    words, counts, hist, h.J, h.rows, h.nnz);
}

// ------------------------------------------------------------------ basis (thread per patient)
// M_k rows by the de Boor triangle; Givens-QR of M_k into Rm (l x l); one-sided Jacobi on the
// rows of Rm gives sigma_j v_j; B_k column c (kept j) = v_j / sigma_j, so C_k = M_k B_k are the
// left singular vectors of M_k with sigma_j > tau * sigma_max (reading R-spline-4).
__global__ void k_basis(const int64_t* prp, const double* times, int64_t K, int l, int d, double tau, double* Bk,
                        int32_t* m, unsigned long long* diag) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  double Rm[kMaxFiberL * kMaxFiberL];
  double a[kMaxFiberL];
  double N[kMaxDeg + 1];
  for (int i = 0; i < l * kMaxFiberL; ++i) Rm[i] = 0.0;
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
    givens_insert(Rm, kMaxFiberL, a, l);
  }
  jacobi_rows(Rm, kMaxFiberL, l);
  double sig[kMaxFiberL], smax = 0.0;
  for (int j = 0; j < l; ++j) {
    double s = 0.0;
    for (int i = 0; i < l; ++i) s = fma(Rm[j * kMaxFiberL + i], Rm[j * kMaxFiberL + i], s);
    sig[j] = sqrt(s);
    smax = fmax(smax, sig[j]);
  }
  if (smax > 0.0) {  // rank-cut diagnostics (copa_stats)
    RatioDiag dg;
    for (int j = 0; j < l; ++j) dg.note(sig[j] / smax, sig[j] > tau * smax, tau);
    ratio_diag_commit(diag, D_BASIS_NEAR, dg);
  }
  // keep in descending sigma order (stable): selection by repeated max
  int used[kMaxFiberL];
  for (int j = 0; j < l; ++j) used[j] = 0;
  int c = 0;
  for (int it = 0; it < l; ++it) {
    int best = -1;
    for (int j = 0; j < l; ++j)
      if (!used[j] && (best < 0 || sig[j] > sig[best])) best = j;
    used[best] = 1;
    if (!(smax > 0.0) || !(sig[best] > tau * smax)) break;
    double inv2 = 1.0 / (sig[best] * sig[best]);
    for (int i = 0; i < l; ++i) B[i * l + c] = Rm[best * kMaxFiberL + i] * inv2;
    ++c;
  }
  for (int cc = c; cc < l; ++cc)
    for (int i = 0; i < l; ++i) B[i * l + cc] = 0.0;
  m[k] = c;
}

// Same computation with the l x l factor in registers (fixed l): Givens insert of each spline row
// (zero entries are skipped), round-robin one-sided Jacobi, kept columns placed by their rank in
// descending sigma (stable) — the order the selection loop above produces.
template <int L>
__global__ void __launch_bounds__(64) k_basis_reg(const int64_t* prp, const double* times, int64_t K, int d,
                                                  double tau, double* Bk, int32_t* m, unsigned long long* diag) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = k < K;
  int64_t r0 = 0, r1 = 0;
  double t1 = 0.0, tn = 0.0;
  if (live) {
    r0 = prp[k];
    r1 = prp[k + 1];
    t1 = times[r0];
    tn = times[r1 - 1];
  }
  const bool active = live && tn > t1;  // single visit: M_k = 0
  double Rm[L][L];
#pragma unroll
  for (int i = 0; i < L; ++i)
#pragma unroll
    for (int j = 0; j < L; ++j) Rm[i][j] = 0.0;
  for (int64_t i = r0; active && i < r1; ++i) {
    double N[kMaxDeg + 1];
    const int mu = spline_eval(times[i], t1, tn, L, d, N);
    double a[L];
#pragma unroll
    for (int b = 0; b < L; ++b) {
      const int r = b - (mu - d);
      a[b] = (r >= 0 && r <= d) ? N[r] : 0.0;
    }
    givens_insert_reg<L>(Rm, a);
  }
  jacobi_rows_reg<L>(Rm);  // warp-collective convergence vote: every lane takes part
  double sig[L], smax = 0.0;
#pragma unroll
  for (int j = 0; j < L; ++j) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i) s = fma(Rm[j][i], Rm[j][i], s);
    sig[j] = sqrt(s);
    smax = fmax(smax, sig[j]);
  }
  {  // rank-cut diagnostics (copa_stats), warp-collective
    RatioDiag dg;
    if (active && smax > 0.0)
#pragma unroll
      for (int j = 0; j < L; ++j) dg.note(sig[j] / smax, sig[j] > tau * smax, tau);
    ratio_diag_warp(diag, D_BASIS_NEAR, dg);
  }
  if (!live) return;
  double* B = Bk + k * (int64_t)L * L;
  int c = 0;
#pragma unroll
  for (int j = 0; j < L; ++j) {
    const bool keep = active && smax > 0.0 && sig[j] > tau * smax;
    c += keep ? 1 : 0;
  }
#pragma unroll
  for (int j = 0; j < L; ++j) {
    if (!(active && smax > 0.0 && sig[j] > tau * smax)) continue;
    int pos = 0;
#pragma unroll
    for (int q = 0; q < L; ++q) pos += (sig[q] > sig[j] || (q < j && sig[q] == sig[j])) ? 1 : 0;
    const double inv2 = 1.0 / (sig[j] * sig[j]);
#pragma unroll
    for (int i = 0; i < L; ++i) B[i * L + pos] = Rm[j][i] * inv2;
  }
  for (int cc = c; cc < L; ++cc)
#pragma unroll
    for (int i = 0; i < L; ++i) B[i * L + cc] = 0.0;
  m[k] = c;
}

void launch_basis(Handle& h) {
  if (h.K == 0) return;
  if (h.rowproj) { launch_basis_warp(h); return; }
  const unsigned blocks = (unsigned)((h.K + 63) / 64);
  if (h.l == 7) {
    k_basis_reg<7><<<blocks, 64, 0, h.stream>>>(h.p.patient_row_ptr, h.p.visit_time, h.K, h.d, h.o.basis_tol, h.Bk, h.m, h.diag);
    return;
  }
  if (h.l == 9) {
    k_basis_reg<9><<<blocks, 64, 0, h.stream>>>(h.p.patient_row_ptr, h.p.visit_time, h.K, h.d, h.o.basis_tol, h.Bk, h.m, h.diag);
    return;
  }
  k_basis<<<blocks, 64, 0, h.stream>>>(h.p.patient_row_ptr, h.p.visit_time, h.K, h.l, h.d, h.o.basis_tol, h.Bk, h.m, h.diag);
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
// Then the tiled stream's counts (k_fibers.cu): tcnt[g][k] = sum_w ceil(n_w / 8) tiles of the run and
// twoff[(g K + k) kWoS + w] = the tile offset of sub-range w inside it.
__global__ void k_count_groups(const int64_t* prp, const int64_t* rp, const int32_t* col, const int32_t* perm,
                               int64_t K, int words, int G, int64_t Jg, int W, int64_t Js, int32_t* gcnt /*[G][K]*/,
                               uint16_t* woff /*[G][K][8]*/, int32_t* tcnt /*[G][K]*/, uint16_t* twoff) {
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
    if (lane < G) {
      const uint16_t* wo = woff + ((int64_t)lane * K + k) * kWoS;
      uint16_t* tw = twoff + ((int64_t)lane * K + k) * kWoS;
      int acc = 0;
      for (int w = 0; w < W; ++w) {
        tw[w] = (uint16_t)acc;
        acc += (wo[w + 1] - wo[w] + 7) >> 3;
      }
      tw[W] = (uint16_t)acc;
      tcnt[(int64_t)lane * K + k] = acc;
    }
    __syncwarp();
  }
}

void launch_count_groups(Handle& h, int32_t* gcnt, int32_t* tcnt) {
  if (h.K == 0) return;
  const int words = (int)((h.Jl + 31) / 32);
  const int warps = 8;
  const size_t smem = (size_t)warps * words * (sizeof(unsigned) + sizeof(int));
  max_smem_attr<k_count_groups>(h, 200 * 1024);
  int64_t blocks = (h.K + warps - 1) / warps;
  if (blocks > h.sms * 16) blocks = h.sms * 16;
  k_count_groups<<<(unsigned)blocks, warps * 32, smem, h.stream>>>(h.p.patient_row_ptr, h.p.row_ptr, h.p.col, h.perm,
                                                                    h.K, words, h.sc_G, h.sc_Jg, h.sc_W, h.sc_Js, gcnt,
                                                                    h.woff, tcnt, h.twoff);
}

// ------------------------------------------------------------------ fibers: build X'_k = C_k^T X_k
// Warp per patient. The fibers of a patient are its distinct labels; the fiber with label j goes to
// stream g = j / Jg at gptr[g][k] + (rank(j) - rank(g Jg)), so every stream is sorted by label within
// each patient. The fibers are accumulated in shared memory, kBfWF ranks per window (patients with
// more distinct labels take several windows), then written out coalesced.
// Per window: rows in chunks (<= 32 rows, <= kBfNZ nonzeros): lane r evaluates the spline row
// C_k(i0 + r, :) = M_k(i, :) B_k into smem and the chunk's (rank, value) pairs are staged in smem;
// then rows one after the other, lanes over the row's (nonzero, a) pairs: a row's nonzeros have
// distinct labels, so the updates Fs(f, a) = fma(x, C(i, a), Fs(f, a)) of one row never collide, and
// every fiber entry is accumulated in ascending row order (deterministic).
constexpr int kBfWF = 128;   // fiber ranks per shared-memory window
constexpr int kBfWarps = 4;  // warps (patients in flight) per block
constexpr int kBfNZ = 256;   // staged nonzeros per row chunk

__host__ __device__ inline size_t bf_warp_doubles(int l, int words) {
  // Fs [WF l] | Cs [32 l] | xz [NZ] | rps [33] i64 | gd [kMaxGroups] i64 | fz [NZ] i32 | lab, dst [WF] i32 |
  // bits, pref [words]
  return (size_t)kBfWF * l + 32 * (size_t)l + kBfNZ + 33 + kMaxGroups + kBfNZ / 2 + kBfWF + (size_t)words;
}

__global__ void __launch_bounds__(32 * kBfWarps) k_build_fibers(
    const int64_t* prp, const int64_t* rp, const int32_t* col, const double* val, const double* times, int64_t K,
    int words, int l, int d, const double* Bk, const int32_t* m, const int64_t* gptr, int G, int Jg,
    const int32_t* perm, int32_t* fiber_col, double* fiber_val, int64_t kb, int64_t ke) {
  extern __shared__ double smem_bf[];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* Fs = smem_bf + (size_t)wib * bf_warp_doubles(l, words);
  double* Cs = Fs + (size_t)kBfWF * l;
  double* xz = Cs + 32 * l;
  int64_t* rps = (int64_t*)(xz + kBfNZ);
  int64_t* gd = rps + 33;
  int32_t* fz = (int32_t*)(gd + kMaxGroups);
  int32_t* lab = fz + kBfNZ;
  int32_t* grp = lab + kBfWF;
  unsigned* bits = (unsigned*)(grp + kBfWF);
  int* pref = (int*)(bits + words);
  const int64_t nwarps = (int64_t)gridDim.x * kBfWarps;
  const int64_t K1 = K + 1;
  for (int64_t k = kb + blockIdx.x * (int64_t)kBfWarps + wib; k < ke; k += nwarps) {  // patients [kb, ke)
    patient_label_bitmap(prp, rp, col, perm, k, words, bits, pref);
    const int nf = pref[words - 1] + __popc(bits[words - 1]);
    if (lane < G) gd[lane] = gptr[lane * K1 + k] - label_rank(bits, pref, words, (int64_t)lane * Jg);
    const int mk = m[k];
    // p / mk = umulhi(p, ceil(2^32 / mk)), exact for p < 2^24 (p < J mk here)
    const unsigned mmagic = mk > 0 ? (unsigned)((0x100000000ull + mk - 1) / mk) : 0u;
    const double* B = Bk + k * (int64_t)l * l;
    const int64_t r0 = prp[k], r1 = prp[k + 1];
    const double t1 = times[r0], tn = times[r1 - 1];
    for (int w0 = 0; w0 < nf; w0 += kBfWF) {
      const int nw = min(kBfWF, nf - w0);
      for (int x = lane; x < nw * l; x += 32) Fs[x] = 0.0;
      __syncwarp();
      int nr = 0;
      for (int64_t i0 = r0; mk > 0 && i0 < r1; i0 += nr) {
        const int n32 = (int)min((int64_t)32, r1 - i0);
        if (lane < n32) rps[lane] = rp[i0 + lane];
        if (lane == 0) rps[n32] = rp[i0 + n32];
        __syncwarp();
        // rows of this chunk: as many as fit kBfNZ staged nonzeros (at least one)
        const unsigned fit = __ballot_sync(FULL, lane < n32 && rps[lane + 1] - rps[0] <= kBfNZ);
        nr = fit ? 32 - __clz(fit) : 1;  // fit is a prefix of lanes (row_ptr is monotone)
        const int64_t e0 = rps[0];
        const int nz = (int)(rps[nr] - e0);
        const bool staged = nz <= kBfNZ;
        if (lane < nr) {
          double N[kMaxDeg + 1];
          const int mu = spline_eval(times[i0 + lane], t1, tn, l, d, N);
          for (int a = 0; a < mk; ++a) {
            double s = 0.0;
            for (int r = 0; r <= d; ++r) s = fma(N[r], B[(mu - d + r) * l + a], s);
            Cs[lane * l + a] = s;
          }
        }
        if (staged)
          for (int e = lane; e < nz; e += 32) {
            fz[e] = label_rank(bits, pref, words, perm[col[e0 + e]]) - w0;
            xz[e] = val[e0 + e];
          }
        __syncwarp();
        for (int r = 0; r < nr; ++r) {
          const int eb = (int)(rps[r] - e0), ne = (int)(rps[r + 1] - rps[r]);
          const double* C = Cs + r * l;
          for (int p = lane; p < ne * mk; p += 32) {  // lanes over the row's (nonzero, a) pairs
            const int e = (int)__umulhi((unsigned)p, mmagic);
            const int a = p - e * mk;
            int f;
            double x;
            if (staged) {
              f = fz[eb + e];
              x = xz[eb + e];
            } else {  // a single row longer than kBfNZ: straight from global memory
              f = label_rank(bits, pref, words, perm[col[e0 + eb + e]]) - w0;
              x = val[e0 + eb + e];
            }
            if (f >= 0 && f < nw) Fs[f * l + a] = fma(x, C[a], Fs[f * l + a]);
          }
          __syncwarp();
        }
      }
      // labels (and streams) of this window's ranks, then the window's fibers
      for (int wd = lane; wd < words; wd += 32) {
        unsigned b = bits[wd];
        int rk = pref[wd];
        if (rk >= w0 + nw || rk + __popc(b) <= w0) continue;
        while (b) {
          const int bit = __ffs(b) - 1;
          b &= b - 1;
          if (rk >= w0 && rk < w0 + nw) {
            const int j = wd * 32 + bit;
            lab[rk - w0] = j;
            grp[rk - w0] = j / Jg;
          }
          ++rk;
        }
      }
      __syncwarp();
      for (int f = lane; f < nw; f += 32) {
        const int64_t dst = gd[grp[f]] + w0 + f;
        fiber_col[dst] = lab[f];
        double* o = fiber_val + dst * l;
        for (int a = 0; a < l; ++a) o[a] = Fs[f * l + a];
      }
      __syncwarp();
    }
  }
}

void launch_build_fibers(Handle& h, int64_t kb, int64_t ke) {
  if (ke < 0) ke = h.K;
  if (ke <= kb) return;
  const int words = (int)((h.Jl + 31) / 32);  // bitmap over relabeled feature ids
  const size_t smem = (size_t)kBfWarps * bf_warp_doubles(h.l, words) * sizeof(double);
  max_smem_attr<k_build_fibers>(h);
  int64_t blocks = (ke - kb + kBfWarps - 1) / kBfWarps;
  if (blocks > h.sms * 32) blocks = h.sms * 32;
  k_build_fibers<<<(unsigned)blocks, kBfWarps * 32, smem, h.stream>>>(
      h.p.patient_row_ptr, h.p.row_ptr, h.p.col, h.p.val, h.p.visit_time, h.K, words, h.l, h.d, h.Bk, h.m, h.gptr,
      h.sc_G, (int)h.sc_Jg, h.perm, h.fiber_col, h.fiber_val, kb, ke);
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
