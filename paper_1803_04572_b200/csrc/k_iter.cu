// k_iter.cu — kernels of one COPA outer iteration (Alg.1 l.3-l.20 + FIT), FP64, sm_100a.
//
// Pass A   spmm    P'_k = X'_k V̄                 (smooth: fibers of X'_k = C_k^T X_k; plain: CSR rows)
//          polar   Q~_k = polar(P'_k S_k H̄^T)   (Givens QR of the tall side + one-sided Jacobi)
//          fh      F_H = sum_k Q~_k^T P'_k S_k   (= Y_(1)(W ⊙ V), Y never formed)          -> C1
// H-ADMM   admm_H  G_H, rho_H, chol, n_inner steps; then H̄^T H̄, G_W, rho_W, chol(G_W + rho_W I)
// Pass B   passB1  F_W(k,:) = colsum((Q~_k H̄) ∘ P'_k) (= Y_(3)(V ⊙ H)), W-row ADMM, N_k = Q~_k H̄ S_k
//          scatter F_V = sum_k X'_k^T N_k         (= Y_(2)(W ⊙ H))                        -> C2
// V-ADMM   admm_V  G_V, rho_V, chol, n_inner steps per row of V̄
// FIT      fit     E = normX - 2<F_V, V̄> + <sum_k N_k^T N_k, V̄^T V̄>
#include <algorithm>

#include "copa_internal.cuh"

namespace copa {

__device__ __forceinline__ int64_t patient_of(int64_t s, const int32_t* row_pat, int l) {
  return row_pat ? (int64_t)row_pat[s] : s / l;
}

// ------------------------------------------------------------------ pass A: SpMM
// Plain (no smoothness): P_k = X_k V̄, thread per (row, r).
__global__ void k_spmm_rows(const int64_t* rp, const int32_t* col, const double* val, int64_t rows, int R,
                            const double* V, double* Pp) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= rows * R) return;
  int64_t i = t / R;
  int r = (int)(t - i * R);
  double acc = 0.0;
  for (int64_t e = rp[i]; e < rp[i + 1]; ++e) acc = fma(val[e], V[(int64_t)col[e] * R + r], acc);
  Pp[t] = acc;
}

int launch_spmm(Handle& h) {
  if (h.K == 0) return 0;
  if (h.fib) {
    launch_spmm_fibers(h);
  } else if (h.rowproj) {
    return launch_rowproj_P(h);  // X_k V per visit row, then B_k^T (M_k^T P_k) (k_rowproj.cu)
  } else {
    int64_t n = h.rows * h.R;
    k_spmm_rows<<<(unsigned)((n + 255) / 256), 256, 0, h.stream>>>(h.p.row_ptr, h.p.col, h.p.val, h.rows, h.R, h.V,
                                                                   h.Pp);
  }
  return 1;
}

// ------------------------------------------------------------------ R x R reductions
// partial[b] = sum over block b's rows s of A(s,:)^T (B(s,:) * w(s,:)); then a fixed-order sum.
constexpr int kGramRows = 32;
__global__ void __launch_bounds__(256) k_gram(const double* A, const double* B, int64_t n, int R,
                                              const double* Wrows, const int32_t* row_pat, int lstride,
                                              double* partial) {
  __shared__ double As[kGramRows * kMaxR];
  __shared__ double Bs[kGramRows * kMaxR];
  const int RR = R * R;
  double acc[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) acc[u] = 0.0;
  int64_t per = (n + gridDim.x - 1) / gridDim.x;
  int64_t s0 = blockIdx.x * per, s1 = s0 + per;
  if (s1 > n) s1 = n;
  for (int64_t c0 = s0; c0 < s1; c0 += kGramRows) {
    int nr = (int)((s1 - c0) < kGramRows ? (s1 - c0) : kGramRows);
    for (int x = threadIdx.x; x < nr * R; x += blockDim.x) {
      int rr = x / R, c = x - rr * R;
      int64_t s = c0 + rr;
      As[rr * R + c] = A[s * R + c];
      double b = B[s * R + c];
      if (Wrows) b *= Wrows[patient_of(s, row_pat, lstride) * R + c];
      Bs[rr * R + c] = b;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      int p = threadIdx.x + 256 * u;
      if (p < RR) {
        int r = p / R, c = p - r * R;
        double s = acc[u];
        for (int rr = 0; rr < nr; ++rr) s = fma(As[rr * R + r], Bs[rr * R + c], s);
        acc[u] = s;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    int p = threadIdx.x + 256 * u;
    if (p < RR) partial[(int64_t)blockIdx.x * RR + p] = acc[u];
  }
}

// C[p] = sum_b partial[b][p] in a fixed order: 32 entries p per block (coalesced 256-byte rows),
// 32 groups of partials b = g, g + 32, ... summed by one thread each, then the 32 group sums in
// ascending g. (One thread per entry walking all nb partials took 23 us per call at nb = 1184: the
// plain path calls it four times per iteration.)
__global__ void __launch_bounds__(1024) k_reduce_partials(const double* __restrict__ partial, int nb, int RR,
                                                          double* __restrict__ C) {
  __shared__ double sm[32][33];
  const int px = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int p = blockIdx.x * 32 + px;
  double s = 0.0;
  if (p < RR) {
#pragma unroll 4
    for (int b = g; b < nb; b += 32) s += partial[(int64_t)b * RR + p];
  }
  sm[g][px] = s;
  __syncthreads();
  if (g == 0 && p < RR) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 32; ++q) t += sm[q][px];
    C[p] = t;
  }
}

// Tall-skinny Gram on the FP64 tensor cores (R <= 40): C = sum_s A(s,:)^T (B(s,:) * w(s,:)) as
// mma.sync m8n8k4 with M = r, N = c, K = 4 rows; warp per contiguous row range (multiple of 4 rows),
// all NT x NT output tiles in its accumulators, U k-steps of loads in flight; the per-warp partials
// are summed in a fixed order (k_reduce_partials): deterministic.
__device__ __forceinline__ void mma_f64(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int NT>
__global__ void __launch_bounds__(128) k_gram_mma(const double* __restrict__ A, const double* __restrict__ B, int64_t n,
                                                  int R, const double* __restrict__ Wrows,
                                                  const int32_t* __restrict__ row_pat, int lstride, int nwarps,
                                                  double* __restrict__ partial) {
  constexpr int U = 4;  // k-steps per load batch
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wid >= nwarps) return;
  const int64_t per = (((n + nwarps - 1) / nwarps) + 3) & ~(int64_t)3;
  const int64_t s0 = (int64_t)wid * per;
  const int64_t s1 = s0 + per < n ? s0 + per : n;
  double acc[NT][NT][2];
#pragma unroll
  for (int i = 0; i < NT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  bool cok[NT];
#pragma unroll
  for (int i = 0; i < NT; ++i) cok[i] = 8 * i + g < R;
  for (int64_t sb = s0; sb < s1; sb += 4 * U) {
    double a[U][NT], b[U][NT];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = sb + 4 * u + t;
      const bool rok = row < s1;
      const double* Ar = A + row * R;
      const double* Br = B + row * R;
      const double* Wr = (Wrows && rok) ? Wrows + patient_of(row, row_pat, lstride) * R : nullptr;
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        const int c = 8 * i + g;
        const bool ok = rok && cok[i];
        a[u][i] = ok ? Ar[c] : 0.0;
        double bv = ok ? Br[c] : 0.0;
        if (Wr && ok) bv *= Wr[c];
        b[u][i] = bv;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) mma_f64(acc[i][j][0], acc[i][j][1], a[u][i], b[u][j]);
  }
  double* out = partial + (int64_t)wid * R * R;
#pragma unroll
  for (int i = 0; i < NT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 8 * i + g, c = 8 * j + 2 * t + e;
        if (r < R && c < R) out[r * R + c] = acc[i][j][e];
      }
}

template <int NT>
static int gram_mma_inst(Handle& h, const double* A, const double* B, int64_t nrows, int wmode, double* C) {
  const int RR = h.R * h.R;
  int nw = 2 * kPartBlocks;  // partial holds 2 kPartBlocks R x R blocks
  const int64_t want = (nrows + 63) / 64;  // at least 64 rows per warp
  if (want < nw) nw = (int)(want > 0 ? want : 1);
  k_gram_mma<NT><<<(unsigned)((nw + 3) / 4), 128, 0, h.stream>>>(A, B, nrows, h.R, wmode ? h.W : nullptr,
                                                                  h.smooth ? nullptr : h.row_patient,
                                                                  h.smooth ? h.l : 1, nw, h.partial);
  k_reduce_partials<<<(RR + 31) / 32, 1024, 0, h.stream>>>(h.partial, nw, RR, C);
  return 2;
}

int launch_gram(Handle& h, const double* A, const double* B, int64_t nrows, int wmode, double* C) {
  // tall (state rows, patients): tensor cores; short (J rows of V̄): the block kernel below, whose
  // 32-row chunks spread over more SMs (measured: FIT phase 0.03 vs 0.04-0.05 ms at J = 300-1300)
  if (nrows >= (int64_t)1 << 16) switch ((h.R + 7) / 8) {
    case 1: return gram_mma_inst<1>(h, A, B, nrows, wmode, C);
    case 2: return gram_mma_inst<2>(h, A, B, nrows, wmode, C);
    case 3: return gram_mma_inst<3>(h, A, B, nrows, wmode, C);
    case 4: return gram_mma_inst<4>(h, A, B, nrows, wmode, C);
    case 5: return gram_mma_inst<5>(h, A, B, nrows, wmode, C);
    default: break;
  }
  int RR = h.R * h.R;
  int nb = kPartBlocks;
  if (nrows < (int64_t)nb * kGramRows) nb = (int)((nrows + kGramRows - 1) / kGramRows);
  if (nb < 1) nb = 1;
  k_gram<<<nb, 256, 0, h.stream>>>(A, B, nrows, h.R, wmode ? h.W : nullptr, h.smooth ? nullptr : h.row_patient,
                                   h.smooth ? h.l : 1, h.partial);
  k_reduce_partials<<<(RR + 31) / 32, 1024, 0, h.stream>>>(h.partial, nb, RR, C);
  return 2;
}

int launch_fh(Handle& h) { return launch_gram(h, h.Qt, h.Pp, h.S, 1, h.FH); }

// ------------------------------------------------------------------ small dense: chol + ADMM
// Cholesky of Ls (R x R in shared memory, lower, in place) by the whole block; returns 0 or 1 on failure.
__device__ int block_chol(double* Ls, int R, int* fail) {
  for (int j = 0; j < R; ++j) {
    if (threadIdx.x == 0) {
      double d = Ls[j * R + j];
      for (int k = 0; k < j; ++k) d -= Ls[j * R + k] * Ls[j * R + k];
      if (!(d > 0.0)) *fail = 1;
      Ls[j * R + j] = d > 0.0 ? sqrt(d) : 1.0;
    }
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < R; i += blockDim.x) {
      double v = Ls[i * R + j];
      for (int k = 0; k < j; ++k) v -= Ls[i * R + k] * Ls[j * R + k];
      Ls[i * R + j] = v / Ls[j * R + j];
    }
    __syncthreads();
  }
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) {
    int i = x / R, j = x - i * R;
    if (j > i) Ls[x] = 0.0;
  }
  __syncthreads();
  return *fail;
}

// Solves L L^T x = b in place; x[r] lives at x[r st] (per-thread vectors interleaved in shared
// memory: thread t's vector at base + t, stride st = number of threads, conflict-free).
__device__ __forceinline__ void chol_solve(const double* L, int R, double* x, int st = 1) {
  for (int i = 0; i < R; ++i) {
    double v = x[i * st];
    for (int k = 0; k < i; ++k) v -= L[i * R + k] * x[k * st];
    x[i * st] = v / L[i * R + i];
  }
  for (int i = R - 1; i >= 0; --i) {
    double v = x[i * st];
    for (int k = i + 1; k < R; ++k) v -= L[k * R + i] * x[k * st];
    x[i * st] = v / L[i * R + i];
  }
}

// Builds G = G1 ∘ G2 and rho (fixed or trace/R) into shared memory; returns rho (<= 0: degenerate).
__device__ double block_G_rho(const double* G1, const double* G2, int R, double rho_fixed, double* Gs) {
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) Gs[x] = G1[x] * G2[x];
  __syncthreads();
  if (rho_fixed > 0.0) return rho_fixed;
  double tr = 0.0;
  for (int i = 0; i < R; ++i) tr += Gs[i * R + i];
  return tr / R;
}

// One row of Alg.1 l.15-l.18, up to n_inner times: z = (f + rho (zb + d)) (G + rho I)^-1;
// zb = prox(z - d); d += zb - z; with tol > 0 the row stops early (reading R-inner-tol).
// f is read in place (global); zb, dd and the scratch z are the thread's interleaved shared-memory
// vectors (stride st). Returns the steps taken.
__device__ __forceinline__ int admm_row(const double* L, int R, const double* f, double* zb, double* dd, double* z,
                                        int st, double rho, int n_inner, int kind, double param, double tol) {
  int it = 0;
  while (it < n_inner) {
    for (int r = 0; r < R; ++r) z[r * st] = f[r] + rho * (zb[r * st] + dd[r * st]);
    chol_solve(L, R, z, st);
    RowResid res;
    for (int r = 0; r < R; ++r) {
      const double zr = z[r * st];
      double nb = prox(kind, param, rho, zr - dd[r * st]);
      res.add(nb, zr, zb[r * st]);
      dd[r * st] += nb - zr;
      zb[r * st] = nb;
    }
    ++it;
    if (res.done(tol)) break;
  }
  return it;
}

// H-mode (1 block) + the W-mode setup that depends only on the new H̄.
__global__ void __launch_bounds__(256) k_admm_H(int R, const double* FH, const double* VtV, const double* WtW,
                                                double rho_fixed, int n_inner, int kind, double param, double tol,
                                                double* H, double* DH, double* HtH, double* LW, double* GWi,
                                                double* scal, int* err, unsigned long long* steps) {
  extern __shared__ double dyn_smem[];
  double* Gs = dyn_smem;
  double* Ls = dyn_smem + R * R;
  __shared__ int fail;
  if (threadIdx.x == 0) {
    fail = 0;
    steps[0] = steps[1] = steps[2] = 0ull;  // this iteration's inner-step counters (H, W, V)
  }
  __syncthreads();
  double rho = block_G_rho(VtV, WtW, R, rho_fixed, Gs);
  if (!(rho > 0.0)) { if (threadIdx.x == 0) set_err(err, ERR_DEGEN); return; }
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) Ls[x] = Gs[x] + ((x / R == x % R) ? rho : 0.0);
  __syncthreads();
  if (block_chol(Ls, R, &fail)) { if (threadIdx.x == 0) set_err(err, ERR_CHOL); return; }
  double* vz = Ls + R * R;  // per-row vectors zb, dd, z: [3][R][R], row i interleaved at + i
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    double *zb = vz + i, *dd = vz + R * R + i, *z = vz + 2 * R * R + i;
    for (int r = 0; r < R; ++r) { zb[r * R] = H[i * R + r]; dd[r * R] = DH[i * R + r]; }
    const int st = admm_row(Ls, R, FH + i * R, zb, dd, z, R, rho, n_inner, kind, param, tol);
    atomicAdd(steps, (unsigned long long)st);
    for (int r = 0; r < R; ++r) { H[i * R + r] = zb[r * R]; DH[i * R + r] = dd[r * R]; }
  }
  __syncthreads();
  // H̄^T H̄ (new), then G_W = (H̄^T H̄) ∘ (V̄^T V̄), rho_W, chol -> LW
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) {
    int a = x / R, b = x - a * R;
    double s = 0.0;
    for (int i = 0; i < R; ++i) s = fma(H[i * R + a], H[i * R + b], s);
    Gs[x] = s;
    HtH[x] = s;
  }
  __syncthreads();
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) Gs[x] *= VtV[x];
  __syncthreads();
  double rho_w = rho_fixed;
  if (!(rho_w > 0.0)) {
    double tr = 0.0;
    for (int i = 0; i < R; ++i) tr += Gs[i * R + i];
    rho_w = tr / R;
  }
  if (!(rho_w > 0.0)) { if (threadIdx.x == 0) set_err(err, ERR_DEGEN); return; }
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) Ls[x] = Gs[x] + ((x / R == x % R) ? rho_w : 0.0);
  __syncthreads();
  if (block_chol(Ls, R, &fail)) { if (threadIdx.x == 0) set_err(err, ERR_CHOL); return; }
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) LW[x] = Ls[x];
  // (G_W + rho I)^-1 from the cached factor: column i solves L L^T x = e_i (used by the wide W pass)
  for (int i = threadIdx.x; i < R; i += blockDim.x) {
    double* x = vz + i;  // column i, interleaved (stride R)
    for (int r = 0; r < R; ++r) x[r * R] = r == i ? 1.0 : 0.0;
    chol_solve(Ls, R, x, R);
    for (int r = 0; r < R; ++r) GWi[r * R + i] = x[r * R];
  }
  if (threadIdx.x == 0) { scal[S_RHO_H] = rho; scal[S_RHO_W] = rho_w; }
}

// shared memory: G and its factor (2 R^2) + three interleaved R-vectors per row / thread
static size_t admm_smem(int R, int vecs) { return sizeof(double) * (2 * (size_t)R * R + 3 * (size_t)R * vecs); }
static int admm_V_threads(int R) { return R > 32 ? 64 : 128; }
constexpr int kAdmmSmemMax = (int)(sizeof(double) * 5 * kMaxR * kMaxR);  // both kernels at R = kMaxR

int launch_admm_H(Handle& h) {
  max_smem_attr<k_admm_H>(h, kAdmmSmemMax);
  k_admm_H<<<1, 256, admm_smem(h.R, h.R), h.stream>>>(h.R, h.FH, h.VtV, h.WtW, h.o.rho, h.o.admm_inner, h.o.on_H.kind,
                                                h.o.on_H.param, h.o.admm_tol, h.H, h.DH, h.HtH, h.LW, h.GWi, h.scal,
                                                h.err, h.steps);
  return 1;
}

// ------------------------------------------------------------------ pass B2: F_V scatter
// Fallback when no F_V slice fits in shared memory: warp per patient, FP64 global atomics.
__global__ void k_scatter_fibers(const int64_t* gptr, int G, const int32_t* fiber_col, const double* fiber_val,
                                 const int32_t* m, const int64_t* srow, int64_t K, int l, int R, const double* Nst,
                                 const int32_t* inv, double* FV) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t k = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); k < K; k += nwarps) {
    const int mk = m[k];
    const double* N = Nst + srow[k] * R;
    double n0[kMaxFiberL], n1[kMaxFiberL];
    const int r0 = lane, r1 = lane + 32;
    for (int a = 0; a < kMaxFiberL; ++a) {
      n0[a] = (a < mk && r0 < R) ? N[a * R + r0] : 0.0;
      n1[a] = (a < mk && r1 < R) ? N[a * R + r1] : 0.0;
    }
    for (int g = 0; g < G; ++g)
    for (int64_t f = gptr[g * (K + 1) + k]; f < gptr[g * (K + 1) + k + 1]; ++f) {
      const int64_t j = inv[fiber_col[f]];  // fibers carry relabeled feature ids
      const double* xv = fiber_val + f * l;
      double s0 = 0.0, s1 = 0.0;
      for (int a = 0; a < mk; ++a) {
        double x = xv[a];
        s0 = fma(x, n0[a], s0);
        s1 = fma(x, n1[a], s1);
      }
      if (r0 < R) atomicAdd(&FV[j * R + r0], s0);
      if (r1 < R) atomicAdd(&FV[j * R + r1], s1);
    }
  }
}

int launch_scatter(Handle& h) {
  if (!h.smooth) return launch_scatter_csc(h, h.Nst);  // deterministic gather over the CSC copy (k_plain.cu)
  if (h.rowproj) return launch_rowproj_N(h) + launch_scatter_csc(h, h.Nrow);  // C_k N'_k per row, then gather
  cudaMemsetAsync(h.FV, 0, sizeof(double) * (size_t)(h.J * h.R), h.stream);
  if (h.K == 0) return 0;
  if (scatter_smem_ok(h)) return launch_scatter_fibers(h);
  // no F_V slice fits in shared memory (J R too large): FP64-atomic fallback (order-dependent rounding)
  int64_t blocks = (h.K + 7) / 8;
  if (blocks > h.sms * 32) blocks = h.sms * 32;
  k_scatter_fibers<<<(unsigned)blocks, 256, 0, h.stream>>>(h.gptr, h.sc_G, h.fiber_col, h.fiber_val, h.m, h.srow,
                                                           h.K, h.l, h.R, h.Nst, h.inv, h.FV);
  return 1;
}

// ------------------------------------------------------------------ V-mode ADMM (rows independent)
__global__ void __launch_bounds__(128) k_admm_V(int64_t J, int R, const double* FV, const double* HtH,
                                                const double* WtW, double rho_fixed, int n_inner, int kind,
                                                double param, double tol, double* V, double* DV, double* scal,
                                                int* err, unsigned long long* steps) {
  extern __shared__ double dyn_smem[];
  double* Gs = dyn_smem;
  double* Ls = dyn_smem + R * R;
  __shared__ int fail;
  if (threadIdx.x == 0) fail = 0;
  __syncthreads();
  double rho = block_G_rho(HtH, WtW, R, rho_fixed, Gs);
  if (!(rho > 0.0)) { if (threadIdx.x == 0 && blockIdx.x == 0) set_err(err, ERR_DEGEN); return; }
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) Ls[x] = Gs[x] + ((x / R == x % R) ? rho : 0.0);
  __syncthreads();
  if (block_chol(Ls, R, &fail)) { if (threadIdx.x == 0 && blockIdx.x == 0) set_err(err, ERR_CHOL); return; }
  if (blockIdx.x == 0 && threadIdx.x == 0) scal[S_RHO_V] = rho;
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int st = 0;
  if (j < J) {
    const int S = blockDim.x;  // per-thread vectors zb, dd, z interleaved (stride = threads)
    double *zb = Ls + R * R + threadIdx.x, *dd = zb + R * S, *z = zb + 2 * R * S;
    for (int r = 0; r < R; ++r) { zb[r * S] = V[j * R + r]; dd[r * S] = DV[j * R + r]; }
    st = admm_row(Ls, R, FV + j * R, zb, dd, z, S, rho, n_inner, kind, param, tol);
    for (int r = 0; r < R; ++r) { V[j * R + r] = zb[r * S]; DV[j * R + r] = dd[r * S]; }
  }
  steps_warp(steps + 2, st);
}

// Zero entries of V̄ (SPARSITY), into steps[3].
__global__ void k_count_zeros(const double* V, int64_t n, unsigned long long* out) {
  int c = 0;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
    c += V[x] == 0.0;
  steps_warp(out, c);
}

void launch_count_zeros(Handle& h) {
  cudaMemsetAsync(h.steps + 3, 0, sizeof(unsigned long long), h.stream);
  const int64_t n = h.J * h.R;
  k_count_zeros<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, h.stream>>>(h.V, n, h.steps + 3);
}

int launch_admm_V(Handle& h) {
  max_smem_attr<k_admm_V>(h, kAdmmSmemMax);
  const int nt = admm_V_threads(h.R);
  k_admm_V<<<(unsigned)((h.J + nt - 1) / nt), nt, admm_smem(h.R, nt), h.stream>>>(h.J, h.R, h.FV, h.HtH, h.WtW, h.o.rho,
                                                                 h.o.admm_inner, h.o.on_V.kind, h.o.on_V.param,
                                                                 h.o.admm_tol, h.V, h.DV, h.scal, h.err, h.steps);
  return 1;
}

// ------------------------------------------------------------------ FIT
__global__ void k_fit(int64_t JR, int RR, const double* FV, const double* V, const double* M, const double* VtV,
                      double* scal, int* err) {
  __shared__ double red[2][256];
  double c = 0.0, q = 0.0;
  for (int64_t x = threadIdx.x; x < JR; x += blockDim.x) c = fma(FV[x], V[x], c);
  for (int x = threadIdx.x; x < RR; x += blockDim.x) q = fma(M[x], VtV[x], q);
  red[0][threadIdx.x] = c;
  red[1][threadIdx.x] = q;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) { red[0][threadIdx.x] += red[0][threadIdx.x + o]; red[1][threadIdx.x] += red[1][threadIdx.x + o]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double normX = scal[S_NORMX];
    double E = normX - 2.0 * red[0][0] + red[1][0];
    double fit = 1.0 - E / normX;
    scal[S_CROSS] = red[0][0];
    scal[S_QUAD] = red[1][0];
    scal[S_E] = E;
    scal[S_FIT] = fit;
    if (!isfinite(fit)) set_err(err, ERR_NONFINITE);
  }
}

int launch_fit(Handle& h) {
  int n = launch_gram(h, h.V, h.V, h.J, 0, h.VtV);
  k_fit<<<1, 256, 0, h.stream>>>(h.J * h.R, h.R * h.R, h.FV, h.V, h.M, h.VtV, h.scal, h.err);
  return n + 1;
}

// ------------------------------------------------------------------ U_k = C_k Q~_k H̄ (output)
__global__ void k_U(const int64_t* prp, const double* times, int64_t k0, int64_t k1, int l, int d, const double* Bk,
                    const int32_t* m, const int64_t* srow, int R, const double* Qt, const double* H, double* U) {
  int64_t k = k0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= k1) return;
  U -= prp[k0] * R;  // row i of the shard -> U[(i - prp[k0]) R]
  int64_t r0 = prp[k], r1 = prp[k + 1];
  const int mk = m[k];
  const double* Q = Qt + srow[k] * R;
  for (int64_t i = r0; i < r1; ++i) {
    double c[kMaxL];
    int mrows;
    if (l > 0) {
      for (int a = 0; a < kMaxL; ++a) c[a] = 0.0;
      if (mk > 0) {
        double N[kMaxDeg + 1];
        double t1 = times[r0], tn = times[r1 - 1];
        int mu = spline_eval(times[i], t1, tn, l, d, N);
        const double* B = Bk + k * (int64_t)l * l;
        for (int a = 0; a < mk; ++a) {
          double s = 0.0;
          for (int r = 0; r <= d; ++r) s = fma(N[r], B[(mu - d + r) * l + a], s);
          c[a] = s;
        }
      }
      mrows = mk;
    } else {
      mrows = 0;
    }
    for (int s = 0; s < R; ++s) {
      double acc = 0.0;
      if (l > 0) {
        for (int a = 0; a < mrows; ++a) {
          double qh = 0.0;
          for (int x = 0; x < R; ++x) qh = fma(Q[a * R + x], H[x * R + s], qh);
          acc = fma(c[a], qh, acc);
        }
      } else {
        for (int x = 0; x < R; ++x) acc = fma(Q[(i - r0) * R + x], H[x * R + s], acc);
      }
      U[i * R + s] = acc;
    }
  }
}

void launch_U(Handle& h, double* U, int64_t k0, int64_t k1) {
  if (k1 <= k0) return;
  k_U<<<(unsigned)((k1 - k0 + 127) / 128), 128, 0, h.stream>>>(h.p.patient_row_ptr, h.p.visit_time, k0, k1,
                                                               h.smooth ? h.l : 0, h.d, h.Bk, h.m, h.srow, h.R, h.Qt,
                                                               h.H, U);
}

}  // namespace copa
