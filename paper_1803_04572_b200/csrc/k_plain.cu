// k_plain.cu — the general ("plain") path of one outer iteration, FP64, sm_100a: no smoothness, or
// smoothness outside the wide kernels' range (l >= R or l > 12). Per-patient state rows: m_k rows
// of P'_k, Q~_k, N_k (m_k = I_k without smoothness). Any R <= 64.
//
//   polar_warp   warp per patient: A_k = P'_k S_k H̄^T built 32 rows at a time (lane per row);
//                Givens QR of the tall side into an upper-triangular Rf (q x q, q = min(m_k, R),
//                shared memory); one-sided Jacobi on the rows of Rf with one lane per disjoint row
//                pair (round-robin ordering); Q~_k = A K (lane per row) or K A with K = V Σ^-1 V^T on the
//                numerical range (the partial isometry U_r V_r^T, reading R-polar-2/3) (Alg.1 l.4-5)
//   passB_warp   warp per patient, lanes over r: T = Q~_k H̄, F_W(k,:) = colsum(T ∘ P'_k), the W-row ADMM
//                with (G_W + rho I)^-1 (one lane per output column), N_k = T S_k      (l.12-19, W mode)
//   scatter_csc  F_V = sum_k X_k^T N_k as a gather over a feature-major (CSC) copy of X built at init:
//                F_V(j,:) = sum over column j's entries x_e N(row_e, :), warp per fixed-size chunk of
//                a column, chunk partials summed in a fixed order (deterministic, no atomics)
//                                                                                   (l.12, V mode)
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "copa_internal.cuh"
#include "k_dense.cuh"  // register Givens / Jacobi helpers

namespace copa {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kPlainWarps = 4;  // warps per block of the warp-per-patient kernels

__host__ __device__ inline int odd_ld(int n) { return n | 1; }

// Shared memory (doubles) per warp of k_polar_warp: Rf (R x LD) + A buffer (R x LD).
__host__ __device__ inline size_t polar_warp_per_warp(int R) { return 2 * (size_t)R * odd_ld(R); }

__device__ __forceinline__ double lane_pick(double v0, double v1, int j) {
  return __shfl_sync(kFull, j < 32 ? v0 : v1, j & 31);
}

// Givens insert of the vector v (length q, lane t holds v[t] in v0 and v[t + 32] in v1) into the
// upper-triangular Rf (q x q, stride LD): Rf^T Rf accumulates v v^T, no Gram matrix is formed.
// Lane t owns column t (and t + 32) of Rf above the diagonal; the diagonal lives in registers
// (lane j holds Rf(j, j) in d0, Rf(j + 32, j + 32) in d1), so no two lanes touch the same word and
// the insertion needs no barrier; warp_givens_flush() stores the diagonal afterwards.
__device__ __forceinline__ void warp_givens_insert(double* Rf, int LD, int q, double v0, double v1, double& d0,
                                                   double& d1) {
  const int lane = threadIdx.x & 31;
  const bool own0 = lane < q, own1 = lane + 32 < q;
  for (int j = 0; j < q; ++j) {
    const double x0 = (own0 && lane > j) ? Rf[j * LD + lane] : 0.0;
    const double x1 = (own1 && lane + 32 > j) ? Rf[j * LD + lane + 32] : 0.0;
    const double vj = lane_pick(v0, v1, j);
    const double r = lane_pick(d0, d1, j);
    if (vj != 0.0) {
      const double n2 = fma(r, r, vj * vj);
      const double inv = rsqrt(n2);
      const double cs = r * inv, sn = vj * inv;
      if (own0 && lane > j) {
        Rf[j * LD + lane] = fma(cs, x0, sn * v0);
        v0 = fma(cs, v0, -sn * x0);
      }
      if (own1 && lane + 32 > j) {
        Rf[j * LD + lane + 32] = fma(cs, x1, sn * v1);
        v1 = fma(cs, v1, -sn * x1);
      }
      if (lane == (j & 31)) {
        if (j < 32) d0 = n2 * inv;
        else d1 = n2 * inv;
      }
    }
  }
}

__device__ __forceinline__ void warp_givens_flush(double* Rf, int LD, int q, double d0, double d1) {
  const int lane = threadIdx.x & 31;
  if (lane < q) Rf[lane * LD + lane] = d0;
  if (lane + 32 < q) Rf[(lane + 32) * LD + lane + 32] = d1;
  __syncwarp();
}

// One-sided Jacobi on the q rows of Rf until mutually orthogonal: round-robin (tournament)
// ordering, lane i rotates the i-th disjoint pair of a round with jacobi_rot() (copa_internal.cuh).
__device__ __forceinline__ void warp_jacobi_rows(double* Rf, int LD, int q) {
  const int lane = threadIdx.x & 31;
  const int N = (q & 1) ? q + 1 : q;
  const double eps = 2.220446049250313e-16 * (double)q;
  const double tol2 = eps * eps;
  double tr = 0.0;  // trace of the Gram (invariant): residue-row threshold (kJacobiNegl2)
  for (int x = lane; x < q; x += 32)
    for (int y = 0; y < q; ++y) tr = fma(Rf[x * LD + y], Rf[x * LD + y], tr);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(kFull, tr, o);
  const double negl = kJacobiNegl2 * tr;
  for (int sweep = 0; sweep < 40; ++sweep) {
    int rotated = 0, big = 0;
    for (int rd = 0; rd < N - 1; ++rd) {
      const int i = lane;
      if (i < N / 2) {
        const int p = i == 0 ? 0 : 1 + (i - 1 + rd) % (N - 1);
        const int r = 1 + (N - 2 - i + rd) % (N - 1);
        if (p < q && r < q) {
          double* xp = Rf + p * LD;
          double* xr = Rf + r * LD;
          double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll 8
          for (int x = 0; x < q; ++x) {  // unrolled: the shared-memory loads of 8 elements in flight
            const double u = xp[x], v = xr[x];
            a = fma(u, u, a);
            b = fma(v, v, b);
            c = fma(u, v, c);
          }
          if (a > negl && b > negl && c * c > tol2 * (a * b)) {
            rotated = 1;
            big |= c * c > kJacobiDoneCos2 * (a * b);
            double cs, sn;
            jacobi_rot(a, b, c, cs, sn);
#pragma unroll 8
            for (int x = 0; x < q; ++x) {
              const double u = xp[x], v = xr[x];
              xp[x] = fma(cs, u, -sn * v);
              xr[x] = fma(sn, u, cs * v);
            }
          }
        }
      }
      __syncwarp();
    }
    if (__all_sync(kFull, rotated == 0 || !big)) break;  // as jacobi_rows_reg
  }
}

// Rows a0 .. a0 + na - 1 of A_k = P'_k S_k H̄^T into Ab (row i at Ab[i LD]), lane i computing row
// a0 + i in blocks of 8 columns: the same products and the same r-ascending FMA chains as a_row,
// 32 rows at a time instead of one row per R shuffles.
__device__ __forceinline__ void a_rows_lane(const double* __restrict__ P, int a0, int na, int R, int LD, double w0,
                                            double w1, const double* __restrict__ HT, double* Ab) {
  const int lane = threadIdx.x & 31;
  const bool live = lane < na;
  const double* Pr = P + (int64_t)(a0 + (live ? lane : 0)) * R;
  for (int sb = 0; sb < R; sb += 8) {
    double acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0;
    for (int r = 0; r < R; ++r) {
      const double wr = lane_pick(w0, w1, r);
      const double pw = live ? Pr[r] * wr : 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (sb + e < R) acc[e] = fma(pw, HT[r * R + sb + e], acc[e]);
    }
    if (live) {
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (sb + e < R) Ab[lane * LD + sb + e] = acc[e];
    }
  }
}

template <int RB>  // bound on R (register array of the Q~ rows); small R: occupancy of the general kernel
__global__ void __launch_bounds__(32 * kPlainWarps, RB <= 16 ? 8 : (RB <= 32 ? 4 : 1)) k_polar_warp(const int32_t* __restrict__ m,
                                                                 const int64_t* __restrict__ srow, int64_t K, int R,
                                                                 const double* __restrict__ Pp,
                                                                 const double* __restrict__ Wg,
                                                                 const double* __restrict__ HT, double tau,
                                                                 double* __restrict__ Qt, int32_t* __restrict__ rank,
                                                                 unsigned long long* __restrict__ diag) {
  extern __shared__ double smp[];
  const int LD = odd_ld(R);  // HT: H̄^T in global memory (L1-resident), HT[r R + s] = H̄(s, r)
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nwb = blockDim.x >> 5;  // warps of this block (fewer at large R: shared memory)
  double* Rf = smp + (size_t)wib * polar_warp_per_warp(R);
  double* Ab = Rf + (size_t)R * LD;
  const int64_t nw = (int64_t)gridDim.x * nwb;
  for (int64_t k = blockIdx.x * (int64_t)nwb + wib; k < K; k += nw) {
    const int mk = m[k];
    if (mk == 0) {
      if (lane == 0) rank[k] = 0;
      continue;
    }
    const double* P = Pp + srow[k] * R;
    double* Q = Qt + srow[k] * R;
    const double w0 = lane < R ? Wg[k * R + lane] : 0.0, w1 = lane + 32 < R ? Wg[k * R + lane + 32] : 0.0;
    const bool tall = mk >= R;
    const int q = tall ? R : mk;
    for (int x = lane; x < q * LD; x += 32) Rf[x] = 0.0;
    __syncwarp();
    double dg0 = 0.0, dg1 = 0.0;  // diagonal of Rf (see warp_givens_insert)
    // ---- QR of the tall side: rows of A (tall) or columns of A (wide) inserted one by one
    const int CR = R < 32 ? R : 32;  // rows of A per chunk in Ab (R x LD doubles)
    if (tall) {
      for (int a0 = 0; a0 < mk; a0 += CR) {
        const int na = mk - a0 < CR ? mk - a0 : CR;
        __syncwarp();
        a_rows_lane(P, a0, na, R, LD, w0, w1, HT, Ab);
        __syncwarp();
        for (int i = 0; i < na; ++i) {
          const double v0 = lane < R ? Ab[i * LD + lane] : 0.0;
          const double v1 = lane + 32 < R ? Ab[i * LD + lane + 32] : 0.0;
          warp_givens_insert(Rf, LD, q, v0, v1, dg0, dg1);
        }
      }
    } else {
      for (int a0 = 0; a0 < mk; a0 += 32)  // A (m x R) into Ab, row a at Ab[a LD]
        a_rows_lane(P, a0, mk - a0 < 32 ? mk - a0 : 32, R, LD, w0, w1, HT, Ab + a0 * LD);
      __syncwarp();
      for (int s = 0; s < R; ++s) {
        const double v0 = lane < mk ? Ab[lane * LD + s] : 0.0;
        const double v1 = lane + 32 < mk ? Ab[(lane + 32) * LD + s] : 0.0;
        warp_givens_insert(Rf, LD, q, v0, v1, dg0, dg1);
      }
    }
    warp_givens_flush(Rf, LD, q, dg0, dg1);
    // ---- SVD of the q x q factor: rows of Rf -> sigma_j v_j^T
    warp_jacobi_rows(Rf, LD, q);
    double n0 = 0.0, n1 = 0.0;  // sigma_j^2 of rows j = lane, lane + 32
    if (lane < q)
      for (int x = 0; x < q; ++x) n0 = fma(Rf[lane * LD + x], Rf[lane * LD + x], n0);
    if (lane + 32 < q)
      for (int x = 0; x < q; ++x) n1 = fma(Rf[(lane + 32) * LD + x], Rf[(lane + 32) * LD + x], n1);
    double smax = fmax(n0, n1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) smax = fmax(smax, __shfl_xor_sync(kFull, smax, o));
    smax = sqrt(smax);
    const double sg0 = sqrt(n0), sg1 = sqrt(n1);
    const bool keep0 = lane < q && smax > 0.0 && sg0 > tau * smax;
    const bool keep1 = lane + 32 < q && smax > 0.0 && sg1 > tau * smax;
    {
      RatioDiag dg;
      if (smax > 0.0) {
        if (lane < q) dg.note(sg0 / smax, keep0, tau);
        if (lane + 32 < q) dg.note(sg1 / smax, keep1, tau);
      }
      ratio_diag_warp(diag, D_POLAR_NEAR, dg);
    }
    const int rk = __popc(__ballot_sync(kFull, keep0)) + __popc(__ballot_sync(kFull, keep1));
    if (lane == 0) rank[k] = rk;
    // u_j = v_j / sqrt(sigma_j) (kept) or 0: K = sum_j u_j u_j^T = V Σ^-1 V^T on the range
    {
      const double c0 = keep0 ? 1.0 / (sg0 * sqrt(sg0)) : 0.0;
      const double c1 = keep1 ? 1.0 / (sg1 * sqrt(sg1)) : 0.0;
      if (lane < q)
        for (int x = 0; x < q; ++x) Rf[lane * LD + x] *= c0;
      if (lane + 32 < q)
        for (int x = 0; x < q; ++x) Rf[(lane + 32) * LD + x] *= c1;
    }
    __syncwarp();
    if (tall) {
      // Q~(a, :) = A(a, :) K = sum_j (A(a, :) . u_j) u_j^T: lane i takes row a0 + i of the chunk
      // (d_j in registers, x and j ascending as before); the rows leave through Ab, coalesced
      for (int a0 = 0; a0 < mk; a0 += CR) {
        const int na = mk - a0 < CR ? mk - a0 : CR;
        __syncwarp();
        a_rows_lane(P, a0, na, R, LD, w0, w1, HT, Ab);
        __syncwarp();
        if (lane < na) {
          double* vr = Ab + lane * LD;
          double d[RB];  // d_j = A(a, :) . u_j, four independent chains at a time
#pragma unroll
          for (int jb = 0; jb < RB; jb += 4) {
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            if (jb < q)
              for (int x = 0; x < q; ++x) {
                const double v = vr[x];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (jb + e < q) acc[e] = fma(v, Rf[(jb + e) * LD + x], acc[e]);
              }
#pragma unroll
            for (int e = 0; e < 4; ++e) d[jb + e] = acc[e];
          }
          for (int s0 = 0; s0 < R; s0 += 4) {  // Q~(a, s) = sum_j d_j u_j(s), four columns at a time
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int j = 0; j < RB; ++j)
              if (j < q) {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (s0 + e < R) acc[e] = fma(d[j], Rf[j * LD + s0 + e], acc[e]);
              }
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (s0 + e < R) vr[s0 + e] = acc[e];
          }
        }
        __syncwarp();
        for (int x = lane; x < na * R; x += 32) {
          const int i = x / R, s2 = x - i * R;
          Q[(int64_t)(a0 + i) * R + s2] = Ab[i * LD + s2];
        }
      }
    } else {
      // Q~(:, s) = K A(:, s) = sum_j u_j (u_j . A(:, s)), column by column in place of A
      for (int s = 0; s < R; ++s) {
        double e0 = 0.0, e1 = 0.0;
        if (lane < q)
          for (int a = 0; a < mk; ++a) e0 = fma(Rf[lane * LD + a], Ab[a * LD + s], e0);
        if (lane + 32 < q)
          for (int a = 0; a < mk; ++a) e1 = fma(Rf[(lane + 32) * LD + a], Ab[a * LD + s], e1);
        double q0 = 0.0, q1 = 0.0;
        for (int j = 0; j < q; ++j) {
          const double ej = lane_pick(e0, e1, j);
          if (lane < mk) q0 = fma(ej, Rf[j * LD + lane], q0);
          if (lane + 32 < mk) q1 = fma(ej, Rf[j * LD + lane + 32], q1);
        }
        __syncwarp();
        if (lane < mk) Ab[lane * LD + s] = q0;
        if (lane + 32 < mk) Ab[(lane + 32) * LD + s] = q1;
        __syncwarp();
      }
      for (int a = 0; a < mk; ++a)
        for (int s = lane; s < R; s += 32) Q[(int64_t)a * R + s] = Ab[a * LD + s];
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ polar, thread per patient (R <= 10)
// Small ranks: the q x q algebra of one patient fits in registers (L = compile-time bound on R, rows
// and columns beyond R or m_k are zero), so one thread runs one patient's QR, Jacobi and Q~ = A K /
// K A with the register helpers of the smooth path (k_dense.cuh: givens_insert_reg, jacobi_rows_reg).
// Same algebra as k_polar_warp; A's rows (tall) or columns (wide) are recomputed from P'_k (L1).
template <int L>
__global__ void __launch_bounds__(128) k_polar_thread(const int32_t* __restrict__ m, const int64_t* __restrict__ srow,
                                                      int64_t K, int R, const double* __restrict__ Pp,
                                                      const double* __restrict__ Wg, const double* __restrict__ Hg,
                                                      double tau, double* __restrict__ Qt, int32_t* __restrict__ rank,
                                                      unsigned long long* __restrict__ diag,
                                                      const int32_t* __restrict__ order) {
  __shared__ double Hs[L * L];  // H̄ zero-padded to L x L: Hs[s L + r] = H̄(s, r)
  for (int x = threadIdx.x; x < L * L; x += blockDim.x) {
    const int s = x / L, r = x - s * L;
    Hs[x] = (s < R && r < R) ? Hg[s * R + r] : 0.0;
  }
  __syncthreads();
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = t < K;
  const int64_t k = live ? (int64_t)order[t] : 0;  // patients in order of m_k: a warp's 32 loops have similar lengths
  const int mk = live ? m[k] : 0;
  const bool tall = mk >= R;
  const double* P = live ? Pp + srow[k] * R : Pp;
  double w[L];
#pragma unroll
  for (int r = 0; r < L; ++r) w[r] = (live && r < R) ? Wg[k * R + r] : 0.0;
  // A(a, s) = sum_r P'(a, r) w(r) H̄(s, r)
  auto a_row = [&](int a, double (&v)[L]) {
    double pw[L];
#pragma unroll
    for (int r = 0; r < L; ++r) pw[r] = r < R ? P[(int64_t)a * R + r] * w[r] : 0.0;
#pragma unroll
    for (int s = 0; s < L; ++s) {
      double acc = 0.0;
#pragma unroll
      for (int r = 0; r < L; ++r) acc = fma(pw[r], Hs[s * L + r], acc);
      v[s] = acc;
    }
  };
  auto a_col = [&](int s, double (&v)[L]) {  // column s of A (m_k < L entries, zero beyond)
#pragma unroll
    for (int a = 0; a < L; ++a) {
      double acc = 0.0;
      if (a < mk)
#pragma unroll
        for (int r = 0; r < L; ++r)
          if (r < R) acc = fma(P[(int64_t)a * R + r] * w[r], Hs[s * L + r], acc);
      v[a] = acc;
    }
  };
  double Rf[L][L];
#pragma unroll
  for (int i = 0; i < L; ++i)
#pragma unroll
    for (int j = 0; j < L; ++j) Rf[i][j] = 0.0;
  if (tall) {
    for (int a = 0; a < mk; ++a) {
      double v[L];
      a_row(a, v);
      givens_insert_reg<L>(Rf, v);
    }
  } else if (mk > 0) {
    for (int s = 0; s < R; ++s) {
      double v[L];
      a_col(s, v);
      givens_insert_reg<L>(Rf, v);
    }
  }
  jacobi_rows_reg<L>(Rf);  // warp-collective convergence vote: every lane takes part
  double sg[L], smax = 0.0;
#pragma unroll
  for (int j = 0; j < L; ++j) {
    double s2 = 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i) s2 = fma(Rf[j][i], Rf[j][i], s2);
    sg[j] = sqrt(s2);
    smax = fmax(smax, sg[j]);
  }
  const int q = tall ? R : mk;
  int rk = 0;
  RatioDiag dg;
#pragma unroll
  for (int j = 0; j < L; ++j) {
    const bool keep = smax > 0.0 && sg[j] > tau * smax;
    if (smax > 0.0 && j < q) dg.note(sg[j] / smax, keep, tau);
    rk += keep ? 1 : 0;
    const double c = keep ? 1.0 / (sg[j] * sqrt(sg[j])) : 0.0;  // u_j = v_j / sqrt(sigma_j)
#pragma unroll
    for (int i = 0; i < L; ++i) Rf[j][i] *= c;
  }
  ratio_diag_warp(diag, D_POLAR_NEAR, dg);
  if (!live) return;
  rank[k] = mk > 0 ? rk : 0;
  double* Q = Qt + srow[k] * R;
  if (tall) {  // Q~(a, :) = sum_j (A(a, :) . u_j) u_j^T
    for (int a = 0; a < mk; ++a) {
      double v[L], d[L];
      a_row(a, v);
#pragma unroll
      for (int j = 0; j < L; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int x = 0; x < L; ++x) acc = fma(v[x], Rf[j][x], acc);
        d[j] = acc;
      }
#pragma unroll
      for (int s = 0; s < L; ++s) {
        if (s < R) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < L; ++j) acc = fma(d[j], Rf[j][s], acc);
          Q[(int64_t)a * R + s] = acc;
        }
      }
    }
  } else if (mk > 0) {  // Q~(:, s) = sum_j u_j (u_j . A(:, s))
    for (int s = 0; s < R; ++s) {
      double v[L], e[L];
      a_col(s, v);
#pragma unroll
      for (int j = 0; j < L; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < L; ++a) acc = fma(Rf[j][a], v[a], acc);
        e[j] = acc;
      }
#pragma unroll
      for (int a = 0; a < L; ++a) {
        if (a < mk) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < L; ++j) acc = fma(e[j], Rf[j][a], acc);
          Q[(int64_t)a * R + s] = acc;
        }
      }
    }
  }
}

template <int L>
static void polar_thread_inst(Handle& h) {
  const unsigned blocks = (unsigned)((h.K + 127) / 128);
  k_polar_thread<L><<<blocks, 128, 0, h.stream>>>(h.m, h.srow, h.K, h.R, h.Pp, h.W, h.H, h.o.rank_tol, h.Qt, h.rank,
                                                  h.diag, h.porder);
}

bool polar_thread_ok(const Handle& h) { return h.R <= 10; }

// Patient order of the thread-per-patient polar: ascending m_k (stable), from the device m (init).
int plan_polar_order(Handle& h) {
  if (h.K == 0 || !polar_thread_ok(h)) return 0;
  std::vector<int32_t> m((size_t)h.K), order((size_t)h.K);
  if (cudaMemcpyAsync(m.data(), h.m, sizeof(int32_t) * m.size(), cudaMemcpyDeviceToHost, h.stream) != cudaSuccess ||
      cudaStreamSynchronize(h.stream) != cudaSuccess)
    return -1;
  for (int64_t k = 0; k < h.K; ++k) order[(size_t)k] = (int32_t)k;
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return m[(size_t)a] < m[(size_t)b]; });
  if (cudaMemcpyAsync(h.porder, order.data(), sizeof(int32_t) * order.size(), cudaMemcpyHostToDevice, h.stream) !=
          cudaSuccess ||
      cudaStreamSynchronize(h.stream) != cudaSuccess)
    return -1;
  return 0;
}

__global__ void k_transpose(const double* __restrict__ A, int R, double* __restrict__ AT) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x < R * R) AT[(x % R) * R + x / R] = A[x];
}

int launch_polar_warp(Handle& h) {
  if (h.K == 0) return 0;
  const int R = h.R;
  if (polar_thread_ok(h)) {  // small ranks: thread per patient, registers
    if (R <= 4) { polar_thread_inst<4>(h); return 1; }
    if (R <= 6) { polar_thread_inst<6>(h); return 1; }
    if (R <= 8) { polar_thread_inst<8>(h); return 1; }
    polar_thread_inst<10>(h);
    return 1;
  }
  int nwb = kPlainWarps;
  auto smem_of = [&](int w) { return sizeof(double) * (size_t)w * polar_warp_per_warp(R); };
  while (nwb > 1 && smem_of(nwb) > 227 * 1024) --nwb;
  const size_t smem = smem_of(nwb);
  const auto fn = R <= 16 ? k_polar_warp<16> : R <= 32 ? k_polar_warp<32> : R <= 48 ? k_polar_warp<48>
                                                                               : k_polar_warp<64>;
  if (R <= 16) max_smem_attr<k_polar_warp<16>>(h);
  else if (R <= 32) max_smem_attr<k_polar_warp<32>>(h);
  else if (R <= 48) max_smem_attr<k_polar_warp<48>>(h);
  else max_smem_attr<k_polar_warp<64>>(h);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * nwb, smem);
  int64_t blocks = (h.K + nwb - 1) / nwb;
  const int64_t cap = (int64_t)h.sms * std::max(per_sm, 1);
  if (blocks > cap) blocks = cap;
  k_transpose<<<(unsigned)((R * R + 255) / 256), 256, 0, h.stream>>>(h.H, R, h.HT);
  fn<<<(unsigned)blocks, 32 * nwb, smem, h.stream>>>(h.m, h.srow, h.K, R, h.Pp, h.W, h.HT, h.o.rank_tol,
                                                               h.Qt, h.rank, h.diag);
  return 2;
}

// ------------------------------------------------------------------ W pass (warp per patient)
// Rows of Q~_k and P'_k are staged 32 at a time into the warp's shared memory with coalesced loads
// (a patient's rows are contiguous), so no row waits on its own global load; lane r then runs the
// sequential row loops of its column exactly as before (same operations, same order).
// rows per stage: 32 for R <= 16, else 8 (keeps several blocks per SM at large R)
__host__ __device__ inline int stage_rows_of(int R) { return R <= 16 ? 32 : 8; }
__host__ __device__ inline size_t passB_warp_per_warp(int R) { return 2 * (size_t)stage_rows_of(R) * R; }

__device__ __forceinline__ void stage_rows(double* dst, const double* __restrict__ src, int n) {
  for (int x = threadIdx.x & 31; x < n; x += 32) dst[x] = src[x];
}

// RB > 0 (R <= RB <= 32): lane r keeps column r of H̄ and of (G_W + rho I)^-1 in registers and the
// row loops are unrolled (the kernel was issue-bound on the per-element shared-memory loads and the
// second-half predicates: 218 instructions per row at R = 10); the FMA order is unchanged.
template <int RB>
__global__ void __launch_bounds__(32 * kPlainWarps) k_passB_warp(const int32_t* __restrict__ m,
                                                                 const int64_t* __restrict__ srow, int64_t K, int R,
                                                                 const double* __restrict__ Pp,
                                                                 const double* __restrict__ Qt,
                                                                 const double* __restrict__ Hg,
                                                                 const double* __restrict__ GWi,
                                                                 const double* __restrict__ scal, int n_inner,
                                                                 int kind, double param, double tol,
                                                                 double* __restrict__ W, double* __restrict__ DW,
                                                                 double* __restrict__ Nst,
                                                                 unsigned long long* __restrict__ steps) {
  extern __shared__ double smb[];
  double* Hs = smb;           // H̄ (R x R): Hs[i R + r]
  double* GT = smb + R * R;   // (G_W + rho I)^-1 transposed: GT[q R + r] = Ginv(r, q)
  for (int x = threadIdx.x; x < R * R; x += blockDim.x) {
    Hs[x] = Hg[x];
    const int r = x / R, q = x - r * R;
    GT[q * R + r] = GWi[x];
  }
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* Qs = smb + 2 * R * R + (size_t)wib * passB_warp_per_warp(R);  // staged rows of Q~_k
  const int SR = stage_rows_of(R);
  double* Ps = Qs + SR * R;                                              // ... and of P'_k
  __syncthreads();
  const double rho = scal[S_RHO_W];
  const bool has0 = lane < R, has1 = lane + 32 < R;
  const int64_t nw = (int64_t)gridDim.x * kPlainWarps;
  int my_steps = 0;
  constexpr int RC = RB > 0 ? RB : 1;
  double hc[RC], gc[RC];  // RB > 0: hc[i] = H̄(i, lane), gc[q] = Ginv(lane, q)
  if (RB > 0) {
#pragma unroll
    for (int i = 0; i < RC; ++i) {
      hc[i] = (has0 && i < R) ? Hs[i * R + lane] : 0.0;
      gc[i] = (has0 && i < R) ? GT[i * R + lane] : 0.0;
    }
  }
  auto t_row = [&](const double* qrow, double& t0, double& t1) {  // T(a, r) = sum_i Q~(a, i) H̄(i, r)
    double s0 = 0.0, s1 = 0.0;
    if (RB > 0) {
#pragma unroll
      for (int i = 0; i < RC; ++i)
        if (i < R) s0 = fma(qrow[i], hc[i], s0);
    } else {
      for (int i = 0; i < R; ++i) {
        const double qa = qrow[i];
        if (has0) s0 = fma(qa, Hs[i * R + lane], s0);
        if (has1) s1 = fma(qa, Hs[i * R + lane + 32], s1);
      }
    }
    t0 = s0;
    t1 = s1;
  };
  for (int64_t k = blockIdx.x * (int64_t)kPlainWarps + wib; k < K; k += nw) {
    const int mk = m[k];
    const double* P = Pp + srow[k] * R;
    const double* Q = Qt + srow[k] * R;
    double f0 = 0.0, f1 = 0.0;  // F_W(k, r) = sum_a T(a, r) P'(a, r), a ascending
    for (int a0 = 0; a0 < mk; a0 += SR) {
      const int na = mk - a0 < SR ? mk - a0 : SR;
      __syncwarp();
      stage_rows(Qs, Q + (int64_t)a0 * R, na * R);
      stage_rows(Ps, P + (int64_t)a0 * R, na * R);
      __syncwarp();
      for (int a = 0; a < na; ++a) {
        double t0, t1;
        t_row(Qs + a * R, t0, t1);
        if (has0) f0 = fma(t0, Ps[a * R + lane], f0);
        if (has1) f1 = fma(t1, Ps[a * R + lane + 32], f1);
      }
    }
    double w0 = has0 ? W[k * R + lane] : 0.0, w1 = has1 ? W[k * R + lane + 32] : 0.0;
    double d0 = has0 ? DW[k * R + lane] : 0.0, d1 = has1 ? DW[k * R + lane + 32] : 0.0;
    int it = 0;
    while (it < n_inner) {  // Alg.1 l.15-l.18 on the row, z = (G_W + rho I)^-1 (f + rho (w̄ + d))
      const double h0 = has0 ? f0 + rho * (w0 + d0) : 0.0;
      const double h1 = has1 ? f1 + rho * (w1 + d1) : 0.0;
      double z0 = 0.0, z1 = 0.0;
      if (RB > 0) {
#pragma unroll
        for (int qq = 0; qq < RC; ++qq)
          if (qq < R) z0 = fma(gc[qq], __shfl_sync(kFull, h0, qq), z0);
      } else {
        for (int qq = 0; qq < R; ++qq) {
          const double hq = lane_pick(h0, h1, qq);
          if (has0) z0 = fma(GT[qq * R + lane], hq, z0);
          if (has1) z1 = fma(GT[qq * R + lane + 32], hq, z1);
        }
      }
      RowResid res;
      if (has0) {
        const double nb = prox(kind, param, rho, z0 - d0);
        res.add(nb, z0, w0);
        d0 = d0 + nb - z0;
        w0 = nb;
      }
      if (has1) {
        const double nb = prox(kind, param, rho, z1 - d1);
        res.add(nb, z1, w1);
        d1 = d1 + nb - z1;
        w1 = nb;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        res.pr += __shfl_xor_sync(kFull, res.pr, o);
        res.du += __shfl_xor_sync(kFull, res.du, o);
        res.nz += __shfl_xor_sync(kFull, res.nz, o);
      }
      ++it;
      if (res.done(tol)) break;
    }
    my_steps += it;
    if (has0) { W[k * R + lane] = w0; DW[k * R + lane] = d0; }
    if (has1) { W[k * R + lane + 32] = w1; DW[k * R + lane + 32] = d1; }
    double* N = Nst + srow[k] * R;  // N_k = T S_k (new w̄_k)
    for (int a0 = 0; a0 < mk; a0 += SR) {
      const int na = mk - a0 < SR ? mk - a0 : SR;
      if (a0 > 0 || mk > SR) {  // (a single stage is still in Qs from the F_W loop)
        __syncwarp();
        stage_rows(Qs, Q + (int64_t)a0 * R, na * R);
        __syncwarp();
      }
      for (int a = 0; a < na; ++a) {
        double t0, t1;
        t_row(Qs + a * R, t0, t1);
        if (has0) N[(int64_t)(a0 + a) * R + lane] = t0 * w0;
        if (has1) N[(int64_t)(a0 + a) * R + lane + 32] = t1 * w1;
      }
    }
  }
  if (lane == 0 && my_steps) atomicAdd(steps + 1, (unsigned long long)my_steps);
}

int launch_passB_warp(Handle& h) {
  if (h.K == 0) return 0;
  const size_t smem = sizeof(double) * (2 * (size_t)h.R * h.R + kPlainWarps * passB_warp_per_warp(h.R));
  const auto fn = h.R <= 16 ? k_passB_warp<16> : h.R <= 32 ? k_passB_warp<32> : k_passB_warp<0>;
  if (h.R <= 16) max_smem_attr<k_passB_warp<16>>(h);
  else if (h.R <= 32) max_smem_attr<k_passB_warp<32>>(h);
  else max_smem_attr<k_passB_warp<0>>(h);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * kPlainWarps, smem);
  int64_t blocks = (h.K + kPlainWarps - 1) / kPlainWarps;
  const int64_t cap = (int64_t)h.sms * std::max(per_sm, 1);
  if (blocks > cap) blocks = cap;
  fn<<<(unsigned)blocks, 32 * kPlainWarps, smem, h.stream>>>(
      h.m, h.srow, h.K, h.R, h.Pp, h.Qt, h.H, h.GWi, h.scal, h.o.admm_inner, h.o.on_W.kind, h.o.on_W.param,
      h.o.admm_tol, h.W, h.DW, h.Nst, h.steps);
  return 1;
}

// ------------------------------------------------------------------ feature-major copy of X (init)
// Stable radix sort of the nonzeros by column (keys) carrying their index; entries of one column
// stay in row order. csc_row[e] = row of the e-th entry in column order, csc_val[e] its value.
__global__ void k_nnz_rows(const int64_t* __restrict__ rp, int64_t rows, int32_t* __restrict__ row_of) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  for (int64_t e = rp[i]; e < rp[i + 1]; ++e) row_of[e] = (int32_t)i;
}

__global__ void k_iota(int32_t* __restrict__ x, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = (int32_t)i;
}

__global__ void k_csc_fill(const int32_t* __restrict__ perm, const int32_t* __restrict__ row_of,
                           const double* __restrict__ val, int64_t nnz, int32_t* __restrict__ csc_row,
                           double* __restrict__ csc_val) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nnz) return;
  const int32_t src = perm[e];
  csc_row[e] = row_of[src];
  csc_val[e] = val[src];
}

__global__ void k_col_counts(const int32_t* __restrict__ sorted_cols, int64_t nnz, int64_t J,
                             int64_t* __restrict__ cptr /*[J+1]*/) {
  // cptr[j] = first position of column j in the sorted order (binary search per column)
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j > J) return;
  int64_t lo = 0, hi = nnz;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (sorted_cols[mid] < j) lo = mid + 1;
    else hi = mid;
  }
  cptr[j] = lo;
}

size_t csc_temp_bytes(const Handle& h) {
  if (h.nnz == 0) return 256;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, (const int32_t*)nullptr, (int32_t*)nullptr, (const int32_t*)nullptr,
                                  (int32_t*)nullptr, (int)h.nnz);
  return tb + 4 * sizeof(int32_t) * (size_t)h.nnz + 1024;
}

// Builds csc_ptr/csc_row/csc_val and the chunk table of the F_V gather (host planning).
int build_csc(Handle& h) {
  if (h.nnz == 0) {
    cudaMemsetAsync(h.csc_ptr, 0, sizeof(int64_t) * (size_t)(h.J + 1), h.stream);
    h.csc_chunks = 0;
    return 0;
  }
  const int64_t n = h.nnz;
  char* t = (char*)h.csc_tmp;
  int32_t* keys_out = (int32_t*)t;
  int32_t* idx_in = keys_out + n;
  int32_t* idx_out = idx_in + n;
  int32_t* row_of = idx_out + n;
  void* cub_tmp = (void*)(row_of + n);
  size_t tb = h.csc_tmp_bytes - 4 * sizeof(int32_t) * (size_t)n;
  const unsigned g = (unsigned)((n + 255) / 256);
  k_iota<<<g, 256, 0, h.stream>>>(idx_in, n);
  k_nnz_rows<<<(unsigned)((h.rows + 255) / 256), 256, 0, h.stream>>>(h.p.row_ptr, h.rows, row_of);
  int end_bit = 1;
  while ((int64_t(1) << end_bit) <= h.J) ++end_bit;
  cub::DeviceRadixSort::SortPairs(cub_tmp, tb, h.p.col, keys_out, idx_in, idx_out, (int)n, 0, end_bit, h.stream);
  k_csc_fill<<<g, 256, 0, h.stream>>>(idx_out, row_of, h.p.val, n, h.csc_row, h.csc_val);
  k_col_counts<<<(unsigned)((h.J + 1 + 255) / 256), 256, 0, h.stream>>>(keys_out, n, h.J, h.csc_ptr);
  std::vector<int64_t> cptr((size_t)h.J + 1);
  if (cudaMemcpyAsync(cptr.data(), h.csc_ptr, sizeof(int64_t) * cptr.size(), cudaMemcpyDeviceToHost, h.stream) !=
          cudaSuccess ||
      cudaStreamSynchronize(h.stream) != cudaSuccess)
    return -1;
  std::vector<int64_t> ch;  // chunk c: entries [ch[2c], ch[2c+1]) of one column
  std::vector<int64_t> first((size_t)h.J + 1);  // first chunk of column j
  for (int64_t j = 0; j < h.J; ++j) {
    first[(size_t)j] = (int64_t)ch.size() / 2;
    for (int64_t a = cptr[(size_t)j]; a < cptr[(size_t)j + 1]; a += kCscChunk) {
      ch.push_back(a);
      ch.push_back(std::min<int64_t>(a + kCscChunk, cptr[(size_t)j + 1]));
    }
  }
  first[(size_t)h.J] = (int64_t)ch.size() / 2;
  h.csc_chunks = (int64_t)ch.size() / 2;
  if (h.csc_chunks > h.csc_chunk_cap) return -2;
  if (h.csc_chunks > 0)
    cudaMemcpyAsync(h.csc_chunk, ch.data(), sizeof(int64_t) * ch.size(), cudaMemcpyHostToDevice, h.stream);
  cudaMemcpyAsync(h.csc_chunk_first, first.data(), sizeof(int64_t) * first.size(), cudaMemcpyHostToDevice, h.stream);
  if (cudaStreamSynchronize(h.stream) != cudaSuccess) return -1;
  return 0;
}

// ------------------------------------------------------------------ F_V gather over the CSC copy
// Warp per chunk: lanes over r, entries in column order (row order within the column), 4 entries
// in flight; the chunk's partial row goes to part[c]. Then F_V(j, :) = sum of column j's chunk
// partials in chunk order.
__global__ void __launch_bounds__(256) k_scatter_csc(const int64_t* __restrict__ chunk, int64_t nchunks, int R,
                                                     const int32_t* __restrict__ csc_row,
                                                     const double* __restrict__ csc_val,
                                                     const double* __restrict__ Nst, double* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const bool has0 = lane < R, has1 = lane + 32 < R;
  for (int64_t c = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); c < nchunks; c += nw) {
    const int64_t e0 = chunk[2 * c], e1 = chunk[2 * c + 1];
    double a0 = 0.0, a1 = 0.0;
    int64_t e = e0;
    for (; e + 4 <= e1; e += 4) {
      int32_t rw[4];
      double x[4], n0[4], n1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        rw[u] = csc_row[e + u];
        x[u] = csc_val[e + u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double* Nr = Nst + (int64_t)rw[u] * R;
        n0[u] = has0 ? Nr[lane] : 0.0;
        n1[u] = has1 ? Nr[lane + 32] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0 = fma(x[u], n0[u], a0);
        a1 = fma(x[u], n1[u], a1);
      }
    }
    for (; e < e1; ++e) {
      const double* Nr = Nst + (int64_t)csc_row[e] * R;
      const double x = csc_val[e];
      if (has0) a0 = fma(x, Nr[lane], a0);
      if (has1) a1 = fma(x, Nr[lane + 32], a1);
    }
    if (has0) part[c * R + lane] = a0;
    if (has1) part[c * R + lane + 32] = a1;
  }
}

// F_V(j, r) = sum of column j's chunk partials in a fixed order: 32 entries (j, r) per block, the
// column's chunks c = first + g, first + g + 32, ... summed by thread g of the entry, then the 32
// group sums in ascending g (columns of up to 32 chunks: plain ascending-chunk order). Under the
// Zipf feature law one column holds hundreds of chunks; one thread walking them took 88 us on Small.
__global__ void __launch_bounds__(1024) k_sum_chunks(int64_t J, int R, const double* __restrict__ part,
                                                     const int64_t* __restrict__ chunk_first /*[J+1] first chunk of column j*/,
                                                     double* __restrict__ FV) {
  __shared__ double sm[32][33];
  const int px = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t x = blockIdx.x * (int64_t)32 + px;
  double s = 0.0;
  if (x < J * R) {
    const int64_t j = x / R, r = x - j * R;
    const int64_t c1 = chunk_first[j + 1];
    for (int64_t c = chunk_first[j] + g; c < c1; c += 32) s += part[c * R + r];
  }
  sm[g][px] = s;
  __syncthreads();
  if (g == 0 && x < J * R) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 32; ++q) t += sm[q][px];
    FV[x] = t;
  }
}

int launch_scatter_csc(Handle& h, const double* Nrows) {
  if (h.csc_chunks == 0) {
    cudaMemsetAsync(h.FV, 0, sizeof(double) * (size_t)(h.J * h.R), h.stream);
    return 0;
  }
  int64_t blocks = (h.csc_chunks + 7) / 8;
  if (blocks > (int64_t)h.sms * 8) blocks = (int64_t)h.sms * 8;
  k_scatter_csc<<<(unsigned)blocks, 256, 0, h.stream>>>(h.csc_chunk, h.csc_chunks, h.R, h.csc_row, h.csc_val, Nrows,
                                                        h.csc_part);
  const int64_t n = h.J * h.R;
  k_sum_chunks<<<(unsigned)((n + 31) / 32), 1024, 0, h.stream>>>(h.J, h.R, h.csc_part,
                                                                  h.csc_chunk_first, h.FV);
  return 2;
}

}  // namespace copa
