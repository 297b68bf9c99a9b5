// k_rowproj.cu — smoothness in the paper's regime: l > 16 basis functions (the
// paper's l = 33 at R = 15), where storing X'_k = C_k^T X_k as projected fibers (l
// values per (patient, feature)) no longer pays. The projection is applied per iteration through
// the sparse spline matrix instead (C_k = M_k B_k, M_k with d + 1 non-zeros per row recomputed from
// the visit times, B_k the l x l basis coefficients):
//
//   basis_warp  init, warp per patient: Givens QR of the rows of M_k (shared memory), one-sided
//               Jacobi, B_k = V Σ^-1 on the kept directions (sigma_j > tau sigma_1), descending
//   rowproj_P   P'_k = C_k^T (X_k V̄) = B_k^T (M_k^T P_k), P_k = X_k V̄ per visit row       (Alg.1 l.4 input)
//   rowproj_N   C_k N'_k = M_k (B_k N'_k) per visit row, then the CSC gather F_V = sum_k X_k^T (C_k N'_k)
//                                                                                    (l.12, V mode)
// The polar, F_H, the W pass and the Grams are the general path's (k_plain.cu, state rows k l).
#include <algorithm>

#include "copa_internal.cuh"

namespace copa {

constexpr unsigned kFullR = 0xffffffffu;
constexpr int kRpWarps = 4;

__device__ __forceinline__ double pick2(double v0, double v1, int j) {
  return __shfl_sync(kFullR, j < 32 ? v0 : v1, j & 31);
}

// ------------------------------------------------------------------ basis (init), warp per patient
__global__ void __launch_bounds__(32 * kRpWarps) k_basis_warp(const int64_t* __restrict__ prp,
                                                              const double* __restrict__ times, int64_t K, int l, int d,
                                                              double tau, double* __restrict__ Bk,
                                                              int32_t* __restrict__ m,
                                                              unsigned long long* __restrict__ diag) {
  extern __shared__ double smr[];
  const int LD = l | 1;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  double* Rm = smr + (size_t)wib * l * LD;
  const int64_t nw = (int64_t)gridDim.x * nwb;
  for (int64_t k = blockIdx.x * (int64_t)nwb + wib; k < K; k += nw) {
    const int64_t r0 = prp[k], r1 = prp[k + 1];
    const double t1 = times[r0], tn = times[r1 - 1];
    double* B = Bk + k * (int64_t)l * l;
    if (!(tn > t1)) {  // single visit: all knots coincide, M_k = 0 (the recursion's 0/0 := 0)
      for (int x = lane; x < l * l; x += 32) B[x] = 0.0;
      if (lane == 0) m[k] = 0;
      continue;
    }
    for (int x = lane; x < l * LD; x += 32) Rm[x] = 0.0;
    __syncwarp();
    double dg0 = 0.0, dg1 = 0.0;
    const bool own0 = lane < l, own1 = lane + 32 < l;
    for (int64_t i = r0; i < r1; ++i) {  // Givens insert of row i of M_k (d + 1 non-zeros)
      double N[kMaxDeg + 1];
      const int mu = spline_eval(times[i], t1, tn, l, d, N);
      double v0 = 0.0, v1 = 0.0;
#pragma unroll
      for (int r = 0; r <= kMaxDeg; ++r) {
        if (r > d) break;
        const int b = mu - d + r;
        if (b == lane) v0 = N[r];
        if (b == lane + 32) v1 = N[r];
      }
      for (int j = mu - d; j < l; ++j) {  // columns < mu - d of the row are zero
        const double x0 = (own0 && lane > j) ? Rm[j * LD + lane] : 0.0;
        const double x1 = (own1 && lane + 32 > j) ? Rm[j * LD + lane + 32] : 0.0;
        const double vj = pick2(v0, v1, j);
        const double rr = pick2(dg0, dg1, j);
        if (vj != 0.0) {
          const double n2 = fma(rr, rr, vj * vj);
          const double inv = rsqrt(n2);
          const double cs = rr * inv, sn = vj * inv;
          if (own0 && lane > j) { Rm[j * LD + lane] = fma(cs, x0, sn * v0); v0 = fma(cs, v0, -sn * x0); }
          if (own1 && lane + 32 > j) { Rm[j * LD + lane + 32] = fma(cs, x1, sn * v1); v1 = fma(cs, v1, -sn * x1); }
          if (lane == (j & 31)) { if (j < 32) dg0 = n2 * inv; else dg1 = n2 * inv; }
        }
      }
    }
    if (own0) Rm[lane * LD + lane] = dg0;
    if (own1) Rm[(lane + 32) * LD + lane + 32] = dg1;
    __syncwarp();
    // one-sided Jacobi on the rows of Rm (round robin, one lane per disjoint pair)
    {
      const int N = (l & 1) ? l + 1 : l;
      const double eps = 2.220446049250313e-16 * (double)l, tol2 = eps * eps;
      double tr = 0.0;  // trace of the Gram (invariant): residue-row threshold (kJacobiNegl2)
      for (int x = lane; x < l; x += 32)
        for (int y = 0; y < l; ++y) tr = fma(Rm[x * LD + y], Rm[x * LD + y], tr);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(kFullR, tr, o);
      const double negl = kJacobiNegl2 * tr;
      for (int sweep = 0; sweep < 40; ++sweep) {
        int rotated = 0;
        for (int rd = 0; rd < N - 1; ++rd) {
          if (lane < N / 2) {
            const int p = lane == 0 ? 0 : 1 + (lane - 1 + rd) % (N - 1);
            const int r = 1 + (N - 2 - lane + rd) % (N - 1);
            if (p < l && r < l) {
              double* xp = Rm + p * LD;
              double* xr = Rm + r * LD;
              double a = 0.0, b = 0.0, c = 0.0;
              for (int x = 0; x < l; ++x) { a = fma(xp[x], xp[x], a); b = fma(xr[x], xr[x], b); c = fma(xp[x], xr[x], c); }
              if (a > negl && b > negl && c * c > tol2 * (a * b)) {
                rotated = 1;
                double cs, sn;
                jacobi_rot(a, b, c, cs, sn);
                for (int x = 0; x < l; ++x) {
                  const double u = xp[x], v = xr[x];
                  xp[x] = fma(cs, u, -sn * v);
                  xr[x] = fma(sn, u, cs * v);
                }
              }
            }
          }
          __syncwarp();
        }
        if (!__any_sync(kFullR, rotated)) break;
      }
    }
    // sigma_j = |row j|; kept rows (sigma_j > tau sigma_max) in descending sigma (stable):
    // B_k column pos = v_j / sigma_j = row_j / sigma_j^2, so C_k = M_k B_k = left singular vectors
    double n0 = 0.0, n1 = 0.0;
    if (own0) for (int x = 0; x < l; ++x) n0 = fma(Rm[lane * LD + x], Rm[lane * LD + x], n0);
    if (own1) for (int x = 0; x < l; ++x) n1 = fma(Rm[(lane + 32) * LD + x], Rm[(lane + 32) * LD + x], n1);
    const double sg0 = sqrt(n0), sg1 = sqrt(n1);
    double smax = fmax(sg0, sg1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) smax = fmax(smax, __shfl_xor_sync(kFullR, smax, o));
    const bool keep0 = own0 && smax > 0.0 && sg0 > tau * smax;
    const bool keep1 = own1 && smax > 0.0 && sg1 > tau * smax;
    {
      RatioDiag dgn;
      if (smax > 0.0) {
        if (own0) dgn.note(sg0 / smax, keep0, tau);
        if (own1) dgn.note(sg1 / smax, keep1, tau);
      }
      ratio_diag_warp(diag, D_BASIS_NEAR, dgn);
    }
    int pos0 = 0, pos1 = 0;  // rank of row j among the kept rows by (sigma desc, index asc)
    for (int q = 0; q < l; ++q) {
      const double sq = pick2(sg0, sg1, q);
      pos0 += (sq > sg0 || (q < lane && sq == sg0)) ? 1 : 0;
      pos1 += (sq > sg1 || (q < lane + 32 && sq == sg1)) ? 1 : 0;
    }
    const int c = __popc(__ballot_sync(kFullR, keep0)) + __popc(__ballot_sync(kFullR, keep1));
    for (int x = lane; x < l * l; x += 32) B[x] = 0.0;
    __syncwarp();
    if (keep0) {
      const double inv2 = 1.0 / (sg0 * sg0);
      for (int i = 0; i < l; ++i) B[i * l + pos0] = Rm[lane * LD + i] * inv2;
    }
    if (keep1) {
      const double inv2 = 1.0 / (sg1 * sg1);
      for (int i = 0; i < l; ++i) B[i * l + pos1] = Rm[(lane + 32) * LD + i] * inv2;
    }
    if (lane == 0) m[k] = c;
    __syncwarp();
  }
}

static int rp_warps(size_t per_warp_doubles, size_t fixed_doubles = 0) {
  int w = kRpWarps;
  while (w > 1 && sizeof(double) * (fixed_doubles + w * per_warp_doubles) > 227 * 1024) --w;
  return w;
}

void launch_basis_warp(Handle& h) {
  if (h.K == 0) return;
  const size_t per = (size_t)h.l * (h.l | 1);
  const int w = rp_warps(per);
  max_smem_attr<k_basis_warp>(h);
  int64_t blocks = (h.K + w - 1) / w;
  if (blocks > (int64_t)h.sms * 16) blocks = (int64_t)h.sms * 16;
  k_basis_warp<<<(unsigned)blocks, 32 * w, sizeof(double) * w * per, h.stream>>>(
      h.p.patient_row_ptr, h.p.visit_time, h.K, h.l, h.d, h.o.basis_tol, h.Bk, h.m, h.diag);
}

// ------------------------------------------------------------------ P'_k = B_k^T (M_k^T (X_k V̄))
// warp per patient, lanes over r: T = M_k^T P_k (l x R) accumulated in shared memory visit by visit
// (row i adds N_b(t_i) P_k(i, :) to rows mu-d..mu), then P'(a, :) = sum_b B_k(b, a) T(b, :), a < m_k.
__global__ void __launch_bounds__(32 * kRpWarps) k_rowproj_P(const int64_t* __restrict__ prp,
                                                             const double* __restrict__ times, int64_t K, int l, int d,
                                                             int R, const double* __restrict__ Bk,
                                                             const int32_t* __restrict__ m,
                                                             const double* __restrict__ Prow, double* __restrict__ Pp) {
  extern __shared__ double smr[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  double* T = smr + (size_t)wib * l * R;
  const bool has0 = lane < R, has1 = lane + 32 < R;
  const int64_t nw = (int64_t)gridDim.x * nwb;
  for (int64_t k = blockIdx.x * (int64_t)nwb + wib; k < K; k += nw) {
    const int mk = m[k];
    if (mk == 0) continue;  // state rows stay zero
    const int64_t r0 = prp[k], r1 = prp[k + 1];
    const double t1 = times[r0], tn = times[r1 - 1];
    for (int x = lane; x < l * R; x += 32) T[x] = 0.0;
    __syncwarp();
    for (int64_t i = r0; i < r1; ++i) {
      double N[kMaxDeg + 1];
      const int mu = spline_eval(times[i], t1, tn, l, d, N);
      const double p0 = has0 ? Prow[i * R + lane] : 0.0, p1 = has1 ? Prow[i * R + lane + 32] : 0.0;
      for (int r = 0; r <= d; ++r) {
        double* Tb = T + (mu - d + r) * R;
        if (has0) Tb[lane] = fma(N[r], p0, Tb[lane]);
        if (has1) Tb[lane + 32] = fma(N[r], p1, Tb[lane + 32]);
      }
    }
    const double* B = Bk + k * (int64_t)l * l;
    double* P = Pp + k * (int64_t)l * R;
    for (int a = 0; a < mk; ++a) {
      double s0 = 0.0, s1 = 0.0;
      for (int b = 0; b < l; ++b) {
        const double bb = B[b * l + a];
        if (has0) s0 = fma(bb, T[b * R + lane], s0);
        if (has1) s1 = fma(bb, T[b * R + lane + 32], s1);
      }
      if (has0) P[(int64_t)a * R + lane] = s0;
      if (has1) P[(int64_t)a * R + lane + 32] = s1;
    }
    __syncwarp();
  }
}

// spmm of the visit rows (k_iter.cu's row kernel) into Prow, then the projection
__global__ void k_spmm_rows_rp(const int64_t* rp, const int32_t* col, const double* val, int64_t rows, int R,
                               const double* V, double* P) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= rows * R) return;
  int64_t i = t / R;
  int r = (int)(t - i * R);
  double acc = 0.0;
  for (int64_t e = rp[i]; e < rp[i + 1]; ++e) acc = fma(val[e], V[(int64_t)col[e] * R + r], acc);
  P[t] = acc;
}

int launch_rowproj_P(Handle& h) {
  if (h.K == 0) return 0;
  const int64_t n = h.rows * h.R;
  k_spmm_rows_rp<<<(unsigned)((n + 255) / 256), 256, 0, h.stream>>>(h.p.row_ptr, h.p.col, h.p.val, h.rows, h.R, h.V,
                                                                     h.Prow);
  const size_t per = (size_t)h.l * h.R;
  const int w = rp_warps(per);
  max_smem_attr<k_rowproj_P>(h);
  int64_t blocks = (h.K + w - 1) / w;
  if (blocks > (int64_t)h.sms * 16) blocks = (int64_t)h.sms * 16;
  k_rowproj_P<<<(unsigned)blocks, 32 * w, sizeof(double) * w * per, h.stream>>>(
      h.p.patient_row_ptr, h.p.visit_time, h.K, h.l, h.d, h.R, h.Bk, h.m, h.Prow, h.Pp);
  return 2;
}

// ------------------------------------------------------------------ C_k N'_k = M_k (B_k N'_k) per visit row
__global__ void __launch_bounds__(32 * kRpWarps) k_rowproj_N(const int64_t* __restrict__ prp,
                                                             const double* __restrict__ times, int64_t K, int l, int d,
                                                             int R, const double* __restrict__ Bk,
                                                             const int32_t* __restrict__ m,
                                                             const double* __restrict__ Nst, double* __restrict__ Nrow) {
  extern __shared__ double smr[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  double* U = smr + (size_t)wib * l * R;
  const bool has0 = lane < R, has1 = lane + 32 < R;
  const int64_t nw = (int64_t)gridDim.x * nwb;
  for (int64_t k = blockIdx.x * (int64_t)nwb + wib; k < K; k += nw) {
    const int mk = m[k];
    const int64_t r0 = prp[k], r1 = prp[k + 1];
    if (mk == 0) {  // M_k = 0: the patient's rows contribute nothing
      for (int64_t i = r0; i < r1; ++i) {
        if (has0) Nrow[i * R + lane] = 0.0;
        if (has1) Nrow[i * R + lane + 32] = 0.0;
      }
      continue;
    }
    const double* B = Bk + k * (int64_t)l * l;
    const double* Nk = Nst + k * (int64_t)l * R;
    for (int b = 0; b < l; ++b) {  // U = B_k N'_k (l x R)
      double s0 = 0.0, s1 = 0.0;
      for (int a = 0; a < mk; ++a) {
        const double bb = B[b * l + a];
        if (has0) s0 = fma(bb, Nk[(int64_t)a * R + lane], s0);
        if (has1) s1 = fma(bb, Nk[(int64_t)a * R + lane + 32], s1);
      }
      if (has0) U[b * R + lane] = s0;
      if (has1) U[b * R + lane + 32] = s1;
    }
    __syncwarp();
    const double t1 = times[r0], tn = times[r1 - 1];
    for (int64_t i = r0; i < r1; ++i) {
      double N[kMaxDeg + 1];
      const int mu = spline_eval(times[i], t1, tn, l, d, N);
      double s0 = 0.0, s1 = 0.0;
      for (int r = 0; r <= d; ++r) {
        const double* Ub = U + (mu - d + r) * R;
        if (has0) s0 = fma(N[r], Ub[lane], s0);
        if (has1) s1 = fma(N[r], Ub[lane + 32], s1);
      }
      if (has0) Nrow[i * R + lane] = s0;
      if (has1) Nrow[i * R + lane + 32] = s1;
    }
    __syncwarp();
  }
}

int launch_rowproj_N(Handle& h) {
  if (h.K == 0) return 0;
  const size_t per = (size_t)h.l * h.R;
  const int w = rp_warps(per);
  max_smem_attr<k_rowproj_N>(h);
  int64_t blocks = (h.K + w - 1) / w;
  if (blocks > (int64_t)h.sms * 16) blocks = (int64_t)h.sms * 16;
  k_rowproj_N<<<(unsigned)blocks, 32 * w, sizeof(double) * w * per, h.stream>>>(
      h.p.patient_row_ptr, h.p.visit_time, h.K, h.l, h.d, h.R, h.Bk, h.m, h.Nst, h.Nrow);
  return 1;
}

}  // namespace copa
