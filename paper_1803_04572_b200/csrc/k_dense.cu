// k_dense.cu — per-patient dense work of the smooth ("wide": m_k <= l < R) path, organised in
// warp rounds of 32 patients: the R-dimension contractions run on the FP64 tensor cores
// (mma.sync m8n8k4 f64, warp-cooperative, one patient per MMA tile) and the small sequential
// m_k x m_k algebra (Givens QR, one-sided Jacobi, row ADMM solves) runs one patient per thread.
//
//   polar_wide : A_k = P'_k S_k H̄^T (MMA, 8-column slabs) -> Givens QR of A_k^T (thread)
//                -> Jacobi (thread) -> Q~_k = K_k A_k (thread, K_k = V Σ^-1 V^T on the range)
//                -> F_H += Q~_k^T P'_k S_k (MMA, per-warp accumulators)        (Alg.1 l.4-6, l.12)
//   passB_wide : T_k = Q~_k H̄ (MMA) -> F_W(k,:) = colsum(T_k ∘ P'_k) -> W-row ADMM (thread)
//                -> N_k = T_k S_k (MMA recompute) -> M += N_k^T N_k, W̄^T W̄ (MMA)  (l.12-19, FIT)
// This file: dispatch of the wide kernels by smooth_l; the kernels and their templates live in
// k_dense.cuh, instantiated per l in k_polar_l*.cu / k_passB_m*.cu.
#include "copa_internal.cuh"

namespace copa {

void polar_wide_L4(Handle& h);
void polar_wide_L7(Handle& h);
void polar_wide_L8(Handle& h);
void polar_wide_L9(Handle& h);
void polar_wide_L12(Handle& h);
bool passB_wide_special(Handle& h);
void passB_wide_g1(Handle& h, int nt);
void passB_wide_g2a(Handle& h);
void passB_wide_g2b(Handle& h);
void passB_wide_g2c(Handle& h);
void passB_wide_g2d(Handle& h);
void passB_wide_g3(Handle& h, int nt);
void passB_wide_g4a(Handle& h);
void passB_wide_g4b(Handle& h);
void passB_wide_g4c(Handle& h);
void passB_wide_g4d(Handle& h);

bool polar_wide_ok(const Handle& h) { return h.smooth && h.l < h.R && h.l <= 12; }

// Polar + F_H for the wide case. Returns kernels launched.
int launch_polar_wide(Handle& h) {
  if (h.l <= 4) polar_wide_L4(h);
  else if (h.l <= 7) polar_wide_L7(h);
  else if (h.l <= 8) polar_wide_L8(h);
  else if (h.l <= 9) polar_wide_L9(h);
  else polar_wide_L12(h);
  return 3;  // polar kernel + two-stage F_H reduction
}

int launch_passB_wide(Handle& h) {
  if (!passB_wide_special(h)) {
    const int nt = (h.R + 7) / 8 < 8 ? (h.R + 7) / 8 : 8;
    static void (*const big[2][4])(Handle&) = {{passB_wide_g2a, passB_wide_g2b, passB_wide_g2c, passB_wide_g2d},
                                               {passB_wide_g4a, passB_wide_g4b, passB_wide_g4c, passB_wide_g4d}};
    if (nt <= 4) (h.l <= 8 ? passB_wide_g1 : passB_wide_g3)(h, nt);
    else big[h.l <= 8 ? 0 : 1][nt - 5](h);
  }
  return 2;
}

}  // namespace copa
