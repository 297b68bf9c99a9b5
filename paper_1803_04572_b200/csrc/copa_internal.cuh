// copa_internal.cuh — internal types, device helpers and kernel launchers of libcopa.so.
// Product path (CUDA, sm_100a, FP64). Shares no code with oracle/ (see DESIGN.md §1).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <vector>

#include "../../include/copa.h"

namespace copa {

constexpr int kMaxR = 64;       // rank limit (local arrays in the per-patient kernels)
constexpr int kMaxL = 64;       // smooth_l limit (row-projection path above kMaxFiberL)
constexpr int kMaxFiberL = 16;  // smooth_l limit of the projected-fiber layout (k_fibers.cu, k_passA.cu)
constexpr int kMaxDeg = 7;      // spline degree limit
constexpr int64_t kMaxJ = 65535;
constexpr int kPartBlocks = 592;  // per-block partials of the R x R reductions (4 x 148 SMs)
constexpr int kPhases = 11;       // timed phases of one outer iteration (copa_get_phase_times)
constexpr int kMaxGroups = 8;     // label groups (fiber streams) of the smooth path
constexpr int kWoS = 16;         // uint16 entries per (group, patient) record of woff (>= sub-ranges + 1)
// entries per chunk of the non-smooth F_V gather (a warp walks its chunk serially: 512 took 123 us on Small)
constexpr int64_t kCscChunk = 128;

constexpr double kJacobiNegl2 = 1e-30;  // see the note at jacobi_rows

enum ErrBits : int { ERR_CHOL = 1, ERR_DEGEN = 2, ERR_NONFINITE = 4, ERR_SHAPE = 8, ERR_INPUT_NONFINITE = 16 };

// Rank-cut diagnostics (copa_stats; SURVEY 8(c) parity protocol): counts, and ratios as the bit
// patterns of non-negative doubles (ordered like unsigned integers).
enum DiagSlot : int { D_POLAR_NEAR = 0, D_POLAR_KEPT, D_POLAR_DROP, D_BASIS_NEAR, D_BASIS_KEPT, D_BASIS_DROP,
                      kDiagSlots = 8 };

// Scalar slots in Handle::scal
enum Scal : int { S_NORMX = 0, S_RHO_H, S_RHO_W, S_RHO_V, S_FIT, S_CROSS, S_QUAD, S_E, S_COUNT = 16 };

struct Handle {
  copa_problem p;      // device pointers of the CSR input
  copa_options o;
  cudaStream_t stream;
  int dev = 0;         // CUDA device of the handle (current device at init)
  int sms = 148;       // its multiprocessor count (queried)
  int smooth;          // smooth_l > 0
  int fib;             // smooth with the projected-fiber layout (l <= kMaxFiberL)
  int rowproj;         // smooth with l > kMaxFiberL: row passes + sparse M_k projection (k_rowproj.cu)
  double *Prow, *Nrow; // rowproj: [rows x R] X_k V and C_k N'_k per visit row
  int l, d;            // basis size / degree (smooth)
  int64_t K, J, rows, nnz;
  int R;
  int64_t S;           // state rows
  int64_t F;           // fibers (smooth)
  int64_t iterations;
  // workspace segments (device)
  int* err;
  double* scal;
  double *H, *DH, *FH, *HtH, *VtV, *LW, *GWi, *partial;  // GWi = (G_W + rho I)^-1
  double* HT;          // H̄^T (general polar, refreshed per launch)
  double* fh_warp;     // smooth: per-warp F_H partials of the polar kernel [kPartBlocks x 4 x (8 ceil(R/8))^2]
  double *comm2;       // [FV (J R) | WtW (R R) | M (R R)]
  double *FV, *WtW, *M;
  double *V, *DV;
  double *W, *DW;
  int32_t *m, *rank;
  int64_t* srow;
  double *Pp, *Qt, *Nst;
  double* Bk;          // smooth: K x l x l basis coefficients (C_k = M_k B_k)
  int64_t* fiber_ptr;  // smooth: [K+1] fibers per patient (prefix), all groups
  int32_t* fiber_col;  // smooth: [Fcap] label of each fiber (g-stream layout, see k_fibers.cu)
  double* fiber_val;   // smooth: [Fcap x l]
  int64_t* gptr;       // smooth: [G x (K+1)] absolute offset of patient k's run in stream g
  int64_t Fcap = 0;    // fiber slots incl. stream padding
  // fiber-pass layout (smooth): relabeled features, pass A order, pass B CTAs and stage table
  int32_t* perm;         // [J] feature -> label
  int32_t* inv;          // [Jl] label -> feature (-1: unused label)
  double* Vl;            // [Jl x R] V̄ in label order (pass A)
  int32_t* fa_col;       // pass A layout: patient k's fibers at [fiber_ptr[k], fiber_ptr[k+1]) (+64 slack)
  double* fa_val;
  int64_t* pa_wk;        // [pa_nw + 1] patient range of each pass-A warp (fiber-balanced)
  int64_t pa_nw = 0;
  int pa_ctas = 0;
  bool pa_vs = false;    // V̄ in shared memory in pass A
  int64_t* block_k;      // [sc_ranges+1] patient range of each pass-B range
  double* fv_part;       // [sc_ranges x Jl x R] per-range F_V partials
  unsigned long long* fhist;  // [J] fibers per feature (init)
  uint16_t* woff;        // [G x K x kWoS] label sub-run offsets inside each patient's group run
  int64_t* st_f;         // [nst_cap x 2] pass-B stage: logical fiber range [f0, f1) in its stream
  int32_t* st_k;         // [nst_cap x 2] pass-B stage: patient range [k0, k1)
  int32_t* cta_st;       // [sc_ranges x G + 1] first stage of each pass-B CTA
  int32_t* st_t;         // [nst_cap + 1] pass-B stage: first entry in st_list
  uint32_t* st_list;     // pass-B stage lists: per stage 8 sub-range offsets + (tile | patient << 16) per tile
  unsigned char* tiles;  // pass-B tiled stream (k_fibers.cu): per group, patient, sub-range: 8-slot tiles
  int64_t* tptr;         // [G x (K + 1)] first tile of each (group, patient) run
  uint16_t* twoff;       // [G x K x kWoS] tile offset of each sub-range inside its run
  int64_t nst = 0, nst_cap = 0, ntiles = 0;
  int64_t Jl = 0;        // labels = G * Jg >= J
  int sc_G = 1, sc_W = 4, sc_RS = 0, sc_ok = 0, sc_ranges = 1;
  int sc_FB = 32, sc_PB = 16, sc_NS = 3;  // pass-B stage: tiles (FB), patients (PB), ring slots (NS)
  int64_t sc_Js = 0, sc_Jg = 0;
  size_t sc_slot = 0, sc_smem = 0;
  void* layout_tmp;
  size_t layout_tmp_bytes = 0;
  int32_t* row_patient;  // non-smooth: [rows]
  int32_t* porder;       // [K] patient order of the thread-per-patient polar (ascending m_k)
  // non-smooth: feature-major (CSC) copy of X for the deterministic F_V gather (k_plain.cu)
  int64_t* csc_ptr;          // [J+1]
  int32_t* csc_row;          // [nnz] row of each entry, column order
  double* csc_val;           // [nnz]
  int64_t* csc_chunk;        // [2 x cap] entry range of each gather chunk (one column per chunk)
  int64_t* csc_chunk_first;  // [J+1] first chunk of each column
  double* csc_part;          // [cap x R] chunk partials
  void* csc_tmp;             // init-only scratch of the sort
  size_t csc_tmp_bytes = 0;
  int64_t csc_chunks = 0, csc_chunk_cap = 0;
  void* cub_temp;
  size_t cub_temp_bytes;
  int64_t* counts_scratch;
  double* fit_ring;    // device ring of per-iteration FIT values
  unsigned long long* diag;   // [kDiagSlots] rank-cut diagnostics (see DiagSlot)
  unsigned long long* steps;  // [4] inner ADMM steps of the H, W, V modes (last iteration) + zero count
  int own_inputs;      // copa_fit: CSR copied into the workspace
  // CUDA graph of one outer iteration (single rank, not profiling; copa_api.cu iterate_step)
  bool use_graph = true;
  bool graph_failed = false;
  int eager_done = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  // phase profiling (copa_set_profiling)
  bool profiling = false;
  std::vector<cudaEvent_t> events;
  std::vector<int> ev_phase;
  int ev_used = 0;
  double phase_ms[kPhases] = {0};
  int64_t phase_calls[kPhases] = {0};
  int64_t launches = 0;  // kernels launched by the iteration (counted while profiling)
};

// ------------------------------------------------------------------ device helpers
// Proximal maps (readings R-l1, R-l0, R-admm-sign). x = Z - D.
__device__ __forceinline__ double prox(int kind, double param, double rho, double x) {
  switch (kind) {
    case COPA_NONNEG: return x > 0.0 ? x : 0.0;
    case COPA_L1: {
      double a = fabs(x) - param / rho;
      return a > 0.0 ? copysign(a, x) : 0.0;
    }
    case COPA_NONNEG_L1: {
      double a = x - param / rho;
      return a > 0.0 ? a : 0.0;
    }
    case COPA_L0: return (x * x >= param) ? x : 0.0;
    default: return x;
  }
}

// Jacobi rotation of two rows x, y (a = x.x, b = y.y, c = x.y) that makes them orthogonal:
// x <- cs x - sn y, y <- sn x + cs y with tan(2 theta) = 2c / (b - a) (Hestenes). With d = (b - a)/2,
// h = sqrt(c^2 + d^2), u = |d| / h = cos(2 theta): cs = sqrt((1 + u)/2) = (1 + u) q and
// sn = sign(d) c / (2 h cs) = sign(d) c (1/h) q with q = 1/sqrt(2 (1 + u)) — two reciprocal square
// roots and no division or square root (the FP64 division and square root are long instruction
// sequences; this is the same rotation as t = sign(d) c / (|d| + h), cs = 1/sqrt(1 + t^2), sn = cs t).
__device__ __forceinline__ void jacobi_rot(double a, double b, double c, double& cs, double& sn) {
  const double d = 0.5 * (b - a);
  const double rh = rsqrt(fma(c, c, d * d));
  const double u = fabs(d) * rh;
  const double q = rsqrt(fma(2.0, u, 2.0));
  cs = (1.0 + u) * q;
  sn = copysign(1.0, d) * c * rh * q;
}

// Insert row a[0..q) into the upper-triangular Rf (q x q, row-major, stride ld) with Givens
// rotations, so that Rf^T Rf accumulates a a^T without ever forming a Gram matrix.
__device__ __forceinline__ void givens_insert(double* Rf, int ld, double* a, int q) {
  for (int j = 0; j < q; ++j) {
    double aj = a[j];
    if (aj == 0.0) continue;
    double r = Rf[j * ld + j];
    double h = hypot(r, aj);
    double c = r / h, s = aj / h;
    Rf[j * ld + j] = h;
    for (int t = j + 1; t < q; ++t) {
      double x = Rf[j * ld + t], y = a[t];
      Rf[j * ld + t] = c * x + s * y;
      a[t] = c * y - s * x;
    }
  }
}

// Rows of a Jacobi sweep whose squared norm is below kJacobiNegl2 times the total (the trace of
// the Gram, invariant under the rotations) are rounding residue of a rank-deficient factor: sigma_j
// below 1e-15 sqrt(trace) is far under both rank cuts (1e-10, 1e-6 sigma_1), and rotating them
// changes the other rows by ~1e-15 relative. They are left alone — otherwise residue rows keep an
// O(1) cosine to each other and the sweep never converges (all 40 sweeps for a rank-deficient
// tall factor, and a warp waits for its slowest patient).
// One-sided (Hestenes) Jacobi on the q row-vectors of Wm (q x q, stride ld): rotates pairs of
// rows until mutually orthogonal. Afterwards row j = sigma_j v_j where v_j are the right singular
// vectors of the upper-triangular factor whose rows were given (polar kernel).
__device__ __forceinline__ void jacobi_rows(double* Wm, int ld, int q) {
  const double tol = 2.220446049250313e-16 * (double)q;
  double tr = 0.0;  // trace of the Gram (invariant): residue-row threshold
  for (int i = 0; i < q * ld; ++i) tr = fma(Wm[i], Wm[i], tr);
  const double negl = kJacobiNegl2 * tr;
  for (int sweep = 0; sweep < 60; ++sweep) {
    int rotated = 0;
    for (int p = 0; p < q - 1; ++p) {
      for (int r = p + 1; r < q; ++r) {
        double a = 0.0, b = 0.0, c = 0.0;
        for (int i = 0; i < q; ++i) {
          double x = Wm[p * ld + i], y = Wm[r * ld + i];
          a = fma(x, x, a);
          b = fma(y, y, b);
          c = fma(x, y, c);
        }
        if (a <= negl || b <= negl) continue;
        if (fabs(c) <= tol * sqrt(a * b)) continue;
        rotated = 1;
        double cs, sn;
        jacobi_rot(a, b, c, cs, sn);
        for (int i = 0; i < q; ++i) {
          double x = Wm[p * ld + i], y = Wm[r * ld + i];
          Wm[p * ld + i] = cs * x - sn * y;
          Wm[r * ld + i] = sn * x + cs * y;
        }
      }
    }
    if (!rotated) break;
  }
}

// Uniform knot beta_idx of the gap-aware knot vector on [t1, tn] (reading R-spline-1).
__device__ __forceinline__ double knot(double t1, double tn, int l, int d, int idx) {
  if (idx <= d) return t1;
  if (idx >= l) return tn;
  int i = idx - d;
  return t1 + (tn - t1) * (double)i / (double)(l - d);
}

// The d+1 non-zero B-spline values N[0..d] of basis functions mu-d..mu at t (de Boor triangle;
// same functions as the paper's recursion P:358). Returns mu (the knot interval index).
__device__ __forceinline__ int spline_eval(double t, double t1, double tn, int l, int d, double* N) {
  int mu = d + (int)floor((t - t1) / (tn - t1) * (double)(l - d));
  if (mu < d) mu = d;
  if (mu > l - 1) mu = l - 1;
  while (mu > d && t < knot(t1, tn, l, d, mu)) --mu;
  while (mu < l - 1 && t >= knot(t1, tn, l, d, mu + 1)) ++mu;
  double left[kMaxDeg + 1], right[kMaxDeg + 1];
  N[0] = 1.0;
  for (int j = 1; j <= d; ++j) {
    left[j] = t - knot(t1, tn, l, d, mu + 1 - j);
    right[j] = knot(t1, tn, l, d, mu + j) - t;
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      double tmp = N[r] / (right[r + 1] + left[j - r]);
      N[r] = saved + right[r + 1] * tmp;
      saved = left[j - r] * tmp;
    }
    N[j] = saved;
  }
  return mu;
}

__device__ __forceinline__ void set_err(int* err, int bit) { atomicOr(err, bit); }

// Summary of one patient's singular-value ratios sigma_j / sigma_1 against a rank cut tau:
// smallest kept ratio (+inf if none), largest dropped ratio (0 if none), any ratio within a factor
// 100 of tau. ratio_note() folds one ratio in.
struct RatioDiag {
  double min_kept = INFINITY;
  double max_drop = 0.0;
  int near = 0;
  __device__ __forceinline__ void note(double ratio, bool kept, double tau) {
    if (kept) min_kept = fmin(min_kept, ratio);
    else max_drop = fmax(max_drop, ratio);
    if (tau > 0.0 && ratio >= 0.01 * tau && ratio <= 100.0 * tau) near = 1;
  }
};
// Accumulate into diag[base + 0..2]: one atomic set per call.
__device__ __forceinline__ void ratio_diag_commit(unsigned long long* diag, int base, const RatioDiag& d) {
  if (d.near) atomicAdd(diag + base, (unsigned long long)d.near);
  atomicMin(diag + base + 1, (unsigned long long)__double_as_longlong(d.min_kept));
  atomicMax(diag + base + 2, (unsigned long long)__double_as_longlong(d.max_drop));
}
// Warp-collective version (all 32 lanes call it; lanes with nothing to report pass a default RatioDiag).
__device__ __forceinline__ void ratio_diag_warp(unsigned long long* diag, int base, RatioDiag d) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d.min_kept = fmin(d.min_kept, __shfl_xor_sync(0xffffffffu, d.min_kept, o));
    d.max_drop = fmax(d.max_drop, __shfl_xor_sync(0xffffffffu, d.max_drop, o));
    d.near += __shfl_xor_sync(0xffffffffu, d.near, o);
  }
  if ((threadIdx.x & 31) == 0) ratio_diag_commit(diag, base, d);
}

// Inner-step counter of one ADMM row batch: warp sum, one atomic per warp (all lanes call it).
__device__ __forceinline__ void steps_warp(unsigned long long* counter, int steps) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) steps += __shfl_xor_sync(0xffffffffu, steps, o);
  if ((threadIdx.x & 31) == 0 && steps) atomicAdd(counter, (unsigned long long)steps);
}

// Per-row inner stop of reading R-inner-tol, accumulated like the oracle (no FMA contraction):
// pr += (zb - z)^2, du += (zb - zb_prev)^2, nz += zb^2; stop when max(pr, du) <= tol^2 nz.
struct RowResid {
  double pr = 0.0, du = 0.0, nz = 0.0;
  __device__ __forceinline__ void add(double zb_new, double z, double zb_prev) {
    const double e = __dsub_rn(zb_new, z), dz = __dsub_rn(zb_new, zb_prev);
    pr = __dadd_rn(pr, __dmul_rn(e, e));
    du = __dadd_rn(du, __dmul_rn(dz, dz));
    nz = __dadd_rn(nz, __dmul_rn(zb_new, zb_new));
  }
  __device__ __forceinline__ bool done(double tol) const {
    return tol > 0.0 && fmax(pr, du) <= __dmul_rn(__dmul_rn(tol, tol), nz);
  }
};

// Opt a kernel into the full 227 KB of dynamic shared memory, once per (kernel, device).
template <auto Fn>
inline void max_smem_attr(const Handle& h, int bytes = 227 * 1024) {
  static unsigned long long done = 0;  // bit per device ordinal (< 64)
  const unsigned long long bit = 1ull << (h.dev & 63);
  if (__atomic_load_n(&done, __ATOMIC_ACQUIRE) & bit) return;
  cudaFuncSetAttribute(Fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  __atomic_fetch_or(&done, bit, __ATOMIC_ACQ_REL);
}

// ------------------------------------------------------------------ launchers
// init
void launch_validate(Handle& h, bool vals = true);
void launch_validate_vals(Handle& h, int64_t e0 = 0, int64_t e1 = -1);  // values [e0, e1)
void launch_count_fibers(Handle& h, int64_t* counts_out /*[K+1], counts at [k+1]*/, unsigned long long* hist);
void launch_basis(Handle& h);
void launch_build_fibers(Handle& h, int64_t kb = 0, int64_t ke = -1);  // patients [kb, ke)
void launch_count_groups(Handle& h, int32_t* gcnt /*[G][K]*/, int32_t* tcnt /*[G][K]*/);
void launch_row_patient(Handle& h);
void launch_sumsq(Handle& h, double* out);
// iteration
int launch_spmm(Handle& h);
int launch_fh(Handle& h);
int launch_admm_H(Handle& h);
int launch_scatter(Handle& h);
int launch_admm_V(Handle& h);
int launch_fit(Handle& h);
void launch_count_zeros(Handle& h);  // zero entries of V̄ -> steps[3]
// reductions: C (R x R) = sum_s A(s,:)^T (B(s,:) * w(s,:)); wsrc: 0 none, 1 W rows by patient of s
int launch_gram(Handle& h, const double* A, const double* B, int64_t nrows, int wmode, double* C);
// U rows of patients [k0, k1) into U (row i of the shard at U[(i - prp[k0]) R])
void launch_U(Handle& h, double* U, int64_t k0, int64_t k1);
// fiber passes (k_fibers.cu)
void launch_spmm_fibers(Handle& h);   // pass A (k_passA.cu)
void launch_relabel_V(Handle& h);
void launch_layoutA(Handle& h);
void launch_build_tiles(Handle& h);
int64_t tiles_cap(const Handle& h);
size_t plan_cub_bytes(const Handle& h);
int64_t plan_tmp_words(const Handle& h);
bool plan_streams_device(Handle& h, const int32_t* gcnt, const int32_t* tcnt, int64_t* tmp, int64_t* gtotal);
inline uint32_t tile_bytes_host(int l) { return 32u + 64u * (uint32_t)l; }
void plan_passA(Handle& h);
void launch_passA_ranges(Handle& h);
int launch_scatter_fibers(Handle& h);
bool scatter_smem_ok(const Handle& h);
void plan_scatter(Handle& h);
void compute_relabel(int64_t J, int ranges, const unsigned long long* hist, int32_t* perm, int32_t* inv, int64_t* Js);
int64_t stage_cap(const Handle& h);                                // pass-B stage table bound
int64_t stage_tab_cap(const Handle& h);                            // pass-B sub-run table bound
void launch_stage_tab(Handle& h);
// host: gptr (G x (K+1), absolute) from per-group counts; stage table; pass-B patient ranges

// wide per-patient dense kernels (k_dense.cu)
bool polar_wide_ok(const Handle& h);
// general path (k_plain.cu)
int launch_polar_warp(Handle& h);
bool polar_thread_ok(const Handle& h);
int plan_polar_order(Handle& h);  // 0 ok, -1 CUDA error
int launch_passB_warp(Handle& h);
size_t csc_temp_bytes(const Handle& h);
int build_csc(Handle& h);  // 0 ok, -1 CUDA error, -2 chunk table overflow
int launch_scatter_csc(Handle& h, const double* Nrows);
// row-projection path (k_rowproj.cu): smooth l > kMaxFiberL
void launch_basis_warp(Handle& h);
int launch_rowproj_P(Handle& h);
int launch_rowproj_N(Handle& h);
int launch_polar_wide(Handle& h);
int launch_passB_wide(Handle& h);

}  // namespace copa
