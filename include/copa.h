/*
 * copa.h — C ABI of the B200-native COPA hot path (libcopa.so).
 *
 * COPA = constrained PARAFAC2 fitted by AO-ADMM (arXiv 1803.04572, "PAPER.md").
 * The library runs the body of Algorithm 1's outer loop ("Alg.1
 * l.3-l.20") plus the FIT metric on one B200, FP64 throughout:
 *
 *   per patient k:   Q_k  = polar factor of X'_k V S_k H^T          (Alg.1 l.4-5, Eq. solv_Q)
 *                    Y_k  = Q_k^T X'_k   (implicit, never written)   (Alg.1 l.6)
 *   per mode n=H,W,V: G = Hadamard of Grams, F = MTTKRP of Y,        (Alg.1 l.11-12)
 *                    rho, L = chol(G + rho I), n_inner ADMM steps      (Alg.1 l.13-19)
 *                    with the element-wise prox of the constraint
 *   smoothness:      X'_k = C_k^T X_k, C_k = orthonormal basis of the
 *                    patient's B-spline ("M-spline") basis M_k
 *
 * Readings of ambiguous passages are listed in DESIGN.md §2 (R-* ids cited below).
 *
 * Conventions
 *   - All matrices are row-major FP64. H is R x R, V is J x R, W is K x R (row k = diag(S_k)).
 *   - The factors the library iterates on are the AUXILIARY variables H̄, V̄, W̄ (reading R-aux);
 *     duals D are kept in the scaled form (reading R-admm-sign).
 *   - Device pointers are CUDA device addresses on the current device; host pointers are
 *     ordinary (ideally pinned) host memory. Each argument states which it takes.
 *   - Ownership: the caller owns every buffer (inputs, workspace, stream). The library never
 *     allocates device memory and borrows the inputs and the workspace for the handle's
 *     lifetime; they must stay valid and unmodified until copa_destroy.
 *   - Errors: every call returns a copa_status and never throws; copa_last_error() returns a
 *     thread-local message for the last failing call. Device-side failures (Cholesky pivot,
 *     non-finite FIT) are detected at the end of copa_iterate.
 */
#ifndef COPA_H
#define COPA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  COPA_OK = 0,
  COPA_E_ARG = -1,         /* bad option / null pointer / R < 1 / smooth without times */
  COPA_E_SHAPE = -2,       /* CSR not monotone, column >= J, duplicate column in a row, times not increasing */
  COPA_E_NONFINITE = -3,   /* NaN/Inf in the inputs or a non-finite FIT */
  COPA_E_CHOL = -4,        /* non-positive pivot in chol(G + rho I) (Alg.1 l.14) */
  COPA_E_DEGENERATE = -5,  /* trace(G) = 0 with automatic rho (reading R-rho) */
  COPA_E_CUDA = -6,        /* CUDA runtime error */
  COPA_E_COMM = -7,        /* the allreduce callback returned non-zero */
  COPA_E_WORKSPACE = -8,   /* workspace too small / misaligned */
  COPA_E_UNSUPPORTED = -9  /* sizes outside this build's kernel limits (see copa_limits) */
} copa_status;

/* Proximal operator of each factor's constraint (reading R-l1, R-l0). */
typedef enum {
  COPA_NONE = 0,      /* identity */
  COPA_NONNEG = 1,    /* max(0, x) */
  COPA_L1 = 2,        /* sign(x) max(0, |x| - lambda/rho)  P:480 (sign kept) */
  COPA_NONNEG_L1 = 3, /* max(0, x - lambda/rho)          exact prox of lambda|.|_1 + indicator(>=0) */
  COPA_L0 = 4         /* x * [x^2 >= mu]                 P:466-470, param = mu */
} copa_kind;

typedef struct {
  int32_t kind;  /* copa_kind */
  double param;  /* lambda (L1, NONNEG_L1) or mu (L0); ignored otherwise */
} copa_constraint;

/* One shard of the irregular tensor {X_k}: a contiguous range of patients (PAPER.md:119,
 * "each slice X_k in R^{I_k x J}"), stored CSR-per-patient. ALL POINTERS ARE DEVICE POINTERS. */
typedef struct {
  int64_t K_local;                 /* patients in this shard (>= 0) */
  int64_t K_global;                /* patients over all ranks */
  int64_t J;                       /* features (columns), 1 <= J <= 65535 */
  int32_t R;                       /* target rank, 1 <= R <= 64 */
  int64_t rows;                    /* sum_k I_k of the shard = patient_row_ptr[K_local] */
  int64_t nnz;                     /* nonzeros of the shard = row_ptr[rows] */
  const int64_t* patient_row_ptr;  /* [K_local+1], 0-based, non-decreasing, I_k >= 1 */
  const int64_t* row_ptr;          /* [rows+1], 0-based, non-decreasing */
  const int32_t* col;              /* [nnz], 0 <= col < J, distinct within a row */
  const double* val;               /* [nnz], finite */
  const double* visit_time;        /* [rows], strictly increasing per patient; NULL unless smooth_l > 0 */
} copa_problem;

/* Allreduce(sum) of `count` doubles at device address `buf`, in place, enqueued on `stream`
 * (a cudaStream_t). Called by the library twice per outer iteration
 * and once at init; NULL means a single rank. Return 0 on success. */
typedef int (*copa_allreduce_fn)(double* buf, int64_t count, void* stream, void* ctx);

typedef struct {
  copa_constraint on_H, on_W, on_V;  /* W rows are diag(S_k) */
  int32_t smooth_l;                  /* 0 = off; l = number of basis functions (reading R-spline-3) */
  int32_t smooth_degree;             /* spline degree d (default 3, reading R-spline-3) */
  double rho;                        /* > 0: fixed rho for every mode; <= 0: trace(G)/R per mode (Alg.1 l.13) */
  int32_t admm_inner;                /* inner ADMM steps per mode (reading R-inner); >= 1 */
  double rank_tol;                   /* polar rank cut tau: sigma > tau*sigma_1 (reading R-polar-3), e.g. 1e-10 */
  double basis_tol;                  /* basis rank cut (reading R-spline-4), e.g. 1e-6 */
  double admm_tol;                   /* inner stop ("while convergence criterion is not met", reading
                                        R-inner-tol): 0 = exactly admm_inner steps; > 0 = each factor row stops
                                        after the step where max(|row(Zbar) - row(Z)|, |row(Zbar) - previous
                                        row(Zbar)|) <= admm_tol |row(Zbar)| (Euclidean), at most admm_inner */
  const double* H0;                  /* DEVICE, R x R initial H (copied at init) */
  const double* V0;                  /* DEVICE, J x R initial V (identical on all ranks) */
  const double* W0_local;            /* DEVICE, K_local x R initial W rows of this shard */
  copa_allreduce_fn allreduce;       /* NULL for a single rank */
  void* allreduce_ctx;
  void* stream;                      /* cudaStream_t the library enqueues on (NULL = legacy default) */
} copa_options;

typedef struct copa_handle copa_handle;

typedef struct {
  double fit;           /* FIT after the last completed outer iteration */
  double rho[3];        /* rho used for H, W, V in the last iteration */
  double normX;         /* sum of squares of all values (all ranks) */
  int64_t iterations;   /* outer iterations completed */
  int64_t fibers;       /* (patient, feature) pairs of the shard (smooth path) */
  int64_t state_rows;   /* rows of the per-patient state (P', Q~) */
  int64_t rank_deficient; /* patients with r_k < min(m_k, R) in the last iteration (shard) */
  double sparsity_V;    /* SPARSITY(V) = zero entries / size */
  int64_t inner_steps[3]; /* ADMM inner steps of the H, W, V modes in the last iteration, summed over the
                             factor rows (W: this shard's rows); admm_inner x rows when admm_tol = 0 */
  /* Parity diagnostics of the two rank cuts (SURVEY 8(c) parity protocol; readings R-polar-3 and
   * R-spline-4), ratios sigma_j / sigma_1. Polar: accumulated over all iterations since init, per
   * (patient, iteration); basis: at init. near = count with some ratio within a factor 100 of the
   * cut (tau/100 <= ratio <= 100 tau); min_kept = smallest kept ratio (1 if none); max_dropped =
   * largest dropped ratio (0 if none). */
  int64_t polar_near;
  double polar_min_kept, polar_max_dropped;
  int64_t basis_near;
  double basis_min_kept, basis_max_dropped;
  int64_t tiles;        /* 8-slot tiles of pass B's tiled stream (smooth path, shard; 0 otherwise) */
} copa_stats;

/* Kernel limits of this build: R <= max_R, q = min(m_k, R) <= max_q (warp polar), smooth_l <= max_smooth_l. */
typedef struct { int32_t max_R; int32_t max_q; int32_t max_smooth_l; int64_t max_J; } copa_limits;
void copa_get_limits(copa_limits* out);

/* Bytes of device workspace needed for this problem (may run a counting kernel on
 * options->stream and synchronise it). problem/options: host structs with device pointers. */
copa_status copa_workspace_size(const copa_problem* problem, const copa_options* options, size_t* bytes);

/* Validate inputs, build the layout (smooth: per-patient basis C_k and projected fibers
 * X'_k = C_k^T X_k), copy H0/V0/W0 into the working factors, zero the duals.
 * workspace: DEVICE pointer, 256-byte aligned, >= copa_workspace_size bytes. */
copa_status copa_init(const copa_problem* problem, const copa_options* options, void* workspace, size_t bytes,
                      copa_handle** out);

/* Run n_outer outer iterations (Alg.1 l.3-l.20) on the handle's stream. fit_host: HOST
 * array of n_outer doubles receiving FIT after each iteration, or NULL. Synchronises the
 * stream once at the end (error check). */
copa_status copa_iterate(copa_handle* h, int32_t n_outer, double* fit_host);

/* Outer loop with a stop ("while convergence criterion is not met", reading R-outer-tol): runs
 * up to max_outer iterations and stops after iteration t >= 2 of this call when
 * |FIT_t - FIT_{t-1}| < outer_tol * max(|FIT_{t-1}|, 1). fit_host: HOST array of max_outer doubles
 * (or NULL); n_done (HOST, may be NULL) receives the number of iterations run. Synchronises the
 * stream after every iteration (the stop is a host decision on the device-computed FIT). */
copa_status copa_iterate_until(copa_handle* h, int32_t max_outer, double outer_tol, double* fit_host,
                               int32_t* n_done);

/* Factors of record (the auxiliary variables, Alg.1 l.21). Each pointer may be a DEVICE or
 * HOST pointer (detected with cudaPointerGetAttributes) or NULL to skip.
 * H: R x R, V: J x R, W_local: K_local x R. */
copa_status copa_get_factors(copa_handle* h, double* H, double* V, double* W_local);

/* Duals (scaled form) with the same layout/pointer rules as copa_get_factors. */
copa_status copa_get_duals(copa_handle* h, double* DH, double* DV, double* DW_local);

/* Checkpoint / resume. The state that carries an outer iteration into the next (Alg.1 l.3-l.20;
 * Q_k is recomputed from it by the Procrustes step, l.4): the working factors, the scaled duals,
 * and the two Grams the next H-mode reads (l.11: V^T V, and W^T W summed over ranks). Every
 * pointer is a DEVICE or HOST pointer (as in copa_get_factors); W_local/DW_local may be NULL when
 * K_local = 0. Shapes: H, DH, WtW, VtV R x R; V, DV J x R; W_local, DW_local K_local x R. */
typedef struct {
  double *H, *V, *W_local, *DH, *DV, *DW_local, *WtW, *VtV;
  int64_t iterations; /* outer iterations completed */
} copa_state;

/* Copy the state out (synchronises the stream). */
copa_status copa_get_state(copa_handle* h, const copa_state* out);

/* Load a state into an initialised handle (same problem, options and rank layout). WtW and VtV may
 * be NULL: they are then recomputed from W and V (W^T W through the allreduce callback, so every
 * rank must call it), equal to the saved ones up to summation order. With all eight arrays the
 * resumed run continues bit-identically. */
copa_status copa_set_state(copa_handle* h, const copa_state* in);

/* U_k = C_k Q_k H (smooth) or Q_k H (Alg.1 l.24), stacked over the shard's rows:
 * U_rows is a DEVICE or HOST pointer to rows x R doubles. */
copa_status copa_get_U(copa_handle* h, double* U_rows);

copa_status copa_get_stats(copa_handle* h, copa_stats* out);

/* init + iterate(n_outer) + get_factors + destroy with HOST inputs (the end-to-end call):
 * problem pointers are HOST pointers here; the library copies them into the workspace
 * (so workspace must be >= copa_fit_workspace_size). Outputs are HOST pointers (or NULL).
 * copa_fit_workspace_size reads the host patient_row_ptr, row_ptr and col arrays (it counts the
 * distinct (patient, feature) pairs the smooth path stores, with host threads); val, visit_time and
 * the option arrays are not read. */
copa_status copa_fit_workspace_size(const copa_problem* host_problem, const copa_options* host_options,
                                    size_t* bytes);
copa_status copa_fit(const copa_problem* host_problem, const copa_options* host_options, void* workspace,
                     size_t bytes, int32_t n_outer, double* fit_host, double* H_out, double* V_out,
                     double* W_local_out);

void copa_destroy(copa_handle* h);
const char* copa_last_error(void);

/* Debug access to per-patient state (parity tests): copies the shard's state rows into
 * DEVICE or HOST buffers (NULL to skip): P' (state_rows x R), Q~ (state_rows x R),
 * m (K_local int32), srow (K_local+1 int64 state-row offsets), rank (K_local int32). */
copa_status copa_debug_state(copa_handle* h, double* Pp, double* Qt, int32_t* m, int64_t* srow, int32_t* rank);

/* Phase timing for measurement (bench.py): when on, copa_iterate records CUDA events around
 * each phase of the iteration on the library stream. Turning it on resets the accumulators. */
copa_status copa_set_profiling(copa_handle* h, int32_t on);
/* Accumulated milliseconds and call counts per phase (arrays of n entries, NULL to skip),
 * the number of phases, and the number of kernels the iterations launched while profiling.
 * Synchronises the handle's stream. */
copa_status copa_get_phase_times(copa_handle* h, double* ms, int64_t* calls, int32_t n, int32_t* n_phases,
                                 int64_t* launches);
const char* copa_phase_name(int32_t i);

#ifdef __cplusplus
}
#endif
#endif /* COPA_H */
