/*
 * copa_oracle.c — ORACLE (test infrastructure; NOT the product path).
 *
 * A plain, slow, serial FP64 CPU implementation of one COPA outer iteration
 * (Algorithm 1 of arXiv 1803.04572) with the readings fixed in
 * DESIGN.md §2. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may call it. It shares no code with the CUDA path
 * (paper_1803_04572_b200/csrc); the only common module is synthgen/ (input synthesis).
 *
 * It deliberately follows the paper's definitions literally:
 *   - Procrustes (Alg.1 l.4-5): SVD of A_k = X'_k V S_k H^T by one-sided
 *     Jacobi (an orthogonal-transformation SVD), Q_k = U_r V_r^T;
 *   - Y_k = Q_k^T X'_k materialised per patient (Alg.1 l.6);
 *   - the three MTTKRPs as Y_(n) times the Khatri-Rao product, entry by entry in
 *     Kolda-Bader order (Alg.1 l.12);
 *   - G = Hadamard of Grams (l.11), rho = trace(G)/R (l.13), L = chol(G+rho I) (l.14),
 *     inner ADMM (l.15-18) with the closed-form proximal maps;
 *   - FIT per patient with U_k = C_k Q_k H.
 * Smoothness: Cox-de Boor basis on gap-aware knots, C_k = left singular
 * vectors of M_k (rank-cut tau_basis), X'_k = C_k^T X_k.
 *
 * Parity pins: tests/test_oracle_pins.py (P1-P18 of SURVEY §8(c)).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { K_NONE = 0, K_NONNEG = 1, K_L1 = 2, K_NONNEG_L1 = 3, K_L0 = 4 };
enum { OR_OK = 0, OR_E_ARG = -1, OR_E_CHOL = -4, OR_E_DEGENERATE = -5, OR_E_NONFINITE = -3, OR_E_NOMEM = -10 };

typedef struct {
  int64_t K, J;
  int32_t R;
  const int64_t* patient_row_ptr; /* [K+1] */
  const int64_t* row_ptr;         /* [rows+1] */
  const int32_t* col;             /* [nnz] */
  const double* val;              /* [nnz] */
  const double* times;            /* [rows] or NULL */
} or_problem;

typedef struct {
  int32_t kind_H, kind_W, kind_V;
  double param_H, param_W, param_V;
  int32_t smooth_l, smooth_d;
  double rho;        /* > 0 fixed; <= 0: trace(G)/R */
  int32_t n_inner;
  double tau_polar;  /* rank cut of A_k: sigma > tau_polar * sigma_1 */
  double tau_basis;  /* rank cut of M_k */
  double admm_tol;   /* > 0: per-row inner stop (reading R-inner-tol); 0: exactly n_inner steps */
} or_options;

/* ---------------------------------------------------------------- prox */
/* Element-wise proximal maps on x = Z - D (scaled ADMM, reading R-admm-sign). */
double oracle_prox(int32_t kind, double param, double rho, double x) {
  switch (kind) {
    case K_NONE: return x;
    case K_NONNEG: return x > 0 ? x : 0.0;                       /* P:492 max(0, .) */
    case K_L1: {                                                 /* P:480 soft threshold, sign kept */
      double a = fabs(x) - param / rho;
      return a > 0 ? copysign(a, x) : 0.0;
    }
    case K_NONNEG_L1: {                                          /* prox of lambda|.|_1 + indicator(>=0) */
      double a = x - param / rho;
      return a > 0 ? a : 0.0;
    }
    case K_L0: return (x * x >= param) ? x : 0.0;                /* P:466-470 hard threshold, mu = param */
    default: return NAN;
  }
}

/* ------------------------------------------------- B-spline basis */
/* Cox-de Boor recursion exactly as P:358; 0/0 := 0; degree-0 base case on half-open
 * intervals [beta_b, beta_{b+1}), the last non-empty interval closed at t_n (reading R-spline-2). */
static double bspline_rec(const double* beta, int b, int d, double t, int last) {
  if (d == 0) {
    if (beta[b] <= t && t < beta[b + 1]) return 1.0;
    if (b == last && t == beta[b + 1]) return 1.0;
    return 0.0;
  }
  double left = 0.0, right = 0.0;
  double den1 = beta[b + d] - beta[b];
  double den2 = beta[b + d + 1] - beta[b + 1];
  if (den1 > 0) left = (t - beta[b]) / den1 * bspline_rec(beta, b, d - 1, t, last);
  if (den2 > 0) right = (beta[b + d + 1] - t) / den2 * bspline_rec(beta, b + 1, d - 1, t, last);
  return left + right;
}

/* Gap-aware knots on [t_1, t_n] (reading R-spline-1): (d+1)-fold boundary
 * knots, l-d-1 interior knots evenly spaced in days. beta has l+d+1 entries. */
void oracle_knots(double t1, double tn, int32_t l, int32_t d, double* beta) {
  for (int i = 0; i <= d; ++i) beta[i] = t1;
  for (int i = 1; i <= l - d - 1; ++i) beta[d + i] = t1 + (tn - t1) * (double)i / (double)(l - d);
  for (int i = 0; i <= d; ++i) beta[l + i] = tn;
}

/* M (n x l, row-major): M(i,b) = m_{b,d}(t_i) for the patient's visit times t[0..n-1]. */
void oracle_bspline_matrix(const double* t, int64_t n, int32_t l, int32_t d, double* M) {
  double beta[64];
  oracle_knots(t[0], t[n - 1], l, d, beta);
  for (int64_t i = 0; i < n; ++i)
    for (int b = 0; b < l; ++b) M[i * l + b] = bspline_rec(beta, b, d, t[i], l - 1);
}

/* -------------------------------------------------------- SVD (one-sided Jacobi) */
/* Thin SVD of an m x n row-major matrix A by Hestenes one-sided Jacobi (orthogonal
 * rotations applied to the columns of A, or of A^T when m < n).
 * Outputs, p = min(m,n): U (m x p), s (p, descending), Vt... as V (n x p). Returns sweeps used. */
int oracle_svd(int64_t m, int64_t n, const double* A, double* U, double* s, double* V) {
  int trans = m < n;
  int64_t rows = trans ? n : m, cols = trans ? m : n; /* work on B = A or A^T: rows x cols, rows >= cols */
  double* B = (double*)malloc(sizeof(double) * (size_t)(rows * cols));
  double* W = (double*)malloc(sizeof(double) * (size_t)(cols * cols)); /* accumulated rotations */
  if (!B || !W) { free(B); free(W); return -1; }
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) B[i * cols + j] = trans ? A[j * n + i] : A[i * n + j];
  for (int64_t i = 0; i < cols; ++i)
    for (int64_t j = 0; j < cols; ++j) W[i * cols + j] = (i == j) ? 1.0 : 0.0;
  const double tol = DBL_EPSILON * (double)rows;
  int sweep = 0;
  for (; sweep < 80; ++sweep) {
    int rotated = 0;
    for (int64_t p = 0; p < cols - 1; ++p) {
      for (int64_t q = p + 1; q < cols; ++q) {
        double a = 0, b = 0, c = 0;
        for (int64_t i = 0; i < rows; ++i) {
          double x = B[i * cols + p], y = B[i * cols + q];
          a += x * x; b += y * y; c += x * y;
        }
        if (a == 0.0 || b == 0.0) continue;
        if (fabs(c) <= tol * sqrt(a * b)) continue;
        rotated = 1;
        double zeta = (b - a) / (2.0 * c);
        double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (int64_t i = 0; i < rows; ++i) {
          double x = B[i * cols + p], y = B[i * cols + q];
          B[i * cols + p] = cs * x - sn * y;
          B[i * cols + q] = sn * x + cs * y;
        }
        for (int64_t i = 0; i < cols; ++i) {
          double x = W[i * cols + p], y = W[i * cols + q];
          W[i * cols + p] = cs * x - sn * y;
          W[i * cols + q] = sn * x + cs * y;
        }
      }
    }
    if (!rotated) break;
  }
  /* singular values = column norms; sort descending (selection sort, stable on ties) */
  double* nrm = (double*)malloc(sizeof(double) * (size_t)cols);
  int64_t* ord = (int64_t*)malloc(sizeof(int64_t) * (size_t)cols);
  for (int64_t j = 0; j < cols; ++j) {
    double acc = 0;
    for (int64_t i = 0; i < rows; ++i) acc += B[i * cols + j] * B[i * cols + j];
    nrm[j] = sqrt(acc);
    ord[j] = j;
  }
  for (int64_t a = 0; a < cols; ++a) {
    int64_t best = a;
    for (int64_t b = a + 1; b < cols; ++b)
      if (nrm[ord[b]] > nrm[ord[best]]) best = b;
    int64_t tmp = ord[a]; ord[a] = ord[best]; ord[best] = tmp;
  }
  /* left vectors of B = normalised columns; right vectors = W columns */
  double* LU = trans ? V : U; /* left singular vectors of B are right ones of A when transposed */
  double* RV = trans ? U : V;
  int64_t lrows = rows, rrows = cols;
  for (int64_t a = 0; a < cols; ++a) {
    int64_t j = ord[a];
    s[a] = nrm[j];
    for (int64_t i = 0; i < lrows; ++i) LU[i * cols + a] = nrm[j] > 0 ? B[i * cols + j] / nrm[j] : 0.0;
    for (int64_t i = 0; i < rrows; ++i) RV[i * cols + a] = W[i * cols + j];
  }
  free(nrm); free(ord); free(B); free(W);
  return sweep;
}

/* Partial-isometry polar factor (P:205 read as R-polar-1/2): Q = U_r V_r^T with
 * r = #{sigma_i > tau * sigma_1}. A is m x n; Q is m x n. Returns r. */
int oracle_polar(int64_t m, int64_t n, const double* A, double tau, double* Q) {
  int64_t p = m < n ? m : n;
  double* U = (double*)malloc(sizeof(double) * (size_t)(m * p));
  double* V = (double*)malloc(sizeof(double) * (size_t)(n * p));
  double* s = (double*)malloc(sizeof(double) * (size_t)p);
  oracle_svd(m, n, A, U, s, V);
  int r = 0;
  if (p > 0 && s[0] > 0)
    for (int64_t a = 0; a < p; ++a) if (s[a] > tau * s[0]) ++r;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0;
      for (int a = 0; a < r; ++a) acc += U[i * p + a] * V[j * p + a];
      Q[i * n + j] = acc;
    }
  free(U); free(V); free(s);
  return r;
}

/* ---------------------------------------------------- Cholesky */
/* In-place lower Cholesky of an R x R SPD matrix (row-major); returns 0 or the failing pivot+1. */
int oracle_cholesky(int32_t R, double* A) {
  for (int j = 0; j < R; ++j) {
    double d = A[j * R + j];
    for (int k = 0; k < j; ++k) d -= A[j * R + k] * A[j * R + k];
    if (!(d > 0)) return j + 1;
    d = sqrt(d);
    A[j * R + j] = d;
    for (int i = j + 1; i < R; ++i) {
      double v = A[i * R + j];
      for (int k = 0; k < j; ++k) v -= A[i * R + k] * A[j * R + k];
      A[i * R + j] = v / d;
    }
    for (int k = j + 1; k < R; ++k) A[j * R + k] = 0.0;
  }
  return 0;
}
/* Solve (L L^T) x = b in place, L lower (l.15: (L^T)^-1 L^-1 (.)). */
void oracle_chol_solve(int32_t R, const double* L, double* x) {
  for (int i = 0; i < R; ++i) {
    double v = x[i];
    for (int k = 0; k < i; ++k) v -= L[i * R + k] * x[k];
    x[i] = v / L[i * R + i];
  }
  for (int i = R - 1; i >= 0; --i) {
    double v = x[i];
    for (int k = i + 1; k < R; ++k) v -= L[k * R + i] * x[k];
    x[i] = v / L[i * R + i];
  }
}

/* ------------------------------------------------------------- ADMM (l.10-l.19) */
/* One mode: given F (n x R), G (R x R), the auxiliary Zbar and dual D (n x R, updated in
 * place), run rho, chol, and up to n_inner steps of
 *   Z = (F + rho (Zbar + D)) (G + rho I)^-1 ; Zbar = prox(Z - D) ; D = D + Zbar - Z.
 * The least-squares step acts on each row separately and the prox is element-wise, so the rows
 * are independent ADMM problems sharing G. Inner stop ("while convergence
 * criterion is not met", reading R-inner-tol): tol = 0 runs exactly n_inner steps; tol > 0 stops
 * a row after the step where max(||Zbar - Z||, ||Zbar - Zbar_prev||) <= tol ||Zbar|| (primal
 * residual and change of the auxiliary row, Euclidean norms, compared squared), at most n_inner.
 * steps (may be NULL) receives the number of steps of each row.
 * Returns OR_OK / error; rho_out receives the step size used. */
int oracle_admm_mode_tol(int64_t n, int32_t R, const double* F, const double* G, double rho_fixed, int32_t n_inner,
                         int32_t kind, double param, double tol, double* Zbar, double* D, double* rho_out,
                         int32_t* steps) {
  double rho = rho_fixed;
  if (!(rho > 0)) {
    double tr = 0;
    for (int i = 0; i < R; ++i) tr += G[i * R + i];
    rho = tr / R; /* Alg.1 l.13 */
    if (!(rho > 0)) return OR_E_DEGENERATE;
  }
  if (rho_out) *rho_out = rho;
  double* L = (double*)malloc(sizeof(double) * (size_t)R * R);
  memcpy(L, G, sizeof(double) * (size_t)R * R);
  for (int i = 0; i < R; ++i) L[i * R + i] += rho;
  if (oracle_cholesky(R, L)) { free(L); return OR_E_CHOL; }
  double* z = (double*)malloc(sizeof(double) * (size_t)R);
  for (int64_t row = 0; row < n; ++row) {
    int it = 0;
    while (it < n_inner) {
      for (int r = 0; r < R; ++r) z[r] = F[row * R + r] + rho * (Zbar[row * R + r] + D[row * R + r]);
      oracle_chol_solve(R, L, z);
      double pr = 0, du = 0, nz = 0;
      for (int r = 0; r < R; ++r) {
        double zb = oracle_prox(kind, param, rho, z[r] - D[row * R + r]);
        double dz = zb - Zbar[row * R + r];
        Zbar[row * R + r] = zb;
        D[row * R + r] += zb - z[r];
        pr += (zb - z[r]) * (zb - z[r]);
        du += dz * dz;
        nz += zb * zb;
      }
      ++it;
      if (tol > 0 && (pr > du ? pr : du) <= tol * tol * nz) break;
    }
    if (steps) steps[row] = it;
  }
  free(z); free(L);
  return OR_OK;
}

int oracle_admm_mode(int64_t n, int32_t R, const double* F, const double* G, double rho_fixed, int32_t n_inner,
                     int32_t kind, double param, double* Zbar, double* D, double* rho_out) {
  return oracle_admm_mode_tol(n, R, F, G, rho_fixed, n_inner, kind, param, 0.0, Zbar, D, rho_out, NULL);
}

/* SPARSITY(V) = nz(V) / size(V), nz = number of zero elements. */
double oracle_sparsity(int64_t n, const double* V) {
  int64_t z = 0;
  for (int64_t i = 0; i < n; ++i) z += V[i] == 0.0;
  return n > 0 ? (double)z / (double)n : 0.0;
}

/* ----------------------------------------------------------- per-patient pieces */
/* Basis of range(M_k): C (n x l, row-major, first lp columns used, rest 0).
 * Returns lp = #{sigma_b > tau * sigma_1}. */
int oracle_patient_basis(const double* t, int64_t n, int32_t l, int32_t d, double tau, double* C) {
  double* M = (double*)malloc(sizeof(double) * (size_t)(n * l));
  int64_t p = n < l ? n : l;
  double* U = (double*)malloc(sizeof(double) * (size_t)(n * p));
  double* V = (double*)malloc(sizeof(double) * (size_t)(l * p));
  double* s = (double*)malloc(sizeof(double) * (size_t)p);
  oracle_bspline_matrix(t, n, l, d, M);
  oracle_svd(n, l, M, U, s, V);
  int lp = 0;
  if (p > 0 && s[0] > 0)
    for (int64_t a = 0; a < p; ++a) if (s[a] > tau * s[0]) ++lp;
  for (int64_t i = 0; i < n; ++i)
    for (int b = 0; b < l; ++b) C[i * l + b] = b < lp ? U[i * p + b] : 0.0;
  free(M); free(U); free(V); free(s);
  return lp;
}

/* Dense X'_k restricted to the patient's distinct columns (sorted ascending).
 * Xp (m x ncols) where m = lp (smooth, X' = C^T X) or I_k (plain). cols gets the column ids. */
static int64_t patient_dense(const or_problem* P, int64_t k, const double* Ck, int32_t l, int32_t m, int32_t* mark,
                             int32_t* cols, double** Xp_out) {
  int64_t r0 = P->patient_row_ptr[k], r1 = P->patient_row_ptr[k + 1];
  int64_t nc = 0;
  for (int64_t i = r0; i < r1; ++i)
    for (int64_t e = P->row_ptr[i]; e < P->row_ptr[i + 1]; ++e)
      if (mark[P->col[e]] < 0) { mark[P->col[e]] = 0; cols[nc++] = P->col[e]; }
  /* sort column ids (insertion sort; patients are small) */
  for (int64_t a = 1; a < nc; ++a) {
    int32_t v = cols[a];
    int64_t b = a - 1;
    while (b >= 0 && cols[b] > v) { cols[b + 1] = cols[b]; --b; }
    cols[b + 1] = v;
  }
  for (int64_t a = 0; a < nc; ++a) mark[cols[a]] = (int32_t)a;
  double* Xp = (double*)calloc((size_t)(m * nc > 0 ? m * nc : 1), sizeof(double));
  for (int64_t i = r0; i < r1; ++i)
    for (int64_t e = P->row_ptr[i]; e < P->row_ptr[i + 1]; ++e) {
      int64_t jl = mark[P->col[e]];
      double x = P->val[e];
      if (Ck) {
        for (int a = 0; a < m; ++a) Xp[a * nc + jl] += Ck[(i - r0) * l + a] * x; /* X' = C^T X */
      } else {
        Xp[(i - r0) * nc + jl] = x;
      }
    }
  for (int64_t a = 0; a < nc; ++a) mark[cols[a]] = -1;
  *Xp_out = Xp;
  return nc;
}

/* O.0: normX; smooth bases C (rows x l) and m_k; state row offsets. */
int oracle_init(const or_problem* P, const or_options* o, double* C, int32_t* m, int64_t* m_off, double* normX) {
  double acc = 0;
  int64_t nnz = P->row_ptr[P->patient_row_ptr[P->K]];
  for (int64_t e = 0; e < nnz; ++e) acc += P->val[e] * P->val[e];
  *normX = acc;
  m_off[0] = 0;
  for (int64_t k = 0; k < P->K; ++k) {
    int64_t r0 = P->patient_row_ptr[k], r1 = P->patient_row_ptr[k + 1];
    if (o->smooth_l > 0) {
      if (!P->times) return OR_E_ARG;
      m[k] = oracle_patient_basis(P->times + r0, r1 - r0, o->smooth_l, o->smooth_d, o->tau_basis, C + r0 * o->smooth_l);
    } else {
      m[k] = (int32_t)(r1 - r0);
    }
    m_off[k + 1] = m_off[k] + m[k];
  }
  return OR_OK;
}

/* Y_k = Q_k^T X'_k (Alg.1 l.6): R x nc */
static void patient_Y(int32_t R, int32_t m, int64_t nc, const double* Qk, const double* Xp, double* Y) {
  for (int i = 0; i < R; ++i)
    for (int64_t jl = 0; jl < nc; ++jl) {
      double acc = 0;
      for (int a = 0; a < m; ++a) acc += Qk[a * R + i] * Xp[a * nc + jl];
      Y[i * nc + jl] = acc;
    }
}

static void gram(int64_t n, int32_t R, const double* Z, double* G) { /* G = Z^T Z */
  for (int a = 0; a < R; ++a)
    for (int b = 0; b < R; ++b) {
      double acc = 0;
      for (int64_t i = 0; i < n; ++i) acc += Z[i * R + a] * Z[i * R + b];
      G[a * R + b] = acc;
    }
}

/* l.3-l.8 for all patients: Q_k (stacked in Qt at m_off[k]) and rank r_k, from the
 * current H, V, W (the auxiliary/working factors, reading R-aux). */
int oracle_procrustes_all(const or_problem* P, const or_options* o, const double* C, const int32_t* m,
                          const int64_t* m_off, const double* H, const double* V, const double* W, double* Qt,
                          int32_t* rank) {
  const int32_t R = P->R;
  const int32_t l = o->smooth_l;
  int32_t* mark = (int32_t*)malloc(sizeof(int32_t) * (size_t)P->J);
  int32_t* cols = (int32_t*)malloc(sizeof(int32_t) * (size_t)P->J);
  for (int64_t j = 0; j < P->J; ++j) mark[j] = -1;
  double* Pp = NULL; double* A = NULL;
  for (int64_t k = 0; k < P->K; ++k) {
    int64_t r0 = P->patient_row_ptr[k];
    const double* Ck = l > 0 ? C + r0 * l : NULL;
    int32_t mk = m[k];
    double* Xp;
    int64_t nc = patient_dense(P, k, Ck, l, mk, mark, cols, &Xp);
    Pp = (double*)realloc(Pp, sizeof(double) * (size_t)(mk * R + 1));
    A = (double*)realloc(A, sizeof(double) * (size_t)(mk * R + 1));
    for (int a = 0; a < mk; ++a)          /* X'_k V */
      for (int r = 0; r < R; ++r) {
        double acc = 0;
        for (int64_t jl = 0; jl < nc; ++jl) acc += Xp[a * nc + jl] * V[(int64_t)cols[jl] * R + r];
        Pp[a * R + r] = acc;
      }
    for (int a = 0; a < mk; ++a)          /* A_k = X'_k V S_k H^T  (l.4) */
      for (int s = 0; s < R; ++s) {
        double acc = 0;
        for (int r = 0; r < R; ++r) acc += Pp[a * R + r] * W[k * R + r] * H[s * R + r];
        A[a * R + s] = acc;
      }
    rank[k] = oracle_polar(mk, R, A, o->tau_polar, Qt + m_off[k] * R); /* l.4-5 */
    free(Xp);
  }
  free(mark); free(cols); free(Pp); free(A);
  return OR_OK;
}

/* l.12: F = Y_(n) (KR of the other factors), Y_k = Q_k^T X'_k materialised per patient (l.6).
 * mode 1 -> F_H (R x R) = Y_(1)(W ⊙ V); mode 2 -> F_V (J x R) = Y_(2)(W ⊙ H);
 * mode 3 -> F_W (K x R) = Y_(3)(V ⊙ H)   (Kolda-Bader unfoldings). F is zeroed first. */
int oracle_mttkrp(const or_problem* P, const or_options* o, const double* C, const int32_t* m, const int64_t* m_off,
                  const double* Qt, const double* H, const double* V, const double* W, int32_t mode, double* F) {
  const int32_t R = P->R;
  const int32_t l = o->smooth_l;
  int64_t nF = mode == 1 ? (int64_t)R * R : mode == 2 ? P->J * R : P->K * R;
  memset(F, 0, sizeof(double) * (size_t)nF);
  int32_t* mark = (int32_t*)malloc(sizeof(int32_t) * (size_t)P->J);
  int32_t* cols = (int32_t*)malloc(sizeof(int32_t) * (size_t)P->J);
  for (int64_t j = 0; j < P->J; ++j) mark[j] = -1;
  double* Y = NULL;
  for (int64_t k = 0; k < P->K; ++k) {
    int64_t r0 = P->patient_row_ptr[k];
    const double* Ck = l > 0 ? C + r0 * l : NULL;
    double* Xp;
    int64_t nc = patient_dense(P, k, Ck, l, m[k], mark, cols, &Xp);
    Y = (double*)realloc(Y, sizeof(double) * (size_t)(R * nc + 1));
    patient_Y(R, m[k], nc, Qt + m_off[k] * R, Xp, Y);
    for (int64_t jl = 0; jl < nc; ++jl) {
      int64_t j = cols[jl];
      for (int i = 0; i < R; ++i) {
        double y = Y[i * nc + jl]; /* the entry Y(i, j, k) */
        for (int r = 0; r < R; ++r) {
          if (mode == 1) F[i * R + r] += y * (W[k * R + r] * V[j * R + r]);       /* KR row j + J k */
          else if (mode == 2) F[j * R + r] += y * (W[k * R + r] * H[i * R + r]);  /* KR row i + R k */
          else F[k * R + r] += y * (V[j * R + r] * H[i * R + r]);                 /* KR row i + R j */
        }
      }
    }
    free(Xp);
  }
  free(mark); free(cols); free(Y);
  return OR_OK;
}

/* FIT: E = sum_k ||X_k - U_k S_k V^T||^2 with U_k = C_k Q_k H (reading R-fit),
 * expanded per patient as ||X_k||^2 - 2<X_k, U_k S_k V^T> + ||U_k S_k V^T||^2. Returns E. */
double oracle_residual(const or_problem* P, const or_options* o, const double* C, const int32_t* m,
                       const int64_t* m_off, const double* Qt, const double* H, const double* V, const double* W) {
  const int32_t R = P->R;
  const int32_t l = o->smooth_l;
  double* VtV = (double*)malloc(sizeof(double) * (size_t)R * R);
  gram(P->J, R, V, VtV);
  double* U = NULL;
  double* UtU = (double*)malloc(sizeof(double) * (size_t)R * R);
  double E = 0;
  for (int64_t k = 0; k < P->K; ++k) {
    int64_t r0 = P->patient_row_ptr[k], r1 = P->patient_row_ptr[k + 1], Ik = r1 - r0;
    const double* Qk = Qt + m_off[k] * R;
    U = (double*)realloc(U, sizeof(double) * (size_t)(Ik * R + 1));
    for (int64_t i = 0; i < Ik; ++i)
      for (int r = 0; r < R; ++r) {
        double acc = 0;
        if (l > 0) {
          for (int a = 0; a < m[k]; ++a) {
            double cq = 0;
            for (int s = 0; s < R; ++s) cq += Qk[a * R + s] * H[s * R + r];
            acc += C[(r0 + i) * l + a] * cq;
          }
        } else {
          for (int s = 0; s < R; ++s) acc += Qk[i * R + s] * H[s * R + r];
        }
        U[i * R + r] = acc;
      }
    double xx = 0, cross = 0;
    for (int64_t i = 0; i < Ik; ++i)
      for (int64_t e = P->row_ptr[r0 + i]; e < P->row_ptr[r0 + i + 1]; ++e) {
        double x = P->val[e], mv = 0;
        for (int r = 0; r < R; ++r) mv += U[i * R + r] * W[k * R + r] * V[(int64_t)P->col[e] * R + r];
        xx += x * x;
        cross += x * mv;
      }
    gram(Ik, R, U, UtU);
    double quad = 0;
    for (int r = 0; r < R; ++r)
      for (int s = 0; s < R; ++s) quad += UtU[r * R + s] * W[k * R + r] * W[k * R + s] * VtV[r * R + s];
    E += xx - 2.0 * cross + quad;
  }
  free(U); free(UtU); free(VtV);
  return E;
}

/* One outer iteration of Alg.1 (l.3-l.20) + FIT. Factors are the auxiliary (working)
 * variables H, V, W (reading R-aux); D* are the scaled duals; mode order H, W, V with
 * fresh factors (reading R-order). diag (may be NULL, else 8 doubles) receives rho_H, rho_W, rho_V, E,
 * normX and the inner ADMM steps of the H, W, V modes summed over rows. */
int oracle_iterate(const or_problem* P, const or_options* o, const double* C, const int32_t* m, const int64_t* m_off,
                   double normX, double* H, double* V, double* W, double* DH, double* DV, double* DW, double* Qt,
                   int32_t* rank, double* fit_out, double* diag) {
  const int32_t R = P->R;
  const int64_t K = P->K, J = P->J;
  double* F = (double*)malloc(sizeof(double) * (size_t)((K > J ? K : J) * R + R * R));
  double* G = (double*)malloc(sizeof(double) * (size_t)R * R);
  double* G1 = (double*)malloc(sizeof(double) * (size_t)R * R);
  double* G2 = (double*)malloc(sizeof(double) * (size_t)R * R);
  double rho_used[3] = {0, 0, 0};
  double E = 0;
  int32_t* steps_H = (int32_t*)calloc((size_t)R, sizeof(int32_t));
  int32_t* steps_W = (int32_t*)calloc((size_t)(K > 0 ? K : 1), sizeof(int32_t));
  int32_t* steps_V = (int32_t*)calloc((size_t)J, sizeof(int32_t));
  int status = oracle_procrustes_all(P, o, C, m, m_off, H, V, W, Qt, rank);
  /* n = 1 (H): G = (V^T V) * (W^T W) (l.11), F_H (l.12), ADMM (l.13-19) */
  if (status == OR_OK) {
    oracle_mttkrp(P, o, C, m, m_off, Qt, H, V, W, 1, F);
    gram(J, R, V, G1); gram(K, R, W, G2);
    for (int i = 0; i < R * R; ++i) G[i] = G1[i] * G2[i];
    status = oracle_admm_mode_tol(R, R, F, G, o->rho, o->n_inner, o->kind_H, o->param_H, o->admm_tol, H, DH,
                                  &rho_used[0], steps_H);
  }
  /* n = 2 (W): with the updated H; G = (H^T H) * (V^T V) */
  if (status == OR_OK) {
    oracle_mttkrp(P, o, C, m, m_off, Qt, H, V, W, 3, F);
    gram(R, R, H, G1); gram(J, R, V, G2);
    for (int i = 0; i < R * R; ++i) G[i] = G1[i] * G2[i];
    status = oracle_admm_mode_tol(K, R, F, G, o->rho, o->n_inner, o->kind_W, o->param_W, o->admm_tol, W, DW,
                                  &rho_used[1], steps_W);
  }
  /* n = 3 (V): with the updated H and W; G = (H^T H) * (W^T W) */
  if (status == OR_OK) {
    oracle_mttkrp(P, o, C, m, m_off, Qt, H, V, W, 2, F);
    gram(R, R, H, G1); gram(K, R, W, G2);
    for (int i = 0; i < R * R; ++i) G[i] = G1[i] * G2[i];
    status = oracle_admm_mode_tol(J, R, F, G, o->rho, o->n_inner, o->kind_V, o->param_V, o->admm_tol, V, DV,
                                  &rho_used[2], steps_V);
  }
  if (status == OR_OK) {
    E = oracle_residual(P, o, C, m, m_off, Qt, H, V, W);
    *fit_out = 1.0 - E / normX;
    if (!isfinite(*fit_out)) status = OR_E_NONFINITE;
  }
  if (diag) {
    int64_t tH = 0, tW = 0, tV = 0;
    for (int i = 0; i < R; ++i) tH += steps_H[i];
    for (int64_t i = 0; i < K; ++i) tW += steps_W[i];
    for (int64_t i = 0; i < J; ++i) tV += steps_V[i];
    diag[0] = rho_used[0]; diag[1] = rho_used[1]; diag[2] = rho_used[2]; diag[3] = E; diag[4] = normX;
    diag[5] = (double)tH; diag[6] = (double)tW; diag[7] = (double)tV; /* inner steps summed over rows */
  }
  free(steps_H); free(steps_W); free(steps_V);
  free(F); free(G); free(G1); free(G2);
  return status;
}
