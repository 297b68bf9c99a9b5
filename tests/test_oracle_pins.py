"""Pins for the oracle: the oracle checked against things OTHER than
itself — closed forms printed in the paper/SPEC, textbook special cases, an independent
library (numpy/scipy LAPACK, scipy BSpline), dense brute force on tiny inputs, invariants.

Each test cites the passage it pins. A plausible slip (dropped term, wrong sign or index,
transposed operand) in the oracle fails at least one of them.
"""
import dataclasses

import numpy as np
import pytest

import oracle
import synthgen
from tests.helpers import dense_slices, make_problem, planted

NONE, NONNEG, L1, NONNEG_L1, L0 = 0, 1, 2, 3, 4


# ------------------------------------------------------------------- P1 prox
def test_p1_prox_closed_forms():
    # S:267-269 worked examples (nonneg clamp; l0 with mu = 0.25 keeps equality; l1 lambda=0.4 rho=2)
    assert np.array_equal(oracle.prox(NONNEG, 0, 1, [-1, 0, 2.5]), [0, 0, 2.5])
    assert np.array_equal(oracle.prox(L0, 0.25, 1, [0.4, 0.5, -0.6, 0.1]), [0, 0.5, -0.6, 0])
    assert np.allclose(oracle.prox(L1, 0.4, 2, [0.5, -0.1, -0.9]), [0.3, 0, -0.7], atol=1e-15)
    assert np.allclose(oracle.prox(NONNEG_L1, 0.4, 2, [0.5, 0.1, -0.9]), [0.3, 0, 0], atol=1e-15)
    assert np.array_equal(oracle.prox(NONE, 0, 1, [-3.0, 7.0]), [-3.0, 7.0])


@pytest.mark.parametrize("kind,param", [(NONNEG, 0.0), (L1, 0.7), (NONNEG_L1, 0.7), (L0, 0.3)])
def test_p1_prox_is_argmin_on_grid(kind, param):
    """prox(x) = argmin_z c(z) + rho/2 (z-x)^2 by brute-force grid minimisation."""
    rho = 1.7
    rng = np.random.default_rng(1)
    xs = rng.uniform(-3, 3, size=60)
    grid = np.linspace(-5, 5, 1_000_001)
    pen = {NONNEG: np.where(grid >= 0, 0.0, np.inf), L1: param * np.abs(grid),
           NONNEG_L1: np.where(grid >= 0, param * grid, np.inf),
           L0: (param * rho / 2.0) * (grid != 0)}[kind]  # l0 with mu = 2 lambda/rho -> lambda = mu rho/2
    for x in xs:
        obj = pen + rho / 2 * (grid - x) ** 2
        zstar = grid[np.argmin(obj)]
        z = oracle.prox(kind, param, rho, [x])[0]
        if kind == L0 and abs(x * x - param) < 1e-3:
            continue  # tie region at the threshold
        assert abs(z - zstar) <= 2e-5, (kind, x, z, zstar)


# ------------------------------------------------------------------- P2 / P17 SVD & polar
def test_p2_polar_special_cases():
    Q, r = oracle.polar(np.diag([5.0, 0.1]))
    assert r == 2 and np.allclose(Q, np.eye(2), atol=1e-14)
    rng = np.random.default_rng(2)
    Q0, _ = np.linalg.qr(rng.standard_normal((8, 3)))
    Q, r = oracle.polar(Q0)
    assert np.allclose(Q, Q0, atol=1e-13)  # orthonormal A is a fixed point
    M = rng.standard_normal((3, 3)); P = M @ M.T + 3 * np.eye(3)  # polar(Q P) = Q for SPD P
    Q, r = oracle.polar(Q0 @ P)
    assert np.allclose(Q, Q0, atol=1e-12)


def test_p2_polar_maximises_trace():
    """Procrustes optimality: tr(A^T Q) >= tr(A^T Z) for orthonormal-column Z."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        A = rng.standard_normal((8, 3))
        Q, _ = oracle.polar(A)
        best = np.trace(A.T @ Q)
        for _ in range(40):
            Z, _ = np.linalg.qr(rng.standard_normal((8, 3)))
            assert best >= np.trace(A.T @ Z) - 1e-12
        assert np.allclose(Q.T @ Q, np.eye(3), atol=1e-13)


@pytest.mark.parametrize("shape", [(9, 4), (4, 9), (7, 7), (30, 5), (3, 40)])
def test_p17_svd_matches_lapack(shape):
    rng = np.random.default_rng(4)
    for cond in (1.0, 1e4, 1e9):
        A = rng.standard_normal(shape)
        U0, s0, Vt0 = np.linalg.svd(A, full_matrices=False)
        s0 = s0[0] * np.logspace(0, -np.log10(cond), len(s0))
        A = (U0 * s0) @ Vt0
        U, s, V = oracle.svd(A)
        ref = np.linalg.svd(A, compute_uv=False)
        assert np.allclose(s, ref, rtol=0, atol=1e-14 * ref[0] * max(shape))
        assert np.allclose((U * s) @ V.T, A, atol=1e-13 * ref[0])
        Q, r = oracle.polar(A)
        Uq, sq, Vqt = np.linalg.svd(A, full_matrices=False)
        Qref = Uq @ Vqt  # full rank here
        assert r == len(sq)
        assert np.linalg.norm(Q - Qref) <= 1e-15 * cond * 50 + 1e-13


def test_p2_partial_isometry_rank_deficient():
    """Reading R-polar-2: Q = U_r V_r^T on the numerical range when rank(A) < min(m, n)."""
    rng = np.random.default_rng(5)
    A = rng.standard_normal((6, 2)) @ rng.standard_normal((2, 5))  # rank 2
    Q, r = oracle.polar(A)
    assert r == 2
    U, s, Vt = np.linalg.svd(A)
    assert np.allclose(Q, U[:, :2] @ Vt[:2], atol=1e-12)
    Q, r = oracle.polar(np.zeros((4, 3)))
    assert r == 0 and not Q.any()


# ------------------------------------------------------------------- P3 SPD solve (l.14, l.16)
def test_p3_cholesky_solve():
    L = oracle.cholesky(np.zeros((2, 2)) + 2 * np.eye(2))
    assert np.allclose(oracle.chol_solve(L, np.array([4.0, 6.0])), [2.0, 3.0], atol=1e-15)
    L = oracle.cholesky(np.eye(3) * 2.0)
    assert np.allclose(oracle.chol_solve(L, np.array([1.0, 0, 0])), [0.5, 0, 0])
    rng = np.random.default_rng(6)
    for R in (3, 10, 40):
        M = rng.standard_normal((R + 5, R)); G = M.T @ M + 0.5 * np.eye(R)
        L = oracle.cholesky(G)
        assert np.allclose(L, np.linalg.cholesky(G), atol=1e-12)
        b = rng.standard_normal(R)
        assert np.allclose(oracle.chol_solve(L, b), np.linalg.solve(G, b), rtol=1e-10, atol=1e-12)
    with pytest.raises(np.linalg.LinAlgError):
        oracle.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))


# ------------------------------------------------------------------- P10 / P11 / P16 ADMM
def test_p10_identity_prox_closed_form():
    """D stays 0 with the identity prox, and Zbar_n = F G^-1 + (Zbar_0 - F G^-1)(rho (G+rho I)^-1)^n."""
    rng = np.random.default_rng(7)
    R, n = 6, 9
    M = rng.standard_normal((20, R)); G = M.T @ M
    F = rng.standard_normal((n, R)); Z0 = rng.standard_normal((n, R))
    rho = np.trace(G) / R
    Ginv = np.linalg.inv(G)
    T = rho * np.linalg.inv(G + rho * np.eye(R))
    for steps in (1, 2, 5):
        Zb, D, rho_used = oracle.admm_mode(F, G, Z0, np.zeros((n, R)), NONE, 0.0, rho=0.0, n_inner=steps)
        assert abs(rho_used - rho) <= 1e-14 * rho
        ref = F @ Ginv + (Z0 - F @ Ginv) @ np.linalg.matrix_power(T, steps)
        assert np.allclose(Zb, ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())
        assert np.abs(D).max() < 1e-12 * np.abs(ref).max()


def test_p11_admm_limits():
    rng = np.random.default_rng(8)
    R, n = 4, 7
    M = rng.standard_normal((12, R)); G = M.T @ M
    F = rng.standard_normal((n, R))
    Zb, D, _ = oracle.admm_mode(F, G, np.zeros((n, R)), np.zeros((n, R)), NONE, 0.0, rho=0.0, n_inner=400)
    assert np.linalg.norm(Zb @ G - F) / np.linalg.norm(F) <= 1e-10  # normal equations (a CP-ALS step)
    # inactive non-negativity: F = X G with X > 0 -> same as unconstrained
    X = rng.uniform(1, 2, size=(n, R)); F2 = X @ G
    Za, _, _ = oracle.admm_mode(F2, G, np.ones((n, R)), np.zeros((n, R)), NONNEG, 0.0, rho=0.0, n_inner=300)
    Zu, _, _ = oracle.admm_mode(F2, G, np.ones((n, R)), np.zeros((n, R)), NONE, 0.0, rho=0.0, n_inner=300)
    assert np.allclose(Za, Zu, atol=1e-8) and np.allclose(Za, X, atol=1e-6)
    Z0, _, _ = oracle.admm_mode(F, G, np.ones((n, R)), np.zeros((n, R)), L0, 1e12, rho=0.0, n_inner=3)
    assert not Z0.any()


def test_p16_cached_factorisation_consistent():
    """caching F and chol(G+rho I) across inner steps = recomputing them each step."""
    rng = np.random.default_rng(9)
    R, n = 5, 11
    M = rng.standard_normal((15, R)); G = M.T @ M
    F = rng.standard_normal((n, R)); Z = rng.uniform(size=(n, R)); D = np.zeros((n, R))
    Zc, Dc, _ = oracle.admm_mode(F, G, Z, D, L1, 0.3, rho=0.0, n_inner=5)
    Zs, Ds = Z, D
    for _ in range(5):
        Zs, Ds, _ = oracle.admm_mode(F.copy(), G.copy(), Zs, Ds, L1, 0.3, rho=0.0, n_inner=1)
    assert np.array_equal(Zc, Zs) and np.array_equal(Dc, Ds)


# ------------------------------------------------------------------- P14 B-spline
def test_p14_bspline_special_cases():
    # d = 0: indicator of [beta_b, beta_b+1), last interval closed at t_n
    t = np.array([0.0, 0.5, 1.0, 1.5, 2.0])
    M0 = oracle.bspline_matrix(t, 2, d=0)
    assert np.array_equal(M0, [[1, 0], [1, 0], [0, 1], [0, 1], [0, 1]])
    # d = 1 on knots (0,0,1,2,2) (l=3): middle basis is the hat with m(0.5)=0.5, m(1)=1, m(1.5)=0.5
    M1 = oracle.bspline_matrix(t, 3, d=1)
    assert np.allclose(M1[:, 1], [0, 0.5, 1, 0.5, 0])
    assert oracle.knots(0.0, 2.0, 3, 1).tolist() == [0, 0, 1, 2, 2]


def test_p14_bspline_matches_scipy_and_properties():
    from scipy.interpolate import BSpline
    rng = np.random.default_rng(10)
    for l in (5, 7, 9):
        t = np.sort(rng.uniform(0, 300, size=40))
        M = oracle.bspline_matrix(t, l)
        beta = oracle.knots(t[0], t[-1], l)
        for b in range(l):
            ref = BSpline.basis_element(beta[b:b + 5], extrapolate=False)(t)
            ref = np.nan_to_num(ref)
            if b == l - 1:
                ref[-1] = 1.0  # right end closed (reading R-spline-2); scipy's element is 0 there
            assert np.allclose(M[:, b], ref, atol=1e-13), b
        assert np.allclose(M.sum(axis=1), 1.0, atol=1e-14)  # partition of unity (clamped knots)
        assert M.min() >= 0
        # local support: m_b = 0 outside [beta_b, beta_{b+d+1}]
        for b in range(l):
            out = (t < beta[b]) | (t > beta[b + 4])
            assert not M[out, b].any()


def test_basis_spans_range_of_M():
    rng = np.random.default_rng(11)
    t = np.sort(rng.uniform(0, 500, size=25))
    C, lp = oracle.patient_basis(t, 7)
    M = oracle.bspline_matrix(t, 7)
    assert lp == np.linalg.matrix_rank(M)
    Cr = C[:, :lp]
    assert np.allclose(Cr.T @ Cr, np.eye(lp), atol=1e-13)
    assert np.linalg.norm(M - Cr @ (Cr.T @ M)) <= 1e-12 * np.linalg.norm(M)
    # I_k < l: basis of the whole row space
    C2, lp2 = oracle.patient_basis(t[:4], 7)
    assert lp2 == 4


# ------------------------------------------------------------------- P5 MTTKRP vs materialised Y (l.12)
def _naive_kr(A, B):
    return np.einsum("ar,br->abr", A, B).reshape(-1, A.shape[1])


@pytest.mark.parametrize("name", ["tiny", "medium"])
def test_p5_mttkrp_equals_materialised_unfolding(name):
    p = synthgen.generate(name, K=12)
    o = oracle.Oracle(p)
    o.procrustes()
    R, J, K = o.R, p.J, p.K
    Y = np.zeros((R, J, K))
    Xs = dense_slices(p)
    for k in range(K):
        Xp = Xs[k] if o.C is None else o.C[p.patient_row_ptr[k]:p.patient_row_ptr[k + 1], :o.m[k]].T @ Xs[k]
        Y[:, :, k] = o.Qk(k).T @ Xp  # Y_k = Q_k^T X'_k (l.6)
    H, V, W = o.H, o.V, o.W
    Y1 = Y.reshape(R, J * K, order="F")
    Y2 = np.moveaxis(Y, 1, 0).reshape(J, R * K, order="F")
    Y3 = np.moveaxis(Y, 2, 0).reshape(K, R * J, order="F")
    for mode, ref in [(1, Y1 @ _naive_kr(W, V)), (2, Y2 @ _naive_kr(W, H)), (3, Y3 @ _naive_kr(V, H))]:
        F = o.mttkrp(mode)
        assert np.linalg.norm(F - ref) <= 1e-12 * np.linalg.norm(ref), mode


def test_p4_naive_kr_index_formula():
    A = np.eye(2); B = np.eye(2)
    assert np.array_equal(_naive_kr(A, B), [[1, 0], [0, 0], [0, 0], [0, 1]])


# ------------------------------------------------------------------- P6 / P8 FIT
@pytest.mark.parametrize("name", ["tiny", "medium"])
def test_p6_fit_equals_dense_brute_force(name):
    p = synthgen.generate(name, K=15)
    o = oracle.Oracle(p)
    fits = o.iterate(2)
    Xs = dense_slices(p)
    E = sum(np.linalg.norm(Xs[k] - o.U(k) @ np.diag(o.W[k]) @ o.V.T) ** 2 for k in range(p.K))
    normX = sum(np.linalg.norm(X) ** 2 for X in Xs)
    assert abs(o.normX - normX) <= 1e-13 * normX
    assert abs(fits[-1] - (1 - E / normX)) <= 1e-12


def test_p6_y_form_of_objective_when_q_orthonormal():
    """P:193-194 / P:148: with Q^T Q = I, sum||X - Q H S V^T||^2 = sum||Y - H S V^T||^2 + sum(||X||^2 - ||Y||^2)."""
    mats, Qs, H, V, W = planted(6, 8, 12, 10, 3, seed=1)
    rng = np.random.default_rng(0)
    mats = [X + 0.1 * rng.standard_normal(X.shape) for X in mats]
    lhs = rhs = 0.0
    for k, X in enumerate(mats):
        Q, _ = np.linalg.qr(rng.standard_normal((X.shape[0], 3)))
        Y = Q.T @ X
        M = H @ np.diag(W[k]) @ V.T
        lhs += np.linalg.norm(X - Q @ M) ** 2
        rhs += np.linalg.norm(Y - M) ** 2 + np.linalg.norm(X) ** 2 - np.linalg.norm(Y) ** 2
    assert abs(lhs - rhs) <= 1e-12 * lhs


def test_p8_smooth_residual_identity():
    p = synthgen.generate("medium", K=20)
    o = oracle.Oracle(p)
    o.iterate(1)
    Xs = dense_slices(p)
    for k in range(p.K):
        r0, r1 = p.patient_row_ptr[k], p.patient_row_ptr[k + 1]
        C = o.C[r0:r1, :o.m[k]]
        M = o.Qk(k) @ o.H @ np.diag(o.W[k]) @ o.V.T
        Xp = C.T @ Xs[k]
        lhs = np.linalg.norm(Xs[k] - C @ M) ** 2
        rhs = np.linalg.norm(Xp - M) ** 2 + np.linalg.norm(Xs[k]) ** 2 - np.linalg.norm(Xp) ** 2
        assert abs(lhs - rhs) <= 1e-11 * max(lhs, 1.0)


# ------------------------------------------------------------------- P7 PARAFAC2 invariants
def test_p7_parafac2_invariants():
    p = synthgen.generate("small", K=300)
    o = oracle.Oracle(p)
    o.iterate(2)
    HtH = o.H.T @ o.H
    n = 0
    for k in range(p.K):
        if o.rank[k] == o.R:
            Q = o.Qk(k)
            assert np.linalg.norm(Q.T @ Q - np.eye(o.R)) <= 1e-12
            U = o.U(k)
            assert np.linalg.norm(U.T @ U - HtH) <= 1e-12 * np.linalg.norm(HtH)
            n += 1
        else:  # partial isometry on the numerical range
            Q = o.Qk(k)
            P = Q.T @ Q
            assert np.linalg.norm(P @ P - P) <= 1e-12
    assert n > 100


# ------------------------------------------------------------------- P9 basis freedom (reading R-spline-5)
def test_p9_basis_rotation_invariance():
    p = synthgen.generate("medium", K=40)
    a = oracle.Oracle(p)
    b = oracle.Oracle(p)
    rng = np.random.default_rng(12)
    for k in range(p.K):
        r0, r1 = p.patient_row_ptr[k], p.patient_row_ptr[k + 1]
        mk = b.m[k]
        O, _ = np.linalg.qr(rng.standard_normal((mk, mk)))
        b.C[r0:r1, :mk] = b.C[r0:r1, :mk] @ O
    fa = a.iterate(2); fb = b.iterate(2)
    assert abs(fa[-1] - fb[-1]) <= 1e-12
    for x, y in [(a.H, b.H), (a.V, b.V), (a.W, b.W)]:
        assert np.linalg.norm(x - y) <= 1e-11 * np.linalg.norm(x)
    Ua, Ub = a.U_all(), b.U_all()
    assert np.linalg.norm(Ua - Ub) <= 1e-11 * np.linalg.norm(Ua)


# ------------------------------------------------------------------- P12 / P13 recovery
def test_p12_procrustes_recovers_planted_q():
    mats, Qs, H, V, W = planted(20, 10, 20, 30, 4, seed=3)
    p = make_problem(mats, 4, H0=H, V0=V, W0=W)
    o = oracle.Oracle(p)
    o.procrustes()
    for k in range(p.K):
        assert np.linalg.norm(o.Qk(k) - Qs[k]) <= 1e-10


@pytest.mark.slow
def test_p12_planted_recovery_fit():
    """Noise-free planted PARAFAC2 (K=50, I_k in [10,20], J=40, R=5): FIT >= 0.999 for >= 4 of 5 seeds."""
    ok = 0
    for seed in range(5):
        mats, _, _, _, _ = planted(50, 10, 20, 40, 5, seed=100 + seed)
        p = make_problem(mats, 5, seed=seed, con_W=(NONNEG, 0.0), con_V=(NONNEG, 0.0), rho=0.0)
        o = oracle.Oracle(p)
        fit = -1
        for _ in range(500):
            fit = o.iterate(1)[-1]
            if fit >= 0.999:
                break
        ok += fit >= 0.999
    assert ok >= 4


def test_p13_rank_one_exact():
    rng = np.random.default_rng(13)
    v = rng.uniform(0.5, 1, size=15)
    mats = [np.outer(rng.uniform(0.5, 1, size=int(rng.integers(3, 8))), v) for _ in range(10)]
    p = make_problem(mats, 1, con_W=(NONNEG, 0.0), con_V=(NONNEG, 0.0), rho=0.0)
    o = oracle.Oracle(p)
    fits = o.iterate(60)
    assert fits[-1] >= 1 - 1e-6
    Vn = o.V[:, 0] / np.linalg.norm(o.V[:, 0])
    assert np.allclose(np.abs(Vn), v / np.linalg.norm(v), atol=1e-6)


# ------------------------------------------------------------------- P15 / P18
def test_p15_fit_quasi_monotone_unconstrained():
    p = synthgen.generate("small", K=200)
    p = dataclasses.replace(p, cfg=dataclasses.replace(p.cfg, con_W=(NONE, 0.0), con_V=(NONE, 0.0)))
    o = oracle.Oracle(p, opts=oracle.options_from_config(p.cfg, n_inner=60))
    fits = o.iterate(12)
    assert all(b >= a - 1e-6 for a, b in zip(fits, fits[1:]))


def test_p18_deterministic():
    p = synthgen.generate("medium", K=50)
    a = oracle.Oracle(p); b = oracle.Oracle(p)
    fa = a.iterate(2); fb = b.iterate(2)
    assert fa == fb and np.array_equal(a.V, b.V) and np.array_equal(a.Q, b.Q)


# ------------------------------------------------------------------- P19 mode order and freshness (Alg.1 l.9-l.20)
def _y_tensor(o, p):
    """Y(:, :, k) = Q_k^T X'_k (Alg.1 l.6) from dense slices and the oracle's stored Q."""
    Xs = dense_slices(p)
    Y = np.zeros((o.R, p.J, p.K))
    for k in range(p.K):
        Xp = Xs[k] if o.C is None else o.C[p.patient_row_ptr[k]:p.patient_row_ptr[k + 1], :o.m[k]].T @ Xs[k]
        Y[:, :, k] = o.Qk(k).T @ Xp
    return Y


@pytest.mark.parametrize("name", ["tiny", "medium"])
def test_p19_mode_order_and_freshness(name):
    """Alg.1 l.9-l.20 (reading R-order): modes are updated H -> W -> V, the W
    update uses the NEW H, the V update the new H and W (Gauss-Seidel, not Jacobi block order).

    With no constraint and many inner steps the ADMM of each mode converges to the normal-equation
    solution F G^-1 (pin P11), so after one outer iteration, from numpy (dense Y, naive Khatri-Rao):
      H1 = Y_(1)(W0 ⊙ V0) [(V0^T V0) * (W0^T W0)]^-1
      W1 = Y_(3)(V0 ⊙ H1) [(H1^T H1) * (V0^T V0)]^-1
      V1 = Y_(2)(W1 ⊙ H1) [(H1^T H1) * (W1^T W1)]^-1
    A stale factor in any mode (e.g. V from the old W) changes the result at O(1)."""
    cfg = dataclasses.replace(synthgen.CONFIGS[name], con_H=(NONE, 0.0), con_W=(NONE, 0.0), con_V=(NONE, 0.0))
    p = synthgen.generate(cfg, K=30)
    o = oracle.Oracle(p, opts=oracle.options_from_config(cfg, n_inner=3000))
    H0, V0, W0 = o.H.copy(), o.V.copy(), o.W.copy()
    o.iterate(1)
    Y = _y_tensor(o, p)  # Q from the Procrustes step on (H0, V0, W0)
    R, J, K = o.R, p.J, p.K
    Y1 = Y.reshape(R, J * K, order="F")
    Y2 = np.moveaxis(Y, 1, 0).reshape(J, R * K, order="F")
    Y3 = np.moveaxis(Y, 2, 0).reshape(K, R * J, order="F")
    H1 = np.linalg.solve(((V0.T @ V0) * (W0.T @ W0)).T, (Y1 @ _naive_kr(W0, V0)).T).T
    W1 = np.linalg.solve(((H1.T @ H1) * (V0.T @ V0)).T, (Y3 @ _naive_kr(V0, H1)).T).T
    V1 = np.linalg.solve(((H1.T @ H1) * (W1.T @ W1)).T, (Y2 @ _naive_kr(W1, H1)).T).T
    for got, ref, what in ((o.H, H1, "H"), (o.W, W1, "W"), (o.V, V1, "V")):
        err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        assert err <= 1e-8, (what, err)
    # the stale (Jacobi-order) alternatives are far away: the pin can tell them apart
    W_stale = np.linalg.solve(((H0.T @ H0) * (V0.T @ V0)).T, (Y3 @ _naive_kr(V0, H0)).T).T
    V_stale = np.linalg.solve(((H1.T @ H1) * (W0.T @ W0)).T, (Y2 @ _naive_kr(W0, H1)).T).T
    assert np.linalg.norm(W_stale - W1) > 1e-3 * np.linalg.norm(W1)
    assert np.linalg.norm(V_stale - V1) > 1e-3 * np.linalg.norm(V1)


# ------------------------------------------------------------------- golden fixtures (tests/golden/, each cited)
def _golden(name):
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", name)
    rows = []
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        rows.append([part.split() for part in line.split("|")])
    return rows


def test_golden_prox_examples():
    kinds = {"none": NONE, "nonneg": NONNEG, "l1": L1, "nonneg_l1": NONNEG_L1, "l0": L0}
    for (kind, param, rho), xs, ys in _golden("prox_examples.txt"):
        got = oracle.prox(kinds[kind], float(param), float(rho), [float(x) for x in xs])
        assert np.allclose(got, [float(y) for y in ys], rtol=0, atol=1e-15), (kind, got, ys)


def test_golden_bspline_examples():
    for (l, d), ts, ms in _golden("bspline_examples.txt"):
        l, d = int(l), int(d)
        M = oracle.bspline_matrix([float(t) for t in ts], l, d=d)
        assert np.allclose(M.ravel(), [float(x) for x in ms], rtol=0, atol=1e-15), (l, d, M)


def test_golden_sparsity_examples():
    for (r, c), vals, (want,) in _golden("sparsity_examples.txt"):
        V = np.array([float(v) for v in vals]).reshape(int(r), int(c))
        assert oracle.sparsity(V) == float(want)


# ------------------------------------------------------------------- P20 inner / outer stops (N3)
def test_p20_inner_stop_identity_prox_closed_form():
    """Reading R-inner-tol: with the identity prox D stays 0 and each row follows the closed form of
    P10, Zbar_n = F G^-1 + (Zbar_0 - F G^-1) T^n with T = rho (G + rho I)^-1. The per-row stop after
    step n is ||Zbar_n - Zbar_{n-1}|| <= tol ||Zbar_n||, so the step count of every row and its final
    value follow from the closed form alone."""
    rng = np.random.default_rng(21)
    R, n, tol, cap = 6, 40, 1e-3, 60
    M = rng.standard_normal((20, R)); G = M.T @ M
    F = rng.standard_normal((n, R)) * rng.uniform(0.1, 10, size=(n, 1))
    Z0 = rng.standard_normal((n, R))
    rho = np.trace(G) / R
    X = F @ np.linalg.inv(G)
    T = rho * np.linalg.inv(G + rho * np.eye(R))
    steps = np.zeros(n, np.int32)
    Zb, D, _ = oracle.admm_mode(F, G, Z0, np.zeros((n, R)), NONE, 0.0, rho=0.0, n_inner=cap, tol=tol, steps=steps)
    checked = 0
    for i in range(n):
        prev = Z0[i]
        want = cap
        margin_ok = True
        for s in range(1, cap + 1):
            cur = X[i] + (Z0[i] - X[i]) @ np.linalg.matrix_power(T, s)
            ratio = np.linalg.norm(cur - prev) / np.linalg.norm(cur)
            if abs(ratio - tol) < 1e-6 * tol:
                margin_ok = False  # too close to the threshold for a rounding-independent decision
            if ratio <= tol:
                want = s
                break
            prev = cur
        if not margin_ok:
            continue
        checked += 1
        assert steps[i] == want, (i, steps[i], want)
        ref = X[i] + (Z0[i] - X[i]) @ np.linalg.matrix_power(T, want)
        assert np.allclose(Zb[i], ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())
    assert checked >= n - 2 and len(set(steps.tolist())) > 3  # rows stop at different steps
    assert not D.any()


def test_p20_inner_stop_is_truncation():
    """A row that stops after s steps holds exactly what the fixed-count ADMM (tol = 0, pinned by
    P10/P11) gives after s steps — for every prox kind."""
    rng = np.random.default_rng(22)
    R, n = 5, 25
    M = rng.standard_normal((15, R)); G = M.T @ M
    F = rng.standard_normal((n, R)) * 3
    Z0 = rng.uniform(size=(n, R))
    for kind, param in ((NONNEG, 0.0), (L1, 0.5), (NONNEG_L1, 0.2), (L0, 0.05)):
        steps = np.zeros(n, np.int32)
        Zt, Dt, _ = oracle.admm_mode(F, G, Z0, np.zeros((n, R)), kind, param, rho=0.0, n_inner=50, tol=1e-4,
                                     steps=steps)
        assert steps.min() >= 1 and steps.max() <= 50
        for i in range(n):
            Zf, Df, _ = oracle.admm_mode(F[i:i + 1], G, Z0[i:i + 1], np.zeros((1, R)), kind, param, rho=0.0,
                                         n_inner=int(steps[i]))
            assert np.array_equal(Zf[0], Zt[i]) and np.array_equal(Df[0], Dt[i]), (kind, i)


def test_p20_outer_stop_matches_fixed_trajectory():
    """Reading R-outer-tol: iterate_until stops at the first t >= 2 with
    |FIT_t - FIT_{t-1}| < tol max(|FIT_{t-1}|, 1); the FIT values are those of the fixed-count run."""
    p = synthgen.generate("tiny", K=60)
    a = oracle.Oracle(p); b = oracle.Oracle(p)
    fa = a.iterate(40)
    tol = 1e-3
    fb = b.iterate_until(40, tol)
    stop = next((t for t in range(1, 40) if abs(fa[t] - fa[t - 1]) < tol * max(abs(fa[t - 1]), 1.0)), 39)
    assert len(fb) == stop + 1 and fb == fa[:stop + 1]
    assert len(fb) < 40


def test_p20_sparsity_l0_total_threshold():
    """SPARSITY: l0 with huge mu zeroes V entirely -> 1.0."""
    rng = np.random.default_rng(23)
    R, n = 4, 9
    M = rng.standard_normal((12, R)); G = M.T @ M
    Z, _, _ = oracle.admm_mode(rng.standard_normal((n, R)), G, np.ones((n, R)), np.zeros((n, R)), L0, 1e12,
                               rho=0.0, n_inner=2)
    assert oracle.sparsity(Z) == 1.0
    assert oracle.sparsity(np.ones((3, 2))) == 0.0
