"""ORACLE — test infrastructure only (see copa_oracle.c header).

Plain serial FP64 CPU implementation of COPA's outer iteration (Alg.1)
written from the paper; pinned by tests/test_oracle_pins.py. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline / --impl reference) may import it.
It never imports the CUDA package, and the CUDA package never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

TAU_POLAR = 1e-10   # DESIGN.md reading R-polar-3
TAU_BASIS = 1e-6    # DESIGN.md reading R-spline-4
SPLINE_DEGREE = 3   # DESIGN.md reading R-spline-3


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "copa_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        # -ffp-contract=off: no FMA contraction; plain IEEE double arithmetic in source order.
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


class _Problem(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int64), ("J", ctypes.c_int64), ("R", ctypes.c_int32),
                ("patient_row_ptr", ctypes.c_void_p), ("row_ptr", ctypes.c_void_p), ("col", ctypes.c_void_p),
                ("val", ctypes.c_void_p), ("times", ctypes.c_void_p)]


class _Options(ctypes.Structure):
    _fields_ = [("kind_H", ctypes.c_int32), ("kind_W", ctypes.c_int32), ("kind_V", ctypes.c_int32),
                ("param_H", ctypes.c_double), ("param_W", ctypes.c_double), ("param_V", ctypes.c_double),
                ("smooth_l", ctypes.c_int32), ("smooth_d", ctypes.c_int32), ("rho", ctypes.c_double),
                ("n_inner", ctypes.c_int32), ("tau_polar", ctypes.c_double), ("tau_basis", ctypes.c_double),
                ("admm_tol", ctypes.c_double)]


_lib = None
_vp = ctypes.c_void_p


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        d, i32, i64 = ctypes.c_double, ctypes.c_int32, ctypes.c_int64
        L.oracle_prox.argtypes = [i32, d, d, d]; L.oracle_prox.restype = d
        L.oracle_knots.argtypes = [d, d, i32, i32, _vp]
        L.oracle_bspline_matrix.argtypes = [_vp, i64, i32, i32, _vp]
        L.oracle_svd.argtypes = [i64, i64, _vp, _vp, _vp, _vp]; L.oracle_svd.restype = ctypes.c_int
        L.oracle_polar.argtypes = [i64, i64, _vp, d, _vp]; L.oracle_polar.restype = ctypes.c_int
        L.oracle_cholesky.argtypes = [i32, _vp]; L.oracle_cholesky.restype = ctypes.c_int
        L.oracle_chol_solve.argtypes = [i32, _vp, _vp]
        L.oracle_admm_mode.argtypes = [i64, i32, _vp, _vp, d, i32, i32, d, _vp, _vp, _vp]
        L.oracle_admm_mode.restype = ctypes.c_int
        L.oracle_admm_mode_tol.argtypes = [i64, i32, _vp, _vp, d, i32, i32, d, d, _vp, _vp, _vp, _vp]
        L.oracle_admm_mode_tol.restype = ctypes.c_int
        L.oracle_sparsity.argtypes = [i64, _vp]; L.oracle_sparsity.restype = d
        L.oracle_patient_basis.argtypes = [_vp, i64, i32, i32, d, _vp]; L.oracle_patient_basis.restype = ctypes.c_int
        P, O = ctypes.POINTER(_Problem), ctypes.POINTER(_Options)
        L.oracle_init.argtypes = [P, O, _vp, _vp, _vp, _vp]; L.oracle_init.restype = ctypes.c_int
        L.oracle_iterate.argtypes = [P, O, _vp, _vp, _vp, d] + [_vp] * 10
        L.oracle_iterate.restype = ctypes.c_int
        L.oracle_procrustes_all.argtypes = [P, O, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        L.oracle_procrustes_all.restype = ctypes.c_int
        L.oracle_mttkrp.argtypes = [P, O, _vp, _vp, _vp, _vp, _vp, _vp, _vp, i32, _vp]
        L.oracle_mttkrp.restype = ctypes.c_int
        L.oracle_residual.argtypes = [P, O, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
        L.oracle_residual.restype = d
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(_vp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ small building blocks
def prox(kind: int, param: float, rho: float, x):
    f = lib().oracle_prox
    return np.array([f(kind, param, rho, float(v)) for v in np.ravel(x)]).reshape(np.shape(x))


def svd(A):
    A = _f64(A)
    m, n = A.shape
    p = min(m, n)
    U = np.zeros((m, p)); s = np.zeros(p); V = np.zeros((n, p))
    lib().oracle_svd(m, n, _p(A), _p(U), _p(s), _p(V))
    return U, s, V


def polar(A, tau: float = TAU_POLAR):
    A = _f64(A)
    Q = np.zeros_like(A)
    r = lib().oracle_polar(A.shape[0], A.shape[1], _p(A), tau, _p(Q))
    return Q, r


def knots(t1, tn, l, d=SPLINE_DEGREE):
    b = np.zeros(l + d + 1)
    lib().oracle_knots(t1, tn, l, d, _p(b))
    return b


def bspline_matrix(t, l, d=SPLINE_DEGREE):
    t = _f64(t)
    M = np.zeros((len(t), l))
    lib().oracle_bspline_matrix(_p(t), len(t), l, d, _p(M))
    return M


def patient_basis(t, l, d=SPLINE_DEGREE, tau=TAU_BASIS):
    t = _f64(t)
    C = np.zeros((len(t), l))
    lp = lib().oracle_patient_basis(_p(t), len(t), l, d, tau, _p(C))
    return C, lp


def cholesky(A):
    L = _f64(A).copy()
    rc = lib().oracle_cholesky(L.shape[0], _p(L))
    if rc:
        raise np.linalg.LinAlgError(f"non-positive pivot {rc - 1}")
    return L


def chol_solve(L, b):
    x = _f64(b).copy()
    lib().oracle_chol_solve(L.shape[0], _p(_f64(L)), _p(x))
    return x


def admm_mode(F, G, Zbar, D, kind, param, rho=0.0, n_inner=5, tol=0.0, steps=None):
    """One mode's cached-Cholesky ADMM (Alg.1 l.13-l.19). Returns (Zbar, D, rho).
    tol > 0: per-row inner stop (reading R-inner-tol); steps (int32 array of n rows) receives each
    row's step count."""
    F = _f64(F); G = _f64(G)
    Zb = _f64(Zbar).copy(); Dd = _f64(D).copy()
    rho_out = ctypes.c_double(0)
    rc = lib().oracle_admm_mode_tol(F.shape[0], F.shape[1], _p(F), _p(G), rho, n_inner, kind, param, tol, _p(Zb),
                                    _p(Dd), ctypes.byref(rho_out), None if steps is None else _p(steps))
    if rc:
        raise RuntimeError(f"oracle_admm_mode failed: {rc}")
    return Zb, Dd, rho_out.value


# ------------------------------------------------------------------ full iteration
def options_from_config(cfg, tau_polar=TAU_POLAR, tau_basis=TAU_BASIS, n_inner=None, rho=None, admm_tol=0.0):
    return _Options(kind_H=cfg.con_H[0], kind_W=cfg.con_W[0], kind_V=cfg.con_V[0],
                    param_H=cfg.con_H[1], param_W=cfg.con_W[1], param_V=cfg.con_V[1],
                    smooth_l=cfg.smooth_l, smooth_d=SPLINE_DEGREE, rho=cfg.rho if rho is None else rho,
                    n_inner=cfg.n_inner if n_inner is None else n_inner, tau_polar=tau_polar, tau_basis=tau_basis,
                    admm_tol=admm_tol)


def sparsity(V) -> float:
    """SPARSITY(V) = number of zero elements / size."""
    V = _f64(V)
    return lib().oracle_sparsity(V.size, _p(V))


class Oracle:
    """Oracle state for one problem (all patients on one host, serial)."""

    def __init__(self, prob, opts=None, R=None):
        self.prob = prob
        self.R = int(R or prob.cfg.R)
        self.o = opts if opts is not None else options_from_config(prob.cfg)
        self._arrays = [np.ascontiguousarray(prob.patient_row_ptr, np.int64), np.ascontiguousarray(prob.row_ptr, np.int64),
                        np.ascontiguousarray(prob.col, np.int32), _f64(prob.val),
                        None if prob.times is None else _f64(prob.times)]
        a = self._arrays
        self.P = _Problem(K=prob.K, J=prob.J, R=self.R, patient_row_ptr=a[0].ctypes.data, row_ptr=a[1].ctypes.data,
                          col=a[2].ctypes.data, val=a[3].ctypes.data,
                          times=None if a[4] is None else a[4].ctypes.data)
        K, J, R = prob.K, prob.J, self.R
        l = self.o.smooth_l
        rows = int(prob.patient_row_ptr[-1])
        self.C = np.zeros((rows, l)) if l > 0 else None
        self.m = np.zeros(K, np.int32)
        self.m_off = np.zeros(K + 1, np.int64)
        nx = ctypes.c_double(0)
        rc = lib().oracle_init(ctypes.byref(self.P), ctypes.byref(self.o), _p(self.C), _p(self.m), _p(self.m_off),
                               ctypes.byref(nx))
        if rc:
            raise RuntimeError(f"oracle_init failed: {rc}")
        self.normX = nx.value
        self.H = _f64(prob.H0[:R, :R]).copy()
        self.V = _f64(prob.V0[:, :R]).copy()
        self.W = _f64(prob.W0[:, :R]).copy()
        self.DH = np.zeros_like(self.H); self.DV = np.zeros_like(self.V); self.DW = np.zeros_like(self.W)
        self.Q = np.zeros((int(self.m_off[-1]), R))
        self.rank = np.zeros(K, np.int32)
        self.fits = []
        self.inner_steps = []
        self.diag = np.zeros(8)

    def iterate(self, n=1):
        for _ in range(n):
            fit = ctypes.c_double(0)
            rc = lib().oracle_iterate(ctypes.byref(self.P), ctypes.byref(self.o), _p(self.C), _p(self.m), _p(self.m_off),
                                      self.normX, _p(self.H), _p(self.V), _p(self.W), _p(self.DH), _p(self.DV),
                                      _p(self.DW), _p(self.Q), _p(self.rank), ctypes.byref(fit), _p(self.diag))
            if rc:
                raise RuntimeError(f"oracle_iterate failed: {rc}")
            self.fits.append(fit.value)
            self.inner_steps.append(tuple(int(x) for x in self.diag[5:8]))
        return self.fits

    def iterate_until(self, max_outer, outer_tol):
        """Outer loop with a stop ("while convergence criterion is not met", reading
        R-outer-tol): after iteration t >= 2, stop when |FIT_t - FIT_{t-1}| < outer_tol * max(|FIT_{t-1}|, 1),
        or after max_outer iterations. Returns the FIT values of this call."""
        out = []
        for _ in range(max_outer):
            f = self.iterate(1)[-1]
            out.append(f)
            if len(out) >= 2 and abs(out[-1] - out[-2]) < outer_tol * max(abs(out[-2]), 1.0):
                break
        return out

    def sparsity_V(self):
        return sparsity(self.V)

    def procrustes(self, H=None, V=None, W=None):
        """l.3-l.8 only, on the given (default: current) factors; fills self.Q, self.rank."""
        H = self.H if H is None else _f64(H); V = self.V if V is None else _f64(V); W = self.W if W is None else _f64(W)
        lib().oracle_procrustes_all(ctypes.byref(self.P), ctypes.byref(self.o), _p(self.C), _p(self.m), _p(self.m_off),
                                    _p(H), _p(V), _p(W), _p(self.Q), _p(self.rank))
        return self.Q

    def mttkrp(self, mode, H=None, V=None, W=None):
        """l.12 with the stored Q: mode 1 -> F_H (R x R), 2 -> F_V (J x R), 3 -> F_W (K x R)."""
        H = self.H if H is None else _f64(H); V = self.V if V is None else _f64(V); W = self.W if W is None else _f64(W)
        n = {1: self.R, 2: self.prob.J, 3: self.prob.K}[mode]
        F = np.zeros((n, self.R))
        lib().oracle_mttkrp(ctypes.byref(self.P), ctypes.byref(self.o), _p(self.C), _p(self.m), _p(self.m_off),
                            _p(self.Q), _p(H), _p(V), _p(W), mode, _p(F))
        return F

    def residual(self):
        """E = sum_k ||X_k - U_k S_k V^T||^2 with the stored Q and current factors."""
        return lib().oracle_residual(ctypes.byref(self.P), ctypes.byref(self.o), _p(self.C), _p(self.m),
                                     _p(self.m_off), _p(self.Q), _p(self.H), _p(self.V), _p(self.W))

    def Qk(self, k):
        return self.Q[self.m_off[k]:self.m_off[k + 1]]

    def U(self, k):
        """U_k = C_k Q_k H or Q_k H."""
        r0, r1 = self.prob.patient_row_ptr[k], self.prob.patient_row_ptr[k + 1]
        QH = self.Qk(k) @ self.H
        if self.C is None:
            return QH
        return self.C[r0:r1, :self.m[k]] @ QH

    def U_all(self):
        return np.concatenate([self.U(k) for k in range(self.prob.K)], axis=0)
