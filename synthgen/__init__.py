"""Seeded synthetic inputs for COPA (input synthesis only — none of the method's arithmetic).

Shared by ``oracle/`` (CPU checker) and ``paper_1803_04572_b200`` (CUDA path); neither imports the
other. The five BASELINE.json configs are encoded in :data:`CONFIGS` with the readings listed in
DESIGN.md §3 ("Input recipe"). Randomness is counter-based per patient (see ``synthgen.c``), so a
patient prefix ``K=k`` or a range ``k_range=(k0, k1)`` is bit-identical to the same patients of
the full workload.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynthgen.so")


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synthgen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


class _GenConfig(ctypes.Structure):
    _fields_ = [
        ("K", ctypes.c_int64), ("J", ctypes.c_int32), ("ik_dist", ctypes.c_int32),
        ("ik_a", ctypes.c_double), ("ik_b", ctypes.c_double),
        ("ik_lo", ctypes.c_int32), ("ik_hi", ctypes.c_int32),
        ("row_lambda", ctypes.c_double), ("zipf_s", ctypes.c_double),
        ("val_dist", ctypes.c_int32), ("times", ctypes.c_int32), ("seed", ctypes.c_uint64),
    ]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        _lib.gen_patient_rows.argtypes = [P(_GenConfig), ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        _lib.gen_row_sizes.argtypes = [P(_GenConfig), ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        _lib.gen_fill.argtypes = [P(_GenConfig), ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib.gen_uniform.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
    return _lib


# Constraint kinds (same integer codes as include/copa.h's copa_kind; plain data, no arithmetic).
NONE, NONNEG, L1, NONNEG_L1, L0 = 0, 1, 2, 3, 4


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    baseline: str            # the exact BASELINE.json configs[] string
    K: int
    J: int
    ik_dist: int             # 0 uniform, 1 geometric, 2 lognormal
    ik_a: float
    ik_b: float
    ik_lo: int
    ik_hi: int
    row_lambda: float
    zipf_s: float
    val_dist: int            # 0 uniform 1..5, 1 1+Poisson(1), 2 const 1
    times: bool
    R: int
    con_H: tuple
    con_W: tuple
    con_V: tuple
    smooth_l: int            # 0 = no smoothness
    rho: float               # > 0 fixed, <= 0 automatic trace(G)/R
    n_inner: int
    n_outer: int
    seed: int = 0


_BASELINE_STRINGS = [
    "Tiny: K=200 patients, J=100 features, I_k uniform in [3,30], each visit row has Poisson(4)+1 distinct features chosen uniformly, values integer counts uniform 1-5 stored FP64 CSR; rank R=5, constraints non-negativity on S_k and V only, ρ=1, 5 ADMM inner steps, 10 outer iterations, seed 0",
    "Small: K=20,000, J=500, I_k geometric mean 15 clipped to [2,200], visit rows Poisson(5)+1 features drawn Zipf(s=1.1) over J, counts 1+Poisson(1); R=10; non-negativity on S_k and V plus L1 on V (λ=0.1); 10 outer iterations",
    "EHR-shaped medium: K=250,000, J=1,300, I_k log-normal (median 20, σ=1.0) clipped to [2,1000], visit timestamps sorted uniform on [0,365·I_k/10] days, rows Poisson(6)+1 Zipf(1.1) features, counts 1+Poisson(1); R=15; full COPA: temporal smoothness on U_k via M-spline basis (l=7 knots over each patient's times), L1 on V (λ=0.1), non-negativity on S_k; 10 outer iterations",
    "EHR-shaped large, high rank: K=1,000,000, J=300, I_k log-normal (median 30, σ=1.2) clipped to [2,2000], rows Poisson(8)+1 Zipf(1.0) features, binary values; R=40; smoothness (l=9) + L1 on V (λ=0.05) + non-negativity on S_k; 5 outer iterations",
    "Multi-GPU scaling: K=4,000,000, J=1,300, I_k log-normal (median 25, σ=1.1) clipped to [2,2000], rows Poisson(6)+1 Zipf(1.1) features, counts 1+Poisson(1) (≈1B nonzeros); R=20; full constraint set; patients sharded nnz-balanced at 1/2/4/8 B200, 5 outer iterations",
]

CONFIGS = {
    "tiny": Config("tiny", _BASELINE_STRINGS[0], K=200, J=100, ik_dist=0, ik_a=0, ik_b=0, ik_lo=3, ik_hi=30,
                   row_lambda=4.0, zipf_s=0.0, val_dist=0, times=False, R=5,
                   con_H=(NONE, 0.0), con_W=(NONNEG, 0.0), con_V=(NONNEG, 0.0), smooth_l=0, rho=1.0,
                   n_inner=5, n_outer=10),
    "small": Config("small", _BASELINE_STRINGS[1], K=20_000, J=500, ik_dist=1, ik_a=1.0 / 15.0, ik_b=0, ik_lo=2,
                    ik_hi=200, row_lambda=5.0, zipf_s=1.1, val_dist=1, times=False, R=10,
                    con_H=(NONE, 0.0), con_W=(NONNEG, 0.0), con_V=(NONNEG_L1, 0.1), smooth_l=0, rho=0.0,
                    n_inner=5, n_outer=10),
    "medium": Config("medium", _BASELINE_STRINGS[2], K=250_000, J=1300, ik_dist=2, ik_a=20.0, ik_b=1.0, ik_lo=2,
                     ik_hi=1000, row_lambda=6.0, zipf_s=1.1, val_dist=1, times=True, R=15,
                     con_H=(NONE, 0.0), con_W=(NONNEG, 0.0), con_V=(L1, 0.1), smooth_l=7, rho=0.0,
                     n_inner=5, n_outer=10),
    "large": Config("large", _BASELINE_STRINGS[3], K=1_000_000, J=300, ik_dist=2, ik_a=30.0, ik_b=1.2, ik_lo=2,
                    ik_hi=2000, row_lambda=8.0, zipf_s=1.0, val_dist=2, times=True, R=40,
                    con_H=(NONE, 0.0), con_W=(NONNEG, 0.0), con_V=(L1, 0.05), smooth_l=9, rho=0.0,
                    n_inner=5, n_outer=5),
    "scale": Config("scale", _BASELINE_STRINGS[4], K=4_000_000, J=1300, ik_dist=2, ik_a=25.0, ik_b=1.1, ik_lo=2,
                    ik_hi=2000, row_lambda=6.0, zipf_s=1.1, val_dist=1, times=True, R=20,
                    con_H=(NONE, 0.0), con_W=(NONNEG, 0.0), con_V=(L1, 0.1), smooth_l=7, rho=0.0,
                    n_inner=5, n_outer=5),
}

# Derived workloads of SURVEY 8(f) (not BASELINE configs; same seeded data as their base config):
#   N4 non-smooth high rank: Large's data and constraints without the spline basis (R = 40 polar on
#   the raw I_k x R factors: tall QR + 40 x 40 Jacobi for I_k >= 40);
#   N4 unconstrained PARAFAC2: Small's data with the identity prox on every factor (a CP-ALS-like
#   step, the SPARTan-style model of PAPER.md:535).
CONFIGS["large_plain"] = dataclasses.replace(
    CONFIGS["large"], name="large_plain", smooth_l=0,
    baseline=CONFIGS["large"].baseline + " [SURVEY 8(f) N4 variant: no smoothness]")
#   N2 smoothness in the paper's regime: Medium's data with l = 33 basis functions at R = 15 (the
#   paper's CHOA setting), l > R.
CONFIGS["medium_l33"] = dataclasses.replace(
    CONFIGS["medium"], name="medium_l33", smooth_l=33,
    baseline=CONFIGS["medium"].baseline + " [SURVEY 8(f) N2 variant: l = 33 basis functions, PAPER.md:584]")
CONFIGS["small_unconstrained"] = dataclasses.replace(
    CONFIGS["small"], name="small_unconstrained", con_H=(NONE, 0.0), con_W=(NONE, 0.0), con_V=(NONE, 0.0),
    baseline=CONFIGS["small"].baseline + " [SURVEY 8(f) N4 variant: unconstrained, identity prox]")


@dataclasses.dataclass
class Problem:
    """One irregular sparse tensor (a contiguous patient range) plus seeded initial factors.

    All arrays are host numpy arrays; the CSR layout matches include/copa.h's copa_problem:
    patient_row_ptr[K_local+1] (int64, rows), row_ptr[rows+1] (int64, nnz), col (int32), val (f64),
    times (f64 per row or None). H0 (R×R), V0 (J×R), W0 (K_local×R) row-major float64.
    """
    cfg: Config
    k0: int
    k1: int
    patient_row_ptr: np.ndarray
    row_ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    times: Optional[np.ndarray]
    H0: np.ndarray
    V0: np.ndarray
    W0: np.ndarray

    @property
    def K(self) -> int:
        return self.k1 - self.k0

    @property
    def J(self) -> int:
        return self.cfg.J

    @property
    def R(self) -> int:
        return self.cfg.R

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def rows(self) -> int:
        return int(self.patient_row_ptr[-1])


def _cstruct(cfg: Config, K: int) -> _GenConfig:
    return _GenConfig(K=K, J=cfg.J, ik_dist=cfg.ik_dist, ik_a=cfg.ik_a, ik_b=cfg.ik_b, ik_lo=cfg.ik_lo,
                      ik_hi=cfg.ik_hi, row_lambda=cfg.row_lambda, zipf_s=cfg.zipf_s, val_dist=cfg.val_dist,
                      times=1 if cfg.times else 0, seed=cfg.seed)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def generate(name_or_cfg, K: Optional[int] = None, k_range: Optional[tuple] = None, seed: Optional[int] = None,
             alloc=np.empty) -> Problem:
    """Generate patients [k0, k1) of a config (default: all K of the config).

    ``K`` truncates the workload to its first K patients; ``k_range`` selects a shard.
    ``alloc(shape, dtype)`` lets the caller place the big arrays (e.g. in pinned memory).
    """
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    if seed is not None:
        cfg = dataclasses.replace(cfg, seed=seed)
    lib = _load()
    Kfull = cfg.K if K is None else int(K)
    k0, k1 = (0, Kfull) if k_range is None else (int(k_range[0]), int(k_range[1]))
    n = k1 - k0
    cs = _cstruct(cfg, Kfull)
    I = np.empty(n, dtype=np.int32)
    lib.gen_patient_rows(ctypes.byref(cs), k0, k1, _ptr(I))
    prp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(I, out=prp[1:])
    rows = int(prp[-1])
    rn = np.empty(rows, dtype=np.int32)
    lib.gen_row_sizes(ctypes.byref(cs), k0, k1, _ptr(prp), _ptr(rn))
    rp = alloc((rows + 1,), np.int64)
    rp[0] = 0
    np.cumsum(rn, out=rp[1:])
    nnz = int(rp[-1])
    col = alloc((nnz,), np.int32)
    val = alloc((nnz,), np.float64)
    times = alloc((rows,), np.float64) if cfg.times else None
    lib.gen_fill(ctypes.byref(cs), k0, k1, _ptr(prp), _ptr(rp), _ptr(col), _ptr(val),
                 _ptr(times) if times is not None else None)
    R = cfg.R
    H0 = np.empty((R, R)); V0 = np.empty((cfg.J, R)); W0 = np.empty((n, R))
    lib.gen_uniform(cfg.seed, 0, 0, R * R, _ptr(H0))
    lib.gen_uniform(cfg.seed, 1, 0, cfg.J * R, _ptr(V0))
    lib.gen_uniform(cfg.seed, 2, k0 * R, n * R, _ptr(W0))
    return Problem(cfg, k0, k1, prp, rp, col, val, times, H0, V0, W0)


def patient_nnz(name_or_cfg, K: Optional[int] = None) -> np.ndarray:
    """nnz per patient of a workload without generating columns/values (for nnz-balanced sharding)."""
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    lib = _load()
    Kfull = cfg.K if K is None else int(K)
    cs = _cstruct(cfg, Kfull)
    I = np.empty(Kfull, dtype=np.int32)
    lib.gen_patient_rows(ctypes.byref(cs), 0, Kfull, _ptr(I))
    prp = np.zeros(Kfull + 1, dtype=np.int64)
    np.cumsum(I, out=prp[1:])
    rn = np.empty(int(prp[-1]), dtype=np.int32)
    lib.gen_row_sizes(ctypes.byref(cs), 0, Kfull, _ptr(prp), _ptr(rn))
    c = np.zeros(len(rn) + 1, dtype=np.int64)
    np.cumsum(rn, out=c[1:])
    return np.diff(c[prp])


def shard_bounds(patient_nnz: np.ndarray, world: int) -> np.ndarray:
    """Contiguous patient ranges with nonzeros balanced: bounds[r]..bounds[r+1].

    Rank r takes the patients whose cumulative nnz midpoint falls in [r/world, (r+1)/world) of the
    total. Pure index bookkeeping (host logic), shared by bench and tests.
    """
    c = np.concatenate([[0], np.cumsum(patient_nnz, dtype=np.int64)])
    total = c[-1]
    K = len(patient_nnz)
    bounds = np.zeros(world + 1, dtype=np.int64)
    for r in range(1, world):
        bounds[r] = int(np.searchsorted(c, (total * r) // world, side="left"))
    bounds[world] = K
    return np.maximum.accumulate(bounds)
