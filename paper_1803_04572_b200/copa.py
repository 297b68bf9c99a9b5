"""Thin ctypes binding of libcopa.so (include/copa.h). Argument marshalling only — every step of
the outer iteration runs in the library's CUDA kernels. PyTorch provides device memory, the stream
and (optionally) the process-group allreduce; there is no CPU fallback: if the library is missing
or fails to load, :func:`lib` raises.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Callable, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libcopa.so")

NONE, NONNEG, L1, NONNEG_L1, L0 = 0, 1, 2, 3, 4
STATUS = {0: "OK", -1: "E_ARG", -2: "E_SHAPE", -3: "E_NONFINITE", -4: "E_CHOL", -5: "E_DEGENERATE", -6: "E_CUDA",
          -7: "E_COMM", -8: "E_WORKSPACE", -9: "E_UNSUPPORTED"}


class CopaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"copa {STATUS.get(status, status)} ({status}): {msg}")
        self.status = status


class _Constraint(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("param", ctypes.c_double)]


class _Problem(ctypes.Structure):
    _fields_ = [("K_local", ctypes.c_int64), ("K_global", ctypes.c_int64), ("J", ctypes.c_int64),
                ("R", ctypes.c_int32), ("rows", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("patient_row_ptr", ctypes.c_void_p), ("row_ptr", ctypes.c_void_p), ("col", ctypes.c_void_p),
                ("val", ctypes.c_void_p), ("visit_time", ctypes.c_void_p)]


ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p)


class _Options(ctypes.Structure):
    _fields_ = [("on_H", _Constraint), ("on_W", _Constraint), ("on_V", _Constraint),
                ("smooth_l", ctypes.c_int32), ("smooth_degree", ctypes.c_int32), ("rho", ctypes.c_double),
                ("admm_inner", ctypes.c_int32), ("rank_tol", ctypes.c_double), ("basis_tol", ctypes.c_double),
                ("admm_tol", ctypes.c_double), ("H0", ctypes.c_void_p), ("V0", ctypes.c_void_p), ("W0_local", ctypes.c_void_p),
                ("allreduce", ALLREDUCE_FN), ("allreduce_ctx", ctypes.c_void_p), ("stream", ctypes.c_void_p)]


class _Stats(ctypes.Structure):
    _fields_ = [("fit", ctypes.c_double), ("rho", ctypes.c_double * 3), ("normX", ctypes.c_double),
                ("iterations", ctypes.c_int64), ("fibers", ctypes.c_int64), ("state_rows", ctypes.c_int64),
                ("rank_deficient", ctypes.c_int64), ("sparsity_V", ctypes.c_double),
                ("inner_steps", ctypes.c_int64 * 3), ("polar_near", ctypes.c_int64),
                ("polar_min_kept", ctypes.c_double), ("polar_max_dropped", ctypes.c_double),
                ("basis_near", ctypes.c_int64), ("basis_min_kept", ctypes.c_double),
                ("basis_max_dropped", ctypes.c_double), ("tiles", ctypes.c_int64)]


class _State(ctypes.Structure):
    _fields_ = [("H", ctypes.c_void_p), ("V", ctypes.c_void_p), ("W_local", ctypes.c_void_p), ("DH", ctypes.c_void_p),
                ("DV", ctypes.c_void_p), ("DW_local", ctypes.c_void_p), ("WtW", ctypes.c_void_p),
                ("VtV", ctypes.c_void_p), ("iterations", ctypes.c_int64)]


class _Limits(ctypes.Structure):
    _fields_ = [("max_R", ctypes.c_int32), ("max_q", ctypes.c_int32), ("max_smooth_l", ctypes.c_int32),
                ("max_J", ctypes.c_int64)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libcopa.so (built by __graft_entry__.build()). Raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"{SO_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(SO_PATH)
        vp, i32, i64, P, O = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(_Problem), ctypes.POINTER(_Options)
        sz = ctypes.POINTER(ctypes.c_size_t)
        L.copa_workspace_size.argtypes = [P, O, sz]
        L.copa_init.argtypes = [P, O, vp, ctypes.c_size_t, ctypes.POINTER(vp)]
        L.copa_iterate.argtypes = [vp, i32, vp]
        L.copa_iterate_until.argtypes = [vp, i32, ctypes.c_double, vp, ctypes.POINTER(i32)]
        L.copa_set_state.argtypes = [vp, ctypes.POINTER(_State)]
        L.copa_get_state.argtypes = [vp, ctypes.POINTER(_State)]
        L.copa_get_factors.argtypes = [vp, vp, vp, vp]
        L.copa_get_duals.argtypes = [vp, vp, vp, vp]
        L.copa_get_U.argtypes = [vp, vp]
        L.copa_get_stats.argtypes = [vp, ctypes.POINTER(_Stats)]
        L.copa_fit_workspace_size.argtypes = [P, O, sz]
        L.copa_fit.argtypes = [P, O, vp, ctypes.c_size_t, i32, vp, vp, vp, vp]
        L.copa_destroy.argtypes = [vp]
        L.copa_destroy.restype = None
        L.copa_last_error.restype = ctypes.c_char_p
        L.copa_debug_state.argtypes = [vp, vp, vp, vp, vp, vp]
        L.copa_set_profiling.argtypes = [vp, i32]
        L.copa_get_phase_times.argtypes = [vp, vp, vp, i32, ctypes.POINTER(i32), ctypes.POINTER(i64)]
        L.copa_phase_name.argtypes = [i32]
        L.copa_phase_name.restype = ctypes.c_char_p
        L.copa_get_limits.argtypes = [ctypes.POINTER(_Limits)]
        L.copa_get_limits.restype = None
        for f in ("copa_workspace_size", "copa_init", "copa_iterate", "copa_iterate_until", "copa_set_state",
                  "copa_get_state",
                  "copa_get_factors", "copa_get_duals",
                  "copa_get_U", "copa_get_stats", "copa_fit_workspace_size", "copa_fit", "copa_debug_state",
                  "copa_set_profiling", "copa_get_phase_times"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise CopaError(st, lib().copa_last_error().decode())


def limits() -> dict:
    lim = _Limits()
    lib().copa_get_limits(ctypes.byref(lim))
    return {"max_R": lim.max_R, "max_q": lim.max_q, "max_smooth_l": lim.max_smooth_l, "max_J": lim.max_J}


@dataclasses.dataclass
class Options:
    """Mirror of copa_options (minus pointers). Defaults follow DESIGN.md's readings."""
    con_H: tuple = (NONE, 0.0)
    con_W: tuple = (NONNEG, 0.0)
    con_V: tuple = (NONE, 0.0)
    smooth_l: int = 0
    smooth_degree: int = 3
    rho: float = 0.0
    admm_inner: int = 5
    rank_tol: float = 1e-10
    basis_tol: float = 1e-6
    admm_tol: float = 0.0

    @staticmethod
    def from_config(cfg, **over) -> "Options":
        kw = dict(con_H=tuple(cfg.con_H), con_W=tuple(cfg.con_W), con_V=tuple(cfg.con_V), smooth_l=cfg.smooth_l,
                  rho=cfg.rho, admm_inner=cfg.n_inner)
        kw.update(over)
        return Options(**kw)

    def c_struct(self, H0, V0, W0, allreduce_cb, stream) -> "_Options":
        return _Options(on_H=_Constraint(*self.con_H), on_W=_Constraint(*self.con_W), on_V=_Constraint(*self.con_V),
                        smooth_l=self.smooth_l, smooth_degree=self.smooth_degree, rho=self.rho,
                        admm_inner=self.admm_inner, rank_tol=self.rank_tol, basis_tol=self.basis_tol,
                        admm_tol=self.admm_tol, H0=H0, V0=V0, W0_local=W0, allreduce=allreduce_cb,
                        allreduce_ctx=None, stream=stream)


def _torch():
    import torch
    return torch


class _CAI:
    """Zero-copy view of a raw device pointer for torch.as_tensor (allreduce callback)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "stream": None}


def torch_allreduce(group=None, device: str = "cuda") -> Callable:
    """Allreduce(sum) callback over torch.distributed for copa_options.allreduce.

    device="cuda": the library passes a device pointer and the stream it enqueues on; the
    all_reduce is issued with that stream as torch's current stream, so NCCL is ordered after the
    producing kernels and before the consuming ones without a host sync, whatever stream the
    handle was created with. device="cpu": host buffers (gloo), used by the multi-rank host-logic
    tests.
    """
    torch = _torch()
    import torch.distributed as dist

    def fn(ptr, n, stream, ctx):
        try:
            if device == "cpu":
                arr = np.ctypeslib.as_array((ctypes.c_double * int(n)).from_address(int(ptr)))
                t = torch.from_numpy(arr)
                dist.all_reduce(t, group=group)
            else:
                t = torch.as_tensor(_CAI(ptr, n), device="cuda")
                with torch.cuda.stream(torch.cuda.ExternalStream(int(stream or 0))):
                    dist.all_reduce(t, group=group)
            return 0
        except Exception:  # noqa: BLE001 - reported to the library as a status
            return 1
    return fn


def _dev(torch, a, dtype):
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


class Copa:
    """One shard of a COPA fit resident on the current CUDA device (copa_init ... copa_destroy)."""

    def __init__(self, prob, options: Options, R: Optional[int] = None, K_global: Optional[int] = None,
                 allreduce: Optional[Callable] = None, stream=None):
        torch = _torch()
        self.torch = torch
        L = lib()
        self.R = int(R or prob.R)
        self.J = int(prob.J)
        self.K = int(len(prob.patient_row_ptr) - 1)
        self.t_prp = _dev(torch, prob.patient_row_ptr, torch.int64)
        self.t_rp = _dev(torch, prob.row_ptr, torch.int64)
        self.t_col = _dev(torch, prob.col, torch.int32)
        self.t_val = _dev(torch, prob.val, torch.float64)
        self.t_times = _dev(torch, prob.times, torch.float64) if options.smooth_l > 0 else None
        self.t_H0 = _dev(torch, np.asarray(prob.H0)[:self.R, :self.R] if not isinstance(prob.H0, torch.Tensor) else prob.H0, torch.float64)
        self.t_V0 = _dev(torch, prob.V0, torch.float64)
        self.t_W0 = _dev(torch, prob.W0, torch.float64)
        self.rows = int(self.t_rp.numel() - 1)
        self.nnz = int(self.t_col.numel())
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self.p = _Problem(K_local=self.K, K_global=int(K_global or self.K), J=self.J, R=self.R, rows=self.rows,
                          nnz=self.nnz, patient_row_ptr=self.t_prp.data_ptr(), row_ptr=self.t_rp.data_ptr(),
                          col=self.t_col.data_ptr() if self.nnz else None, val=self.t_val.data_ptr() if self.nnz else None,
                          visit_time=self.t_times.data_ptr() if self.t_times is not None else None)
        self._cb = ALLREDUCE_FN(allreduce) if allreduce is not None else ALLREDUCE_FN()
        self.options = options
        self.o = options.c_struct(self.t_H0.data_ptr(), self.t_V0.data_ptr(), self.t_W0.data_ptr() if self.K else None,
                                  self._cb, self.stream.cuda_stream)
        nbytes = ctypes.c_size_t(0)
        _check(L.copa_workspace_size(ctypes.byref(self.p), ctypes.byref(self.o), ctypes.byref(nbytes)))
        self.ws = torch.empty(int(nbytes.value), dtype=torch.uint8, device="cuda")
        h = ctypes.c_void_p(0)
        _check(L.copa_init(ctypes.byref(self.p), ctypes.byref(self.o), self.ws.data_ptr(), nbytes.value,
                           ctypes.byref(h)))
        self.h = h
        self.fits: list = []

    # ---------------------------------------------------------------- iteration
    def iterate(self, n: int = 1) -> list:
        fits = np.zeros(max(n, 1))
        _check(lib().copa_iterate(self.h, n, fits.ctypes.data_as(ctypes.c_void_p)))
        self.fits.extend(fits[:n].tolist())
        return fits[:n].tolist()

    def iterate_until(self, max_outer: int, outer_tol: float) -> list:
        """copa_iterate_until: outer loop with the FIT-change stop (reading R-outer-tol)."""
        fits = np.zeros(max(max_outer, 1))
        done = ctypes.c_int32(0)
        _check(lib().copa_iterate_until(self.h, max_outer, outer_tol, fits.ctypes.data_as(ctypes.c_void_p),
                                        ctypes.byref(done)))
        out = fits[:done.value].tolist()
        self.fits.extend(out)
        return out

    _STATE_KEYS = ("H", "V", "W", "DH", "DV", "DW", "WtW", "VtV")

    def get_state(self) -> dict:
        """copa_get_state (checkpoint): factors, scaled duals and the two Grams, as device tensors."""
        t = self.torch
        R, J, K = self.R, self.J, self.K
        shapes = {"H": (R, R), "V": (J, R), "W": (max(K, 1), R), "DH": (R, R), "DV": (J, R), "DW": (max(K, 1), R),
                  "WtW": (R, R), "VtV": (R, R)}
        out = {k: t.empty(shapes[k], dtype=t.float64, device="cuda") for k in self._STATE_KEYS}
        st = _State(*[out[k].data_ptr() for k in self._STATE_KEYS], 0)
        _check(lib().copa_get_state(self.h, ctypes.byref(st)))
        out["W"] = out["W"][:K]
        out["DW"] = out["DW"][:K]
        out["iterations"] = self.stats()["iterations"]
        return out

    def set_state(self, state: dict):
        """copa_set_state (resume). WtW / VtV may be missing (recomputed from W and V)."""
        t = self.torch
        keep = {k: _dev(t, state[k], t.float64).contiguous() for k in self._STATE_KEYS if state.get(k) is not None}
        ptr = [keep[k].data_ptr() if k in keep and keep[k].numel() else None for k in self._STATE_KEYS]
        st = _State(*ptr, int(state.get("iterations", 0)))
        _check(lib().copa_set_state(self.h, ctypes.byref(st)))

    def iterate_async(self, n: int = 1):
        """Enqueue n outer iterations without a FIT host copy (the library still syncs once at the end)."""
        _check(lib().copa_iterate(self.h, n, None))

    # ---------------------------------------------------------------- outputs
    def factors(self):
        t = self.torch
        H = t.empty((self.R, self.R), dtype=t.float64, device="cuda")
        V = t.empty((self.J, self.R), dtype=t.float64, device="cuda")
        W = t.empty((max(self.K, 1), self.R), dtype=t.float64, device="cuda")
        _check(lib().copa_get_factors(self.h, H.data_ptr(), V.data_ptr(), W.data_ptr()))
        return H, V, W[:self.K]

    def duals(self):
        t = self.torch
        DH = t.empty((self.R, self.R), dtype=t.float64, device="cuda")
        DV = t.empty((self.J, self.R), dtype=t.float64, device="cuda")
        DW = t.empty((max(self.K, 1), self.R), dtype=t.float64, device="cuda")
        _check(lib().copa_get_duals(self.h, DH.data_ptr(), DV.data_ptr(), DW.data_ptr()))
        return DH, DV, DW[:self.K]

    def U(self):
        t = self.torch
        U = t.empty((max(self.rows, 1), self.R), dtype=t.float64, device="cuda")
        _check(lib().copa_get_U(self.h, U.data_ptr()))
        return U[:self.rows]

    def U_host(self) -> np.ndarray:
        """copa_get_U into a HOST buffer (the library stages patient chunks through device state)."""
        U = np.zeros((max(self.rows, 1), self.R))
        _check(lib().copa_get_U(self.h, U.ctypes.data_as(ctypes.c_void_p)))
        return U[:self.rows]

    def stats(self) -> dict:
        s = _Stats()
        _check(lib().copa_get_stats(self.h, ctypes.byref(s)))
        return {"fit": s.fit, "rho": list(s.rho), "normX": s.normX, "iterations": s.iterations, "fibers": s.fibers, "tiles": s.tiles,
                "state_rows": s.state_rows, "rank_deficient": s.rank_deficient, "sparsity_V": s.sparsity_V,
                "inner_steps": list(s.inner_steps), "polar_near": s.polar_near, "polar_min_kept": s.polar_min_kept,
                "polar_max_dropped": s.polar_max_dropped, "basis_near": s.basis_near,
                "basis_min_kept": s.basis_min_kept, "basis_max_dropped": s.basis_max_dropped}

    def set_profiling(self, on: bool = True):
        """Record CUDA events around each phase of the iteration (on the library's stream)."""
        _check(lib().copa_set_profiling(self.h, 1 if on else 0))

    def phase_times(self) -> dict:
        """{phase: (total_ms, calls)} accumulated since set_profiling(True), plus '_launches'."""
        ms = (ctypes.c_double * 32)()
        calls = (ctypes.c_int64 * 32)()
        n = ctypes.c_int32(0)
        launches = ctypes.c_int64(0)
        _check(lib().copa_get_phase_times(self.h, ms, calls, 32, ctypes.byref(n), ctypes.byref(launches)))
        out = {lib().copa_phase_name(i).decode(): (ms[i], int(calls[i])) for i in range(n.value)}
        out["_launches"] = int(launches.value)
        return out

    def debug_state(self):
        t = self.torch
        st = self.stats()
        S = st["state_rows"]
        Pp = t.empty((max(S, 1), self.R), dtype=t.float64, device="cuda")
        Qt = t.empty((max(S, 1), self.R), dtype=t.float64, device="cuda")
        m = t.empty(max(self.K, 1), dtype=t.int32, device="cuda")
        srow = t.empty(self.K + 1, dtype=t.int64, device="cuda")
        rank = t.empty(max(self.K, 1), dtype=t.int32, device="cuda")
        _check(lib().copa_debug_state(self.h, Pp.data_ptr(), Qt.data_ptr(), m.data_ptr(), srow.data_ptr(),
                                      rank.data_ptr()))
        return {"Pp": Pp[:S], "Qt": Qt[:S], "m": m[:self.K], "srow": srow, "rank": rank[:self.K]}

    def close(self):
        if getattr(self, "h", None):
            lib().copa_destroy(self.h)
            self.h = None
            self.ws = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def fit_host(prob, options: Options, n_outer: int, R: Optional[int] = None, stream=None, workspace=None,
             allreduce: Optional[Callable] = None):
    """End-to-end call with HOST inputs (copa_fit): H2D copies, init, n_outer iterations and D2H of
    the factors all happen inside the library. Returns (fits, H, V, W) as numpy arrays."""
    torch = _torch()
    L = lib()
    R = int(R or prob.R)
    J = int(prob.J)
    K = int(len(prob.patient_row_ptr) - 1)
    keep = []

    def hp(a, dtype):
        a = np.ascontiguousarray(a, dtype=dtype)
        keep.append(a)
        return a.ctypes.data

    prp = np.asarray(prob.patient_row_ptr)
    rp = np.asarray(prob.row_ptr)
    p = _Problem(K_local=K, K_global=K, J=J, R=R, rows=len(rp) - 1, nnz=len(prob.col),
                 patient_row_ptr=hp(prp, np.int64), row_ptr=hp(rp, np.int64), col=hp(prob.col, np.int32),
                 val=hp(prob.val, np.float64),
                 visit_time=hp(prob.times, np.float64) if options.smooth_l > 0 else None)
    stream = stream if stream is not None else torch.cuda.current_stream()
    cb = ALLREDUCE_FN(allreduce) if allreduce is not None else ALLREDUCE_FN()
    o = options.c_struct(hp(np.asarray(prob.H0)[:R, :R], np.float64), hp(prob.V0, np.float64),
                         hp(prob.W0, np.float64), cb, stream.cuda_stream)
    if workspace is None:
        nbytes = ctypes.c_size_t(0)
        _check(L.copa_fit_workspace_size(ctypes.byref(p), ctypes.byref(o), ctypes.byref(nbytes)))
        workspace = torch.empty(int(nbytes.value), dtype=torch.uint8, device="cuda")
    fits = np.zeros(max(n_outer, 1))
    H = np.zeros((R, R)); V = np.zeros((J, R)); W = np.zeros((max(K, 1), R))
    _check(L.copa_fit(ctypes.byref(p), ctypes.byref(o), workspace.data_ptr(), workspace.numel(), n_outer,
                      fits.ctypes.data, H.ctypes.data, V.ctypes.data, W.ctypes.data))
    return fits[:n_outer], H, V, W[:K]


def fit_workspace_bytes(prob, options: Options, R: Optional[int] = None) -> int:
    """copa_fit_workspace_size for host inputs (so callers can allocate the workspace outside a timed region)."""
    L = lib()
    R = int(R or prob.R)
    prp = np.ascontiguousarray(prob.patient_row_ptr, np.int64)
    rp = np.ascontiguousarray(prob.row_ptr, np.int64)
    col = np.ascontiguousarray(prob.col, np.int32)  # read: the fibers are counted from the host CSR
    p = _Problem(K_local=len(prp) - 1, K_global=len(prp) - 1, J=int(prob.J), R=R, rows=len(rp) - 1,
                 nnz=len(prob.col), patient_row_ptr=prp.ctypes.data, row_ptr=rp.ctypes.data, col=col.ctypes.data,
                 val=1,
                 visit_time=1 if options.smooth_l > 0 else None)
    o = options.c_struct(1, 1, 1, ALLREDUCE_FN(), None)
    nbytes = ctypes.c_size_t(0)
    _check(L.copa_fit_workspace_size(ctypes.byref(p), ctypes.byref(o), ctypes.byref(nbytes)))
    return int(nbytes.value)
