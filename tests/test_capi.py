"""C ABI checks that need no GPU: the library loads, exports every function include/copa.h declares,
reports its limits, and validates arguments on the host before touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def copa():
    from paper_1803_04572_b200 import _build
    _build.build()
    import paper_1803_04572_b200 as c
    c.lib()
    return c


def header_functions():
    src = open(os.path.join(ROOT, "include", "copa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(copa_[a-z_]+)\s*\(", src)) - {"copa_allreduce_fn"})


def test_exports_every_header_symbol(copa):
    names = header_functions()
    assert len(names) >= 15
    lib = ctypes.CDLL(copa.copa.SO_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_limits_and_phase_names(copa):
    lim = copa.limits()
    assert lim["max_R"] >= 40 and lim["max_q"] >= 10 and lim["max_smooth_l"] >= 9 and lim["max_J"] >= 1300
    L = copa.lib()
    names = [L.copa_phase_name(i).decode() for i in range(11)]
    assert names[0] == "spmm" and "scatter" in names and L.copa_phase_name(99) == b""


def _structs(copa, R=5, J=10, K=2, smooth=0, kind_V=1, param_V=0.0, admm=5, admm_tol=0.0):
    m = copa.copa
    p = m._Problem(K_local=K, K_global=K, J=J, R=R, rows=4, nnz=4, patient_row_ptr=8, row_ptr=8, col=8, val=8,
                   visit_time=8 if smooth else None)
    o = m._Options(on_H=m._Constraint(0, 0.0), on_W=m._Constraint(1, 0.0), on_V=m._Constraint(kind_V, param_V),
                   smooth_l=smooth, smooth_degree=3, rho=0.0, admm_inner=admm, rank_tol=1e-10, basis_tol=1e-6,
                   admm_tol=admm_tol, H0=8, V0=8, W0_local=8, allreduce=m.ALLREDUCE_FN(), allreduce_ctx=None, stream=None)
    return p, o


@pytest.mark.parametrize("kw,status", [
    ({"R": 0}, -1),                      # R < 1
    ({"R": 65}, -9),                     # beyond this build's limit
    ({"J": 0}, -9),                      # J outside [1, 65535]
    ({"admm": 0}, -1),                   # no inner steps
    ({"kind_V": 7}, -1),                 # unknown constraint
    ({"kind_V": 2, "param_V": -1.0}, -1),  # negative lambda
    ({"kind_V": 4, "param_V": 0.0}, -1),   # mu must be > 0
    ({"smooth": 65}, -9),                # l beyond the limit (64)
    ({"admm_tol": -1.0}, -1),            # negative inner-stop tolerance
])
def test_host_side_validation(copa, kw, status):
    p, o = _structs(copa, **kw)
    nbytes = ctypes.c_size_t(0)
    st = copa.lib().copa_workspace_size(ctypes.byref(p), ctypes.byref(o), ctypes.byref(nbytes))
    assert st == status, (kw, st, copa.lib().copa_last_error())
    assert copa.lib().copa_last_error()  # message set


def test_smooth_requires_times(copa):
    p, o = _structs(copa, smooth=7)
    p.visit_time = None
    nbytes = ctypes.c_size_t(0)
    assert copa.lib().copa_workspace_size(ctypes.byref(p), ctypes.byref(o), ctypes.byref(nbytes)) == -1


def test_null_handle_calls_fail_cleanly(copa):
    L = copa.lib()
    assert L.copa_iterate(None, 1, None) == -1
    assert L.copa_get_factors(None, None, None, None) == -1
    assert L.copa_get_stats(None, None) == -1
    L.copa_destroy(None)  # no-op


def test_no_cpu_fallback_in_binding():
    """The product binding never imports the oracle or runs compute on the host."""
    src = open(os.path.join(ROOT, "paper_1803_04572_b200", "copa.py")).read()
    assert "oracle" not in src.replace("oracle/", "")
    assert "import synthgen" not in src
