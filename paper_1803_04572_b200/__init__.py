"""B200-native COPA hot path (constrained PARAFAC2 via AO-ADMM, arXiv 1803.04572).

The compute lives in ``libcopa.so`` (csrc/*.cu, sm_100a, FP64) behind the C ABI in
``include/copa.h``; :mod:`.copa` is the thin ctypes binding. No CPU fallback.
"""
from .copa import (ALLREDUCE_FN, L0, L1, NONE, NONNEG, NONNEG_L1, Copa, CopaError, Options, fit_host,
                   fit_workspace_bytes, lib, limits, torch_allreduce)

__all__ = ["Copa", "CopaError", "Options", "fit_host", "fit_workspace_bytes", "lib", "limits", "torch_allreduce",
           "ALLREDUCE_FN", "NONE", "NONNEG", "L1", "NONNEG_L1", "L0"]
