"""Shared test helpers: planted / hand-built problems (input construction only)."""
from __future__ import annotations

import dataclasses

import numpy as np

import synthgen


def csr_from_dense(mats):
    """Stack dense patient matrices X_k (I_k x J) into the copa_problem CSR layout."""
    prp = [0]
    rp = [0]
    cols, vals = [], []
    for X in mats:
        for row in X:
            nz = np.nonzero(row)[0]
            cols.extend(nz.tolist())
            vals.extend(row[nz].tolist())
            rp.append(rp[-1] + len(nz))
        prp.append(prp[-1] + X.shape[0])
    return (np.array(prp, np.int64), np.array(rp, np.int64), np.array(cols, np.int32), np.array(vals, np.float64))


def make_problem(mats, R, base="tiny", times=None, H0=None, V0=None, W0=None, seed=0, **cfg_over):
    """A synthgen.Problem from explicit dense slices (for planted / special-case tests)."""
    J = mats[0].shape[1]
    cfg = dataclasses.replace(synthgen.CONFIGS[base], K=len(mats), J=J, R=R, **cfg_over)
    rng = np.random.default_rng(seed)
    prp, rp, col, val = csr_from_dense(mats)
    H0 = rng.uniform(size=(R, R)) if H0 is None else H0
    V0 = rng.uniform(size=(J, R)) if V0 is None else V0
    W0 = rng.uniform(size=(len(mats), R)) if W0 is None else W0
    return synthgen.Problem(cfg, 0, len(mats), prp, rp, col, val, times, np.ascontiguousarray(H0),
                            np.ascontiguousarray(V0), np.ascontiguousarray(W0))


def dense_slices(prob):
    """Dense X_k (I_k x J) for every patient of a (small) problem."""
    out = []
    for k in range(prob.K):
        r0, r1 = prob.patient_row_ptr[k], prob.patient_row_ptr[k + 1]
        X = np.zeros((r1 - r0, prob.J))
        for i in range(r0, r1):
            a, b = prob.row_ptr[i], prob.row_ptr[i + 1]
            X[i - r0, prob.col[a:b]] = prob.val[a:b]
        out.append(X)
    return out


def planted(K, Ilo, Ihi, J, R, seed, nonneg=True):
    """Noise-free PARAFAC2 model X_k = Q*_k H* S*_k V*^T with I_k >= R (SPEC S:66-73 style)."""
    rng = np.random.default_rng(seed)
    H = rng.uniform(size=(R, R))
    V = rng.uniform(size=(J, R)) if nonneg else rng.standard_normal((J, R))
    W = rng.uniform(0.5, 1.5, size=(K, R))
    mats, Qs = [], []
    for k in range(K):
        I = int(rng.integers(Ilo, Ihi + 1))
        Q, _ = np.linalg.qr(rng.standard_normal((I, R)))
        Qs.append(Q)
        mats.append(Q @ H @ np.diag(W[k]) @ V.T)
    return mats, Qs, H, V, W
