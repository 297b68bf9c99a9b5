"""GPU parity: the CUDA path (through the C ABI) against the oracle on identical seeded inputs.

Tolerances are BASELINE.json north_star's: every factor within 1e-9 relative Frobenius after one
outer iteration; FIT within 1e-7 absolute after 10 iterations. Sizes: the oracle finishes in
seconds (full Tiny and Small; prefixes of Medium/Large/Scale that still span many warps/blocks
and a ragged tail of patient lengths).
"""
import numpy as np
import pytest

import oracle
import synthgen

pytestmark = pytest.mark.gpu

CASES = [("tiny", None), ("small", None), ("medium", 6000), ("large", 1500), ("scale", 4000)]


def rel(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def copa_mod():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1803_04572_b200 as copa
    copa.lib()
    return copa


def _pair(copa, name, K):
    p = synthgen.generate(name, K=K)
    g = copa.Copa(p, copa.Options.from_config(p.cfg))
    o = oracle.Oracle(p)
    return p, g, o


@pytest.mark.parametrize("name,K", CASES)
def test_one_iteration_factors(copa_mod, name, K):
    p, g, o = _pair(copa_mod, name, K)
    fg = g.iterate(1)
    fo = o.iterate(1)
    H, V, W = [t.cpu().numpy() for t in g.factors()]
    DH, DV, DW = [t.cpu().numpy() for t in g.duals()]
    errs = {"H": rel(H, o.H), "V": rel(V, o.V), "W": rel(W, o.W), "DH": rel(DH, o.DH), "DV": rel(DV, o.DV),
            "DW": rel(DW, o.DW), "U": rel(g.U().cpu().numpy(), o.U_all())}
    if p.cfg.smooth_l == 0:
        errs["Q"] = rel(g.debug_state()["Qt"].cpu().numpy(), o.Q)
    assert abs(fg[0] - fo[0]) <= 1e-9, (fg, fo)
    for k, e in errs.items():
        assert e <= 1e-9, (name, k, e, errs)


@pytest.mark.parametrize("name,K", CASES)
def test_fit_after_ten_iterations(copa_mod, name, K):
    p, g, o = _pair(copa_mod, name, K)
    fg = g.iterate(10)
    fo = o.iterate(10)
    assert max(abs(a - b) for a, b in zip(fg, fo)) <= 1e-7, (fg, fo)


# NEXT N1: the paper's remaining constraint variants are prox-only changes — l0 on V
# (P:452-475), l1 on H, non-negativity + l1 on S_k and V. (Non-negativity on H as well drives H̄ to
# 0 in the first H update on this data, trace(G_W) = 0: both sides report that case, reading Z33.)
VARIANTS = [
    ("medium", 1500, dict(con_W=(3, 0.01), con_V=(3, 0.05))),
    ("medium", 1500, dict(con_V=(4, 1e-4))),
    ("small", 2000, dict(con_H=(2, 0.05), con_W=(3, 0.01), con_V=(4, 1e-4))),
]


@pytest.mark.parametrize("name,K,cons", VARIANTS)
def test_constraint_variants(copa_mod, name, K, cons):
    import dataclasses
    cfg = dataclasses.replace(synthgen.CONFIGS[name], **cons)
    p = synthgen.generate(cfg, K=K)
    g = copa_mod.Copa(p, copa_mod.Options.from_config(cfg))
    o = oracle.Oracle(p)
    fg = g.iterate(1)
    fo = o.iterate(1)
    H, V, W = [t.cpu().numpy() for t in g.factors()]
    for a, b, what in ((H, o.H, "H"), (V, o.V, "V"), (W, o.W, "W")):
        assert rel(a, b) <= 1e-9, (name, cons, what, rel(a, b))
    fg += g.iterate(4)
    fo += o.iterate(4)
    assert max(abs(a - b) for a, b in zip(fg, fo)) <= 1e-7, (fg, fo)


# N4: the second workload — non-smooth R = 40 (tall QR + 40 x 40 Jacobi per patient
# for I_k >= 40, the wide factorisation otherwise) and unconstrained PARAFAC2
# (identity prox on every factor).
N4_CASES = [("large_plain", 1200), ("small_unconstrained", 3000)]
# N2: smoothness with l = 33 > R = 15, the row-projection path
# (k_rowproj.cu: sparse M_k recomputed from the visit times, B_k per patient)
N2_CASES = [("medium_l33", 3000)]


def _q_parity(p, Qg, o):
    """Q~_k parity with the conditioning of the partial isometry: a kept direction
    with sigma_r = rho sigma_1 is determined only to ~eps / rho, so patients whose smallest kept
    ratio rho is below 1e-6 are checked against that first-order bound (x 1e3) one by one, and the
    rest, stacked, at north_star's 1e-9. Returns the stacked error of the well-conditioned patients."""
    from tests.helpers import dense_slices
    Xs = dense_slices(p)
    R = p.cfg.R
    good_g, good_o = [], []
    n_ill = 0
    for k in range(p.K):
        A = Xs[k] @ p.V0[:, :R] @ np.diag(p.W0[k, :R]) @ p.H0[:R, :R].T
        s = np.linalg.svd(A, compute_uv=False)
        kept = s[s > 1e-10 * s[0]] if s[0] > 0 else s[:0]
        rho = kept[-1] / s[0] if len(kept) else 1.0
        a, b = o.m_off[k], o.m_off[k + 1]
        if rho >= 1e-6:
            good_g.append(Qg[a:b]); good_o.append(o.Q[a:b])
        else:
            n_ill += 1
            err = np.linalg.norm(Qg[a:b] - o.Q[a:b])
            assert err <= 1e3 * 2.2e-16 / rho, (k, err, rho)
    print(f"[Q parity] {n_ill} of {p.K} patients with a kept sigma ratio < 1e-6 checked against eps/ratio")
    return rel(np.concatenate(good_g), np.concatenate(good_o))


@pytest.mark.parametrize("name,K", N4_CASES + N2_CASES)
def test_n4_one_iteration_factors(copa_mod, name, K):
    p, g, o = _pair(copa_mod, name, K)
    fg = g.iterate(1)
    fo = o.iterate(1)
    H, V, W = [t.cpu().numpy() for t in g.factors()]
    errs = {"H": rel(H, o.H), "V": rel(V, o.V), "W": rel(W, o.W), "U": rel(g.U().cpu().numpy(), o.U_all())}
    if p.cfg.smooth_l == 0:  # Q~ itself is basis-dependent under smoothness (reading R-spline-5)
        errs["Q"] = _q_parity(p, g.debug_state()["Qt"].cpu().numpy(), o)
    print(f"[margin] {name}: FIT {abs(fg[0] - fo[0]):.2e} " + " ".join(f"{k} {v:.2e}" for k, v in errs.items()))
    assert abs(fg[0] - fo[0]) <= 1e-9
    for k, e in errs.items():
        assert e <= 1e-9, (name, k, e, errs)
    st = g.stats()
    print(f"[rank-cut] {name}: near {st['polar_near']} min-kept {st['polar_min_kept']:.2e} "
          f"max-dropped {st['polar_max_dropped']:.2e}")


@pytest.mark.parametrize("name,K", N4_CASES + N2_CASES)
def test_n4_fit_after_ten_iterations(copa_mod, name, K):
    p, g, o = _pair(copa_mod, name, K)
    fg = g.iterate(10)
    fo = o.iterate(10)
    err = max(abs(a - b) for a, b in zip(fg, fo))
    print(f"[margin] {name} FIT(10): {err:.2e} / 1e-7")
    assert err <= 1e-7, (fg, fo)
