"""More GPU tests through the C ABI: multi-rank on one GPU (threads + host allreduce; no kernels
wait on each other), edge cases, kernel-limit shape sweep, determinism, and sampled parity at
BASELINE.json's full sizes (the bench launch configuration)."""
import dataclasses
import threading

import numpy as np
import pytest

import oracle
import synthgen
from tests.helpers import make_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def copa():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1803_04572_b200 as c
    c.lib()
    return c


def rel(a, b):
    a = np.asarray(a); b = np.asarray(b)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ------------------------------------------------------------------ multi-rank (virtual, one GPU)
def _run_ranks(copa, shards, opts, K_global, n_iter):
    import torch
    from paper_1803_04572_b200.copa import _CAI
    world = len(shards)
    barrier = threading.Barrier(world)
    bufs = [None] * world
    out = [None] * world
    errs = []

    def make_cb(r):
        def cb(ptr, n, stream, ctx):
            try:
                torch.cuda.ExternalStream(stream).synchronize()
                t = torch.as_tensor(_CAI(ptr, n), device="cuda")
                bufs[r] = t.cpu().numpy().copy()
                barrier.wait()
                total = bufs[0].copy()
                for x in bufs[1:]:
                    total += x
                barrier.wait()
                t.copy_(torch.from_numpy(total).cuda())
                torch.cuda.synchronize()
                return 0
            except Exception as e:  # noqa: BLE001
                errs.append(e)
                return 1
        return cb

    def run(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                g = copa.Copa(shards[r], opts, K_global=K_global, allreduce=make_cb(r), stream=s)
                fits = g.iterate(n_iter)
                H, V, W = [x.cpu().numpy() for x in g.factors()]
                out[r] = (fits, H, V, W)
                g.close()
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not errs, errs
    return out


@pytest.mark.parametrize("name,K", [("small", 3000), ("medium", 3000)])
def test_two_virtual_ranks_match_single(copa, name, K):
    full = synthgen.generate(name, K=K)
    opts = copa.Options.from_config(full.cfg)
    nnz_k = np.diff(full.row_ptr[full.patient_row_ptr])
    b = synthgen.shard_bounds(nnz_k, 2)
    shards = [synthgen.generate(name, K=K, k_range=(int(b[r]), int(b[r + 1]))) for r in range(2)]
    res = _run_ranks(copa, shards, opts, K, 3)
    g = copa.Copa(full, opts)
    fits1 = g.iterate(3)
    H1, V1, W1 = [x.cpu().numpy() for x in g.factors()]
    # replicas are bit-identical across ranks (same allreduced sums, same redundant solves)
    assert np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[0][2], res[1][2])
    assert res[0][0] == res[1][0]
    assert rel(res[0][1], H1) <= 1e-11 and rel(res[0][2], V1) <= 1e-11
    assert rel(np.concatenate([res[0][3], res[1][3]]), W1) <= 1e-11
    assert max(abs(a - c) for a, c in zip(res[0][0], fits1)) <= 1e-11
    o = oracle.Oracle(full)
    fo = o.iterate(3)
    assert max(abs(a - c) for a, c in zip(res[0][0], fo)) <= 1e-9


def test_empty_shard_rank(copa):
    full = synthgen.generate("medium", K=800)
    opts = copa.Options.from_config(full.cfg)
    shards = [full, synthgen.generate("medium", K=800, k_range=(800, 800))]
    res = _run_ranks(copa, shards, opts, 800, 2)
    o = oracle.Oracle(full)
    fo = o.iterate(2)
    assert max(abs(a - c) for a, c in zip(res[1][0], fo)) <= 1e-9
    assert res[1][3].shape[0] == 0


# ------------------------------------------------------------------ edge cases
def _expect_status(copa, prob, opts, status):
    with pytest.raises(copa.CopaError) as e:
        g = copa.Copa(prob, opts)
        g.iterate(1)
    assert e.value.status == status, str(e.value)


def test_invalid_inputs(copa):
    p = synthgen.generate("small", K=50)
    opts = copa.Options.from_config(p.cfg)
    bad = dataclasses.replace(p, col=p.col.copy())
    bad.col[10] = p.J  # column out of range
    _expect_status(copa, bad, opts, -2)
    bad = dataclasses.replace(p, val=p.val.copy())
    bad.val[3] = np.nan
    _expect_status(copa, bad, opts, -3)
    bad = dataclasses.replace(p, col=p.col.copy())
    r0 = p.row_ptr[0]
    if p.row_ptr[1] - r0 >= 2:
        bad.col[r0 + 1] = bad.col[r0]  # duplicate column in a row
        _expect_status(copa, bad, opts, -2)
    m = synthgen.generate("medium", K=30)
    mo = copa.Options.from_config(m.cfg)
    t = m.times.copy()
    t[1] = t[0]  # not strictly increasing
    _expect_status(copa, dataclasses.replace(m, times=t), mo, -2)


def test_single_visit_patients_and_tiny_patients(copa):
    """I_k = 1 under smoothness: all knots coincide, M_k = 0, the patient contributes nothing
    (oracle: same via the recursion's 0/0 := 0); I_k < l: basis = whole row space."""
    rng = np.random.default_rng(5)
    J, R = 40, 6
    mats, times = [], []
    for k in range(60):
        I = 1 if k % 7 == 0 else int(rng.integers(2, 25))
        X = (rng.uniform(size=(I, J)) < 0.15) * rng.integers(1, 4, size=(I, J)).astype(float)
        X[:, k % J] += 1.0  # at least one nonzero per row
        mats.append(X)
        times.append(np.sort(rng.uniform(0, 36.5 * I, size=I)))
    p = make_problem(mats, R, base="medium", times=np.concatenate(times), con_V=(2, 0.1))
    g = copa.Copa(p, copa.Options.from_config(p.cfg))
    o = oracle.Oracle(p)
    fg = g.iterate(3)
    fo = o.iterate(3)
    assert max(abs(a - b) for a, b in zip(fg, fo)) <= 1e-9
    H, V, W = [x.cpu().numpy() for x in g.factors()]
    assert rel(H, o.H) <= 1e-9 and rel(V, o.V) <= 1e-9 and rel(W, o.W) <= 1e-9
    assert rel(g.U().cpu().numpy(), o.U_all()) <= 1e-9


def test_fiber_build_dense_rows_and_wide_patients(copa):
    """Init fiber build edge cases: rows with more nonzeros than a staged row chunk holds (256;
    read straight from global memory), row chunks cut short by the nonzero cap, and patients with
    more distinct features than one shared-memory window (256 ranks -> several windows)."""
    rng = np.random.default_rng(11)
    J, R = 700, 10
    mats, times = [], []
    for k in range(40):
        I = int(rng.integers(2, 30))
        dens = 0.02 if k % 3 else 0.45  # every third patient: dense rows (~315 nonzeros each)
        X = (rng.uniform(size=(I, J)) < dens) * rng.integers(1, 4, size=(I, J)).astype(float)
        if k % 5 == 0:
            X[0, :] = rng.integers(1, 4, size=J)  # one row with all 700 features
        X[:, k % J] += 1.0
        mats.append(X)
        times.append(np.sort(rng.uniform(0, 36.5 * I, size=I)))
    p = make_problem(mats, R, base="medium", times=np.concatenate(times), con_V=(2, 0.1))
    g = copa.Copa(p, copa.Options.from_config(p.cfg))
    o = oracle.Oracle(p)
    fg = g.iterate(1)
    fo = o.iterate(1)
    H, V, W = [x.cpu().numpy() for x in g.factors()]
    assert abs(fg[0] - fo[0]) <= 1e-9
    for a, b, what in ((H, o.H, "H"), (V, o.V, "V"), (W, o.W, "W")):
        assert rel(a, b) <= 1e-9, (what, rel(a, b))


@pytest.mark.parametrize("R,l,J", [(3, 0, 120), (16, 0, 120), (8, 5, 120), (24, 9, 120), (40, 12, 120), (20, 16, 120),
                                   (64, 16, 120), (20, 7, 4000), (40, 7, 30000), (8, 12, 120), (10, 20, 120),
                                   (40, 48, 300), (5, 60, 120)])
def test_shape_sweep(copa, R, l, J):
    """Kernel template/limit coverage: tall and wide polar, MMA tile counts, smooth l up to 16, and
    pass B's label groups: J = 4000 needs G = 4 F_V slices; J = 30000 (R = 40) fits no smem slice
    and takes the FP64-atomic fallback; l >= R (SURVEY N2 regime: smooth patients with l'_k >= R take
    the tall polar)."""
    base = "medium" if l else "small"
    cfg = dataclasses.replace(synthgen.CONFIGS[base], R=R, smooth_l=l, K=400, J=J)
    p = synthgen.generate(cfg)
    g = copa.Copa(p, copa.Options.from_config(cfg))
    o = oracle.Oracle(p)
    fg = g.iterate(1)
    fo = o.iterate(1)
    H, V, W = [x.cpu().numpy() for x in g.factors()]
    assert abs(fg[0] - fo[0]) <= 1e-9
    for a, b, what in ((H, o.H, "H"), (V, o.V, "V"), (W, o.W, "W")):
        assert rel(a, b) <= 1e-9, (R, l, what, rel(a, b))


def test_deterministic_smooth_path(copa):
    p = synthgen.generate("medium", K=5000)
    outs = []
    for _ in range(2):
        g = copa.Copa(p, copa.Options.from_config(p.cfg))
        f = g.iterate(3)
        outs.append((f, [x.cpu().numpy() for x in g.factors()]))
        g.close()
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a, b)


# ------------------------------------------------------------------ full sizes: sampled outputs
@pytest.mark.parametrize("name", ["medium", "large", "scale"])
def test_full_size_sampled_patients(copa, name):
    """BASELINE.json full size, bench launch configuration: one GPU outer iteration; for a random
    sample of patients the oracle recomputes U_k = C_k Q_k H̄_new and the W-row update one by one
    (given the GPU's H̄_new, which needs every patient) and they must agree."""
    cfg = synthgen.CONFIGS[name]
    p = synthgen.generate(cfg)
    g = copa.Copa(p, copa.Options.from_config(cfg))
    g.iterate(1)
    Hn, Vn, Wn = [x.cpu().numpy() for x in g.factors()]
    U = g.U()
    rng = np.random.default_rng(7)
    ks = np.sort(rng.choice(p.K, size=40, replace=False))
    num_u = den_u = num_w = den_w = 0.0
    for k in ks:
        sub = synthgen.generate(cfg, k_range=(int(k), int(k) + 1))
        o = oracle.Oracle(sub)
        o.procrustes(H=p.H0, V=p.V0, W=p.W0[k:k + 1])
        r0, r1 = p.patient_row_ptr[k], p.patient_row_ptr[k + 1]
        Uref = o.C[:, :o.m[0]] @ o.Qk(0) @ Hn if o.C is not None else o.Qk(0) @ Hn
        Ug = U[r0:r1].cpu().numpy()
        num_u += np.linalg.norm(Ug - Uref) ** 2
        den_u += np.linalg.norm(Uref) ** 2
        FW = o.mttkrp(3, H=Hn, V=p.V0, W=p.W0[k:k + 1])
        G = (Hn.T @ Hn) * (p.V0.T @ p.V0)
        wk, _, _ = oracle.admm_mode(FW, G, p.W0[k:k + 1], np.zeros((1, cfg.R)), cfg.con_W[0], cfg.con_W[1],
                                    rho=cfg.rho, n_inner=cfg.n_inner)
        num_w += np.linalg.norm(Wn[k] - wk[0]) ** 2
        den_w += np.linalg.norm(wk[0]) ** 2
    assert np.sqrt(num_u / den_u) <= 1e-9
    assert np.sqrt(num_w / den_w) <= 1e-9
    st = g.stats()
    assert 0.0 < st["fit"] < 1.0
