"""Input generator: determinism, prefix/shard consistency, CSR invariants, distribution shape."""
import numpy as np
import pytest

import synthgen


def test_deterministic_and_prefix_consistent():
    a = synthgen.generate("small", K=500)
    b = synthgen.generate("small", K=500)
    for x, y in [(a.patient_row_ptr, b.patient_row_ptr), (a.row_ptr, b.row_ptr), (a.col, b.col), (a.val, b.val),
                 (a.W0, b.W0), (a.V0, b.V0), (a.H0, b.H0)]:
        assert np.array_equal(x, y)
    # a shard [100, 300) equals the same patients of the prefix
    s = synthgen.generate("small", K=500, k_range=(100, 300))
    r0, r1 = a.patient_row_ptr[100], a.patient_row_ptr[300]
    assert np.array_equal(s.patient_row_ptr, a.patient_row_ptr[100:301] - r0)
    e0, e1 = a.row_ptr[r0], a.row_ptr[r1]
    assert np.array_equal(s.col, a.col[e0:e1]) and np.array_equal(s.val, a.val[e0:e1])
    assert np.array_equal(s.W0, a.W0[100:300])


@pytest.mark.parametrize("name", ["tiny", "small", "medium", "large", "scale"])
def test_csr_invariants(name):
    p = synthgen.generate(name, K=300)
    cfg = p.cfg
    I = np.diff(p.patient_row_ptr)
    assert I.min() >= cfg.ik_lo and I.max() <= cfg.ik_hi
    rn = np.diff(p.row_ptr)
    assert rn.min() >= 1 and rn.max() <= cfg.J
    assert p.col.min() >= 0 and p.col.max() < cfg.J
    for i in range(p.rows):  # distinct, sorted columns within each row
        c = p.col[p.row_ptr[i]:p.row_ptr[i + 1]]
        assert np.all(np.diff(c) > 0)
    assert np.all(np.isfinite(p.val)) and p.val.min() >= 1
    if cfg.times:
        for k in range(p.K):
            t = p.times[p.patient_row_ptr[k]:p.patient_row_ptr[k + 1]]
            assert np.all(np.diff(t) > 0) and t.min() >= 0 and t.max() <= 36.5 * len(t)
    else:
        assert p.times is None


def test_distribution_shapes():
    # Tiny: I_k ~ U{3..30} (mean 16.5), rows Poisson(4)+1 (mean 5), values U{1..5}
    t = synthgen.generate("tiny")
    assert abs(np.diff(t.patient_row_ptr).mean() - 16.5) < 1.5
    assert abs(np.diff(t.row_ptr).mean() - 5.0) < 0.15
    assert set(np.unique(t.val)) == {1.0, 2.0, 3.0, 4.0, 5.0}
    # Small: geometric mean 15 (clip [2,200] barely moves it), rows Poisson(5)+1, Zipf: feature 0 most frequent
    s = synthgen.generate("small", K=5000)
    assert abs(np.diff(s.patient_row_ptr).mean() - 15.5) < 1.0
    assert abs(np.diff(s.row_ptr).mean() - 6.0) < 0.1
    cnt = np.bincount(s.col, minlength=500)
    assert cnt[0] == cnt.max() and cnt[0] > 5 * cnt[50]
    # Medium: lognormal median 20
    m = synthgen.generate("medium", K=20000)
    assert abs(np.median(np.diff(m.patient_row_ptr)) - 20) <= 2
    # Large: binary values
    g = synthgen.generate("large", K=200)
    assert np.all(g.val == 1.0)


def test_shard_bounds_balanced():
    p = synthgen.generate("small", K=4000)
    nnz_k = np.diff(p.row_ptr[p.patient_row_ptr])
    for world in (1, 2, 3, 8):
        b = synthgen.shard_bounds(nnz_k, world)
        assert b[0] == 0 and b[-1] == p.K and np.all(np.diff(b) >= 0)
        per = np.array([nnz_k[b[r]:b[r + 1]].sum() for r in range(world)])
        assert per.sum() == nnz_k.sum()
        assert per.max() - per.min() <= 2 * nnz_k.max()
