"""Full-size parity (BASELINE.json sizes, the bench launch configuration): one GPU outer iteration
against the oracle run over the WHOLE workload on all host cores (oracle/sharded.py: the serial C
oracle per nnz-balanced patient shard, per-patient sums added in shard order; pinned against the
single-process oracle by tests/test_multirank_cpu.py). Every row of H̄, V̄, W̄ and the FIT are
compared at north_star's 1e-9 after one iteration (Alg.1 l.3-l.20, FIT P:541-546)."""
import os

import numpy as np
import pytest

import synthgen

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
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name", ["medium", "large", "scale"])
def test_full_size_one_iteration_all_rows(copa, name):
    from oracle.sharded import ShardedOracle
    cfg = synthgen.CONFIGS[name]
    so = ShardedOracle(cfg, procs=os.cpu_count())
    try:
        fo = so.iterate(1)
        Wo, DWo = so.W_all()
        p = synthgen.generate(cfg)
        g = copa.Copa(p, copa.Options.from_config(cfg))
        fg = g.iterate(1)
        H, V, W = [x.cpu().numpy() for x in g.factors()]
        DH, DV, DW = [x.cpu().numpy() for x in g.duals()]
        g.close()
        errs = {"FIT": abs(fg[0] - fo[0]), "H": rel(H, so.H), "V": rel(V, so.V), "W": rel(W, Wo), "DH": rel(DH, so.DH),
                "DV": rel(DV, so.DV), "DW": rel(DW, DWo)}
        print(f"[full-size {name}] oracle {so.iter_s[-1]:.1f} s/iteration on {len(so.bounds)} processes; "
              + " ".join(f"{k} {v:.2e}" for k, v in errs.items()))
        for k, e in errs.items():
            assert e <= 1e-9, (name, k, e, errs)
    finally:
        so.close()
