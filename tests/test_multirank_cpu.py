"""N > 1 host logic on CPU with torch.distributed gloo, world_size 2 (no GPU):
nnz-balanced sharding, shard generation, the allreduce callback glue of the binding, and the
claim that the C1/C2 payloads (F_H; F_V, W^T W) are plain sums of per-shard partials."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synthgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synthgen
        from paper_1803_04572_b200.copa import torch_allreduce

        out = {}
        # 1) the binding's allreduce callback on host buffers
        buf = np.full(7, rank + 1.0)
        fn = torch_allreduce(device="cpu")
        out["cb_rc"] = fn(buf.ctypes.data, 7, None, None)
        out["cb_sum"] = buf.tolist()
        # 2) nnz-balanced shards of a workload prefix
        for name, K in (("small", 3000), ("medium", 1200)):
            nnz_k = synthgen.patient_nnz(name, K=K)
            b = synthgen.shard_bounds(nnz_k, world)
            k0, k1 = int(b[rank]), int(b[rank + 1])
            shard = synthgen.generate(name, K=K, k_range=(k0, k1))
            full = synthgen.generate(name, K=K)
            # per-shard oracle pieces with the GLOBAL H0, V0 and this shard's W0 rows
            o = oracle.Oracle(shard)
            o.procrustes()
            FH = torch.from_numpy(o.mttkrp(1).copy())
            FV = torch.from_numpy(o.mttkrp(2).copy())
            WtW = torch.from_numpy((o.W.T @ o.W).copy())
            nnz = torch.tensor([float(shard.nnz)])
            for t in (FH, FV, WtW, nnz):
                dist.all_reduce(t)
            of = oracle.Oracle(full)
            of.procrustes()
            out[name] = {
                "FH": float(np.linalg.norm(FH.numpy() - of.mttkrp(1)) / np.linalg.norm(of.mttkrp(1))),
                "FV": float(np.linalg.norm(FV.numpy() - of.mttkrp(2)) / np.linalg.norm(of.mttkrp(2))),
                "WtW": float(np.linalg.norm(WtW.numpy() - of.W.T @ of.W) / np.linalg.norm(of.W.T @ of.W)),
                "nnz_total": float(nnz.item()), "nnz_full": float(full.nnz), "shard_nnz": shard.nnz,
                "W0_rows_match": bool(np.array_equal(shard.W0, full.W0[k0:k1])),
            }
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        o = res[r]
        assert o["cb_rc"] == 0 and o["cb_sum"] == [3.0] * 7
        for name in ("small", "medium"):
            d = o[name]
            assert d["FH"] <= 1e-12 and d["FV"] <= 1e-12 and d["WtW"] <= 1e-12, d
            assert d["nnz_total"] == d["nnz_full"] and d["W0_rows_match"]
    for name in ("small", "medium"):
        a, b = res[0][name]["shard_nnz"], res[1][name]["shard_nnz"]
        assert abs(a - b) <= 0.05 * (a + b)  # nnz-balanced


@pytest.mark.parametrize("name,K,kw", [("tiny", None, {}), ("medium", 600, {}), ("small", 800, {"admm_tol": 1e-3})])
def test_sharded_oracle_matches_serial(name, K, kw):
    """oracle/sharded.py (the full-size parity reference and the all-cores CPU baseline) equals the
    serial oracle: the per-patient sums are only regrouped by shard (rounding-level differences)."""
    import oracle
    from oracle.sharded import ShardedOracle
    cfg = synthgen.CONFIGS[name]
    p = synthgen.generate(cfg, K=K)
    o = oracle.Oracle(p, opts=oracle.options_from_config(cfg, **kw))
    so = ShardedOracle(cfg, procs=3, K=p.K, **kw)
    try:
        fo = o.iterate(3)
        fs = so.iterate(3)
        assert max(abs(a - b) for a, b in zip(fo, fs)) <= 1e-12
        W, DW = so.W_all()
        for a, b in ((so.H, o.H), (so.V, o.V), (W, o.W), (DW, o.DW), (so.DV, o.DV)):
            assert np.linalg.norm(a - b) <= 1e-11 * max(np.linalg.norm(b), 1e-300)
        assert so.inner_steps[-1] == o.inner_steps[-1]
        ks = [0, p.K // 2, p.K - 1]
        U = so.U_rows(ks)
        for k in ks:
            assert np.allclose(U[k], o.U(k), rtol=0, atol=1e-11 * max(1.0, np.abs(o.U(k)).max()))
    finally:
        so.close()
