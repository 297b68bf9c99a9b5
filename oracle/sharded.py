"""ORACLE, sharded over host processes — test infrastructure only (see copa_oracle.c header).

One outer iteration of Algorithm 1 over a full BASELINE workload, computed by
the serial C oracle's own functions on contiguous patient shards in a process pool, with the
per-patient contributions summed in shard order. Only sums cross shards, exactly as the method
defines them:

  l.3-8   Procrustes Q_k                         per patient        (shard-local)
  l.11-19 H: F_H = Y_(1)(W ⊙ V) = sum over shards, G_H = (V^T V) * (W^T W) with W^T W summed;
          ADMM on the R x R problem (master)
  W:      F_W = Y_(3)(V ⊙ H_new) rows are per patient; G_W = (H^T H) * (V^T V); the row ADMM runs
          on each shard's rows (rows are independent, pin P20)
  V:      F_V = Y_(2)(W_new ⊙ H_new) = sum over shards; G_V = (H^T H) * (W^T W) summed; ADMM (master)
  FIT:    E = sum over patients

The decomposition into per-patient sums is the oracle's own (its MTTKRPs loop over patients and
accumulate); tests/test_multirank_cpu.py pins it against the single-process oracle. The pool also
gives the all-cores CPU baseline of bench.py (SURVEY 8(d) "How the oracle is timed").
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

_W = {}  # per-worker state (one shard per forked process)


def _init_worker(cfg, K, k0, k1, opts_kw):
    import oracle
    import synthgen
    p = synthgen.generate(cfg, K=K, k_range=(k0, k1))
    o = oracle.Oracle(p, opts=oracle.options_from_config(cfg, **opts_kw))
    _W.update(p=p, o=o)


def _setup(args):
    cfg, K, k0, k1, opts_kw = args
    _init_worker(cfg, K, k0, k1, opts_kw)
    o = _W["o"]
    return o.normX, o.W.T @ o.W, int(_W["p"].nnz)


def _phase_h(args):
    """Procrustes on (H, V, W_shard) and the shard's F_H partial (l.3-l.12, mode 1)."""
    H, V = args
    o = _W["o"]
    o.H = np.ascontiguousarray(H); o.V = np.ascontiguousarray(V)
    o.procrustes()
    return o.mttkrp(1)


def _phase_w(args):
    """F_W rows with the new H and the shard's W-row ADMM (mode 2 of Alg.1: W)."""
    import oracle
    H, G_W = args
    o = _W["o"]
    cfg = _W["p"].cfg
    o.H = np.ascontiguousarray(H)
    FW = o.mttkrp(3)
    steps = np.zeros(o.W.shape[0], np.int32)
    o.W, o.DW, rho = oracle.admm_mode(FW, G_W, o.W, o.DW, cfg.con_W[0], cfg.con_W[1], rho=o.o.rho,
                                      n_inner=o.o.n_inner, tol=o.o.admm_tol, steps=steps)
    return o.W.T @ o.W, rho, int(steps.sum())


def _phase_v(args):
    """The shard's F_V partial with the new H and W (mode 3 of Alg.1: V)."""
    return _W["o"].mttkrp(2)


def _phase_fit(args):
    V = args
    o = _W["o"]
    o.V = np.ascontiguousarray(V)
    return o.residual()


def _get_w(_):
    o = _W["o"]
    return _W["p"].k0, o.W.copy(), o.DW.copy()


def _get_u(args):
    ks = args
    o = _W["o"]
    k0 = _W["p"].k0
    return {int(k): o.U(int(k) - k0) for k in ks if k0 <= k < _W["p"].k1}


_FUNCS = {"setup": _setup, "h": _phase_h, "w": _phase_w, "v": _phase_v, "fit": _phase_fit, "get_w": _get_w,
          "get_u": _get_u}


def _worker(conn):
    while True:
        msg = conn.recv()
        if msg is None:
            break
        name, arg = msg
        try:
            conn.send((True, _FUNCS[name](arg)))
        except Exception as e:  # noqa: BLE001
            conn.send((False, repr(e)))


class ShardedOracle:
    """The oracle's outer iteration over a whole workload on `procs` host processes."""

    def __init__(self, cfg, procs=None, K=None, **opts_kw):
        import oracle
        import synthgen
        self.cfg = cfg
        self.K = cfg.K if K is None else int(K)
        self.procs = int(procs or os.cpu_count() or 1)
        nnz_k = synthgen.patient_nnz(cfg, K=self.K)
        nsh = min(self.procs, self.K)
        b = synthgen.shard_bounds(nnz_k, nsh)
        self.bounds = [(int(b[i]), int(b[i + 1])) for i in range(nsh) if b[i + 1] > b[i]]
        self.opts = oracle.options_from_config(cfg, **opts_kw)
        # spawn, not fork: the input generator runs OpenMP in this process, and libgomp's thread pool
        # does not survive fork (a forked child that enters OpenMP again deadlocks)
        ctx = mp.get_context("spawn")
        self.conns, self.workers = [], []
        for _ in self.bounds:  # one process per shard; its state stays in that process
            a_, b_ = ctx.Pipe()
            w = ctx.Process(target=_worker, args=(b_,), daemon=True)
            w.start()
            self.conns.append(a_)
            self.workers.append(w)
        t0 = time.perf_counter()
        for c, (k0, k1) in zip(self.conns, self.bounds):
            c.send(("setup", (cfg, self.K, k0, k1, opts_kw)))
        flat = [self._recv(c, w) for c, w in zip(self.conns, self.workers)]
        self.init_s = time.perf_counter() - t0
        self.normX = float(sum(x[0] for x in flat))
        self.WtW = sum((x[1] for x in flat), np.zeros((cfg.R, cfg.R)))
        self.nnz = int(sum(x[2] for x in flat))
        R = cfg.R
        p0 = synthgen.generate(cfg, K=1)
        self.H = p0.H0.copy()
        self.V = p0.V0.copy()
        self.DH = np.zeros((R, R))
        self.DV = np.zeros_like(self.V)
        self.fits = []
        self.inner_steps = []
        self.iter_s = []

    @staticmethod
    def _recv(c, w):
        while not c.poll(1.0):
            if not w.is_alive():
                raise RuntimeError(f"sharded oracle worker {w.pid} died (exit code {w.exitcode})")
        ok, val = c.recv()
        if not ok:
            raise RuntimeError(f"sharded oracle worker failed: {val}")
        return val

    def _map(self, fn, arg):
        """Run fn(arg) in every shard process; results in shard order (fixed-order sums)."""
        for c in self.conns:
            c.send((fn, arg))
        return [self._recv(c, w) for c, w in zip(self.conns, self.workers)]

    def iterate(self, n=1):
        import oracle
        cfg, o = self.cfg, self.opts
        for _ in range(n):
            t0 = time.perf_counter()
            FH = sum(self._map("h", (self.H, self.V)), np.zeros((cfg.R, cfg.R)))
            G_H = (self.V.T @ self.V) * self.WtW
            sH = np.zeros(cfg.R, np.int32)
            self.H, self.DH, _ = oracle.admm_mode(FH, G_H, self.H, self.DH, cfg.con_H[0], cfg.con_H[1], rho=o.rho,
                                                  n_inner=o.n_inner, tol=o.admm_tol, steps=sH)
            G_W = (self.H.T @ self.H) * (self.V.T @ self.V)
            outw = self._map("w", (self.H, G_W))
            self.WtW = sum((x[0] for x in outw), np.zeros((cfg.R, cfg.R)))
            FV = sum(self._map("v", None), np.zeros((cfg.J, cfg.R)))
            G_V = (self.H.T @ self.H) * self.WtW
            sV = np.zeros(cfg.J, np.int32)
            self.V, self.DV, _ = oracle.admm_mode(FV, G_V, self.V, self.DV, cfg.con_V[0], cfg.con_V[1], rho=o.rho,
                                                  n_inner=o.n_inner, tol=o.admm_tol, steps=sV)
            E = float(sum(self._map("fit", self.V)))
            self.fits.append(1.0 - E / self.normX)
            self.inner_steps.append((int(sH.sum()), int(sum(x[2] for x in outw)), int(sV.sum())))
            self.iter_s.append(time.perf_counter() - t0)
        return self.fits

    def W_all(self):
        parts = sorted(self._map("get_w", None), key=lambda x: x[0])
        return np.concatenate([x[1] for x in parts]), np.concatenate([x[2] for x in parts])

    def U_rows(self, ks):
        out = {}
        for d in self._map("get_u", list(ks)):
            out.update(d)
        return out

    def close(self):
        for c in getattr(self, "conns", []):
            try:
                c.send(None)
            except Exception:  # noqa: BLE001
                pass
        for w in getattr(self, "workers", []):
            w.join(5)
            if w.is_alive():
                w.terminate()
        self.conns, self.workers = [], []

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
