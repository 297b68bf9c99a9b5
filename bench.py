#!/usr/bin/env python
"""bench.py — throughput of one COPA outer iteration (Alg.1 l.3-l.20 + FIT) on B200, FP64.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config scale] [--impl ours|reference]

A "step" is one outer iteration over all patients of the workload (BASELINE.json configs[4],
"Multi-GPU scaling", by default; --config picks another). With N > 1 (torchrun) the patients are
sharded nnz-balanced over the ranks and the two per-iteration allreduces (F_H; [F_V | W^T W | M])
run over NCCL — strong scaling. Timing: W untimed warm-up iterations, then exactly K iterations
bracketed by barrier + synchronize, CUDA events on the library's stream, max over ranks. The
inputs (tens of GB for the default workload) are far larger than L2, so no L2 flush is done.

Prints ONE JSON line on rank 0 (schema in DESIGN.md §6). --impl reference times the FP64 CPU
oracle (oracle/) on a bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthgen  # noqa: E402

METRIC = "COPA outer iteration throughput (nonzeros per second; sec/iteration = ms_per_step/1000)"
# Patients per host core of the bounded oracle sample: ~2-3 s of one oracle outer iteration per
# core; the sample is this many patients times the cores used, times SAMPLE_SCALE.
ORACLE_PER_CORE = {"tiny": 200, "small": 20000, "medium": 12000, "large": 1500, "scale": 8000}
SAMPLE_SCALE = 4
FP64_PEAK_TFLOPS = 34.2  # measured DFMA loop on this pool's B200 at 1965 MHz (tools/probe_fp64.cu, profiles/)
DMMA_PEAK_TFLOPS = 36.9  # measured mma.sync m8n8k4 f64 (SASS DMMA) loop, same box (tools/probe_dmma*.cu)
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="scale", choices=sorted(synthgen.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return FALLBACK_HBM_GBS, "fallback"


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.samples = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append((time.time(), parts))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self, t0: float, t1: float):
        sel = [p for (t, p) in self.samples if t0 <= t <= t1]
        if len(sel) < 3:
            sel = [p for (t, p) in self.samples if t >= t0 - 5]
        if not sel:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(p[0]) for p in sel if p[0].replace(".", "").isdigit()]
        mx = [float(p[1]) for p in sel if p[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for p in sel for i in range(4) if p[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sel)}


# ------------------------------------------------------------------------------------ roofline
def phase_model(st: dict, cfg, R: int, K: int, J: int, rows: int, nnz: int, m: np.ndarray, Ik: np.ndarray):
    """Algorithmic bytes / flops per launch of each phase, from SURVEY.md §8(d):

      B_X   = 12 nnz + 4 sum I_k + 8 (K+1)        CSR bytes (int32 col + f64 val, int32 row ptr, int64 patient ptr)
      C     = 8 sum_k I_k l'_k                    the basis C_k (smooth), read once per pass
      U     = 8 R sum_k min(m_k, R)               one pass over the per-patient state (P', Q~ or N)
      B_iter = 2 B_X + 4 U + 2 C + 5 (8 K R)      the fused two-pass minimum of §8(d)

    assigned per kernel of this build: pass A (spmm) B_X + C + U (P' write) + V; polar 2U + W;
    W pass 3U + 4 (8KR) (Q~, P' read, N write, W/D_W read+write); pass B (scatter) B_X + C + U (N
    read) + F_V partial; solves O(JR). The layout's own bytes (projected fibers, padded state rows)
    are reported beside them as layout_bytes. Flops: §8(d)'s 2 nnz R + 2 R sum I_k l'_k per
    sparse pass; polar = the QR + Jacobi count of DESIGN.md §4."""
    S, F = st["state_rows"], st["fibers"]
    l = cfg.smooth_l
    q = np.minimum(m, R).astype(np.float64)
    mm = m.astype(np.float64)
    BX = 12.0 * nnz + 4.0 * rows + 8.0 * (K + 1)
    C = 8.0 * float(np.sum(Ik.astype(np.float64) * mm)) if l > 0 else 0.0
    U = 8.0 * R * float(np.sum(q))
    KR8, JR8 = 8.0 * K * R, 8.0 * J * R
    pass_flops = 2.0 * nnz * R + (2.0 * R * float(np.sum(Ik.astype(np.float64) * mm)) if l > 0 else 0.0)
    SR8 = 8.0 * S * R
    stream = F * (4 + 8 * l) + 16.0 * (K + 1) + 4.0 * K if l > 0 else 12.0 * nnz + 8.0 * (rows + 1)
    polar_flops = float(np.sum(2 * mm * R * R + 6 * np.maximum(mm, R) * q * q + 5 * 7 * q ** 3 + 2 * q ** 3
                               + 2 * mm * R * q))
    model = {
        "spmm": {"bytes": BX + C + U + JR8, "layout_bytes": stream + SR8 + JR8, "flops": pass_flops, "bound": "hbm"},
        "polar": {"bytes": 2 * U + KR8, "layout_bytes": 2 * SR8 + KR8, "flops": polar_flops, "bound": "alu"},
        "fh": {"bytes": 2 * U + KR8, "layout_bytes": 2 * SR8 + KR8, "flops": 2.0 * S * R * R, "bound": "hbm"},
        "passB1": {"bytes": 3 * U + 4 * KR8, "layout_bytes": 3 * SR8 + 4 * KR8, "flops": float(np.sum(4 * mm * R * R)),
                   "bound": "hbm"},
        "grams_B": {"bytes": U + KR8, "layout_bytes": SR8 + KR8, "flops": 2.0 * (S + K) * R * R, "bound": "hbm"},
        "scatter": {"bytes": BX + C + U + JR8, "layout_bytes": stream + SR8 + JR8, "flops": pass_flops,
                    "bound": "hbm"},
        "admm_V": {"bytes": 4 * JR8, "layout_bytes": 4 * JR8, "flops": 0.0, "bound": "hbm"},
        "fit": {"bytes": 3 * JR8, "layout_bytes": 3 * JR8, "flops": 0.0, "bound": "hbm"},
        "admm_H": {"bytes": 0.0, "layout_bytes": 0.0, "flops": 0.0, "bound": "hbm"},
    }
    # DMMA instructions the fiber passes issue (m8n8k4: 512 flops each, padding included): pass A one
    # k-step per 4 fibers per (M tile, N tile); pass B KS k-steps per 8-slot tile per N tile
    if l > 0:
        nt, mt, ks = (R + 7) // 8, (l + 7) // 8, (l + 3) // 4
        model["spmm"]["dmma"] = float(F) / 4.0 * mt * nt
        model["scatter"]["dmma"] = float(st.get("tiles", 0)) * ks * nt
    b_iter = 2 * BX + 4 * U + 2 * C + 5 * KR8
    return model, b_iter


def load_traffic():
    """dram bytes per launch from the committed ncu --set full summaries (profiles/*traffic*.json)."""
    import glob
    out = {}
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*traffic*.json"))):
        try:
            with open(f) as fh:
                out.update({k: v for k, v in json.load(fh).items() if not k.startswith("_")})
        except Exception:  # noqa: BLE001
            pass
    return out


# ------------------------------------------------------------------------------------ CPU oracle
def host_cpu():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:  # noqa: BLE001
        pass
    return os.cpu_count() or 1, model


def oracle_sample(cfg, iters: int = 1, warm: int = 0):
    """The oracle as it stands, on all host cores (oracle/sharded.py: one serial C oracle per process
    over nnz-balanced patient shards), on the first n patients of the same workload. Returns
    (nnz/s, seconds per iteration, description)."""
    from oracle.sharded import ShardedOracle
    cores, model = host_cpu()
    n = min(cfg.K, ORACLE_PER_CORE[cfg.name] * cores * SAMPLE_SCALE)
    so = ShardedOracle(cfg, procs=cores, K=n)
    try:
        if warm:
            so.iterate(warm)
        t0 = time.perf_counter()
        so.iterate(iters)
        sec = (time.perf_counter() - t0) / iters
    finally:
        so.close()
    desc = (f"first {n} of {cfg.K} patients ({so.nnz} nnz) of the same workload; {iters} outer iteration(s) of the "
            f"serial C oracle in {len(so.bounds)} processes (one per host core, nnz-balanced patient shards, "
            f"fixed-order sums); host: {cores} cores, {model}")
    return so.nnz / sec, sec, desc, cores


def config_line(cfg, world: int, total_nnz: int):
    big = 12 * total_nnz > 4 * 126e6
    return {"workload": cfg.baseline, "name": cfg.name, "K": cfg.K, "nnz": total_nnz, "R": cfg.R,
            "parallelism": f"patients sharded nnz-balanced over {world} GPU(s)",
            "l2": "inputs far larger than L2 (no flush)" if big else
                  "inputs fit in L2 and stay resident between iterations (no flush; the workload is that small)"}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    cfg = synthgen.CONFIGS[args.config]
    from oracle.sharded import ShardedOracle
    cores, model = host_cpu()
    n = min(cfg.K, ORACLE_PER_CORE[cfg.name] * cores * SAMPLE_SCALE)
    so = ShardedOracle(cfg, procs=cores, K=n)
    try:
        so.iterate(args.warmup)
        t0 = time.perf_counter()
        so.iterate(args.steps)
        sec = (time.perf_counter() - t0) / args.steps
    finally:
        so.close()
    value = so.nnz / sec
    sample = (f"each step = one outer iteration over the first {n} of {cfg.K} patients ({so.nnz} nnz) of the same "
              f"workload; serial C oracle in {len(so.bounds)} processes (one per host core); host: {cores} cores, "
              f"{model}")
    total_nnz = int(synthgen.patient_nnz(cfg).sum()) if cfg.K <= 4_000_000 else so.nnz
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded synthgen, BASELINE.json recipe)",
            "config": config_line(cfg, world, total_nnz),
            "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------ ours
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist
    import paper_1803_04572_b200 as copa

    copa.lib()  # fail loudly if the CUDA extension is missing
    torch.cuda.set_device(local_rank)
    cfg = synthgen.CONFIGS[args.config]
    if world > 1:
        nnz_k = synthgen.patient_nnz(cfg)
        b = synthgen.shard_bounds(nnz_k, world)
        k0, k1 = int(b[rank]), int(b[rank + 1])
        total_nnz = int(nnz_k.sum())
    else:
        k0, k1 = 0, cfg.K
    prob = synthgen.generate(cfg, k_range=(k0, k1))
    if world == 1:
        total_nnz = prob.nnz
    opts = copa.Options.from_config(cfg)
    allreduce = copa.torch_allreduce() if world > 1 else None

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler(local_rank if os.environ.get("CUDA_VISIBLE_DEVICES") is None else
                          int(os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local_rank]))
    t_init0 = time.perf_counter()
    g = copa.Copa(prob, opts, K_global=cfg.K, allreduce=allreduce)
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t_init0
    stream = g.stream
    if args.warmup > 0:
        g.iterate_async(args.warmup)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    tw0 = time.time()
    e0.record(stream)
    g.iterate_async(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    tw1 = time.time()
    barrier()
    ms_local = e0.elapsed_time(e1)
    ms = max_over_ranks(ms_local)
    ms_per_step = ms / args.steps
    # phase breakdown: a second, profiled pass of K iterations (CUDA event pairs around every phase on
    # the library stream; eager launches, so single-rank runs lose the CUDA-graph replay there). The
    # headline value above is the unprofiled pass.
    g.set_profiling(True)
    g.iterate_async(args.steps)
    phases = g.phase_times()
    g.set_profiling(False)
    launches = phases.pop("_launches")
    st = g.stats()
    fit_last = st["fit"]
    clk = clocks.summary(tw0, tw1)
    m = g.debug_state()["m"].cpu().numpy() if g.K > 0 else np.zeros(0, np.int32)
    Ik = np.diff(prob.patient_row_ptr)
    model, b_iter = phase_model(st, cfg, g.R, g.K, g.J, g.rows, g.nnz, m, Ik)
    value = total_nnz * args.steps / (ms / 1e3)
    hbm_peak, hbm_src = peaks()

    # dominant phase (largest share of the step) and its roofline
    per_launch = {k: (v[0] / max(v[1], 1), v[1]) for k, v in phases.items() if v[1] > 0}
    dom = max(per_launch, key=lambda k: per_launch[k][0]) if per_launch else None
    roof = None
    if dom is not None:
        ms_launch = per_launch[dom][0]
        mdl = model.get(dom, {"bytes": 0, "flops": 0, "bound": "hbm"})
        traffic = load_traffic().get(f"{args.config}:{dom}")
        if mdl["bound"] == "alu":
            ach = mdl["flops"] / (ms_launch / 1e3) / 1e12
            roof = {"kernel": dom, "bound": "alu", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                    "frac": ach / FP64_PEAK_TFLOPS, "traffic": traffic, "peak_source": "measured DFMA loop (FP64)",
                    "ms_per_launch": ms_launch}
        else:
            ach = mdl["bytes"] / (ms_launch / 1e3) / 1e9
            roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                    "frac": ach / hbm_peak, "traffic": traffic, "peak_source": hbm_src, "ms_per_launch": ms_launch,
                    "alg_bytes": mdl["bytes"], "bytes_source": "SURVEY.md 8(d): B_X + C + U + 8JR per sparse pass",
                    "layout_bytes": mdl["layout_bytes"],
                    "layout_frac": mdl["layout_bytes"] / (ms_launch / 1e3) / 1e9 / hbm_peak}
            if mdl["flops"] > 0:  # the fiber passes also sit at the FP64 tensor-core (DMMA) ridge
                tf = mdl["flops"] / (ms_launch / 1e3) / 1e12
                roof["fp64_tensor"] = {"achieved": tf, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                                       "frac": tf / DMMA_PEAK_TFLOPS,
                                       "flops": "SURVEY 8(d): 2 nnz R + 2 R sum I_k l'_k per pass"}
                if mdl.get("dmma"):  # what the tensor pipe actually issues (padded tiles), vs its peak
                    ex = mdl["dmma"] * 512.0 / (ms_launch / 1e3) / 1e12
                    roof["fp64_tensor"].update({"executed_dmma": mdl["dmma"], "executed": ex,
                                                "executed_frac": ex / DMMA_PEAK_TFLOPS})
    phase_report = {k: {"ms_per_launch": per_launch[k][0], "share": per_launch[k][0] / ms_per_step,
                        "alg_GBps": (model[k]["bytes"] / (per_launch[k][0] / 1e3) / 1e9) if k in model else None,
                        "alg_frac": (model[k]["bytes"] / (per_launch[k][0] / 1e3) / 1e9 / hbm_peak) if k in model
                        else None}
                    for k in per_launch}

    # ---------------------------------------------------------------- end to end (host buffers)
    e2e = None
    if not args.no_e2e:
        del g
        torch.cuda.empty_cache()

        def pin(a):
            return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

        hp = synthgen.Problem(prob.cfg, prob.k0, prob.k1, pin(prob.patient_row_ptr), pin(prob.row_ptr),
                              pin(prob.col), pin(prob.val), pin(prob.times), pin(prob.H0), pin(prob.V0), pin(prob.W0))
        wsb = copa.fit_workspace_bytes(hp, opts)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fits, H, V, W = copa.fit_host(hp, opts, args.steps, workspace=ws, allreduce=allreduce)
        torch.cuda.synchronize()
        e2e_s = max_over_ranks(time.perf_counter() - t0)
        h2d = (hp.patient_row_ptr.nbytes + hp.row_ptr.nbytes + hp.col.nbytes + hp.val.nbytes +
               (hp.times.nbytes if hp.times is not None else 0) + 8 * cfg.R * cfg.R + hp.V0.nbytes + hp.W0.nbytes)
        d2h = 8 * (cfg.R * cfg.R + cfg.J * cfg.R + prob.K * cfg.R + args.steps)
        e2e = {"value": total_nnz * args.steps / e2e_s, "unit": "nnz/s",
               "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
               "seconds": e2e_s, "what": f"copa_fit(host CSR, n_outer={args.steps}): H2D + init (basis, fibers) "
                                         f"+ {args.steps} iterations + D2H factors"}
        del ws
        torch.cuda.empty_cache()

    # ---------------------------------------------------------------- CPU oracle baseline
    cpu = None
    clocks.stop()
    if rank == 0 and not args.no_cpu_baseline:  # after the timed region; other ranks wait at the barrier
        v, sec, desc, cores = oracle_sample(cfg)
        cpu = {"value": v, "unit": "nnz/s", "cores": cores, "kind": "oracle", "sample": desc,
               "sec_per_iter": sec}
    barrier()

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded synthgen, BASELINE.json recipe)",
            "config": config_line(cfg, world, total_nnz),
            "sec_per_iter": ms_per_step / 1e3,
            "iteration_alg_GBps": b_iter * world / (ms_per_step / 1e3) / 1e9,
            "iteration_alg_frac": b_iter * world / (ms_per_step / 1e3) / 1e9 / hbm_peak / world,
            "roofline": roof, "phases": phase_report, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk, "fit_last": fit_last, "init_s": init_s,
        }
        print(json.dumps(line), flush=True)


def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # not launched by torchrun: start one rank per GPU ourselves (same contract as the driver's launch)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
