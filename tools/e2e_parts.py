"""Breakdown of the end-to-end copa_fit time (H2D, init, iterations, D2H) at one config."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import synthgen
from paper_1803_04572_b200 import copa

name = sys.argv[1] if len(sys.argv) > 1 else "scale"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
p = synthgen.generate(synthgen.CONFIGS[name])
opts = copa.Options.from_config(p.cfg)
pin = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
hp = synthgen.Problem(p.cfg, p.k0, p.k1, pin(p.patient_row_ptr), pin(p.row_ptr), pin(p.col), pin(p.val),
                      pin(p.times), pin(p.H0), pin(p.V0), pin(p.W0))
# H2D alone (same bytes, pinned)
dev = [torch.empty(a.nbytes, dtype=torch.uint8, device="cuda") for a in (hp.col, hp.val, hp.times, hp.row_ptr)]
torch.cuda.synchronize(); t0 = time.perf_counter()
for d, a in zip(dev, (hp.col, hp.val, hp.times, hp.row_ptr)):
    d.copy_(torch.from_numpy(a.view(np.uint8).reshape(-1)), non_blocking=True)
torch.cuda.synchronize(); th = time.perf_counter() - t0
del dev
torch.cuda.empty_cache()
ws = torch.empty(copa.fit_workspace_bytes(hp, opts), dtype=torch.uint8, device="cuda")
for n in (1, steps):
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        copa.fit_host(hp, opts, n, workspace=ws)
        torch.cuda.synchronize(); t = time.perf_counter() - t0
        print(f"{name} fit_host n_outer={n}: {t:.3f} s")
print(f"{name} H2D of X (col, val, times, row_ptr) alone: {th:.3f} s")
del ws
torch.cuda.empty_cache()
# init alone from device-resident inputs (the bench's value path)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g = copa.Copa(p, opts)
    torch.cuda.synchronize(); print(f"{name} Copa(...) (H2D via torch + init): {time.perf_counter() - t0:.3f} s")
    del g
