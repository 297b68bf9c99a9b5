import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import torch, synthgen
import paper_1803_04572_b200 as copa
names = sys.argv[1:] or ['medium', 'scale']
for name in names:
    t0 = time.time(); p = synthgen.generate(name); tg = time.time() - t0
    t0 = time.time(); g = copa.Copa(p, copa.Options.from_config(p.cfg)); torch.cuda.synchronize(); ti = time.time() - t0
    g.iterate(2)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    n = 3
    e0.record(); g.iterate_async(n); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{name}: K={p.K} nnz={p.nnz} gen={tg:.1f}s init={ti:.2f}s  {ms:.2f} ms/iter  {p.nnz/ms/1e6:.3f} Gnnz/s fit={g.fits[-1]:.6f} stats={g.stats()}", flush=True)
    del g; torch.cuda.empty_cache()
