import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import torch, synthgen, oracle
import paper_1803_04572_b200 as copa
def rel(a,b): return np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-300)
for name,K in [('tiny',None),('small',2000),('medium',2000),('large',500),('scale',2000)]:
    p = synthgen.generate(name, K=K)
    try:
        g = copa.Copa(p, copa.Options.from_config(p.cfg))
        fg = g.iterate(1)
    except Exception as e:
        print(name, 'ERR', e); continue
    o = oracle.Oracle(p); fo = o.iterate(1)
    H,V,W = [t.cpu().numpy() for t in g.factors()]
    print(name, 'fit', fg[0], fo[0], 'H', rel(H,o.H), 'V', rel(V,o.V), 'W', rel(W,o.W), 'U', rel(g.U().cpu().numpy(), o.U_all()), g.stats())
