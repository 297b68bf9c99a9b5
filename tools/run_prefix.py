"""One or two outer iterations of a workload prefix through the C ABI (for ncu captures of kernels
whose full-size launch is too long to replay): python tools/run_prefix.py CONFIG K [ITERS]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthgen  # noqa: E402
import paper_1803_04572_b200 as copa  # noqa: E402

name, K = sys.argv[1], int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
p = synthgen.generate(name, K=K)
g = copa.Copa(p, copa.Options.from_config(p.cfg))
print(name, K, g.iterate(iters))
