"""Runs copa_init once (for profiling the init kernels)."""
import sys
import torch
sys.path.insert(0, ".")
import synthgen
from paper_1803_04572_b200 import copa
name = sys.argv[1] if len(sys.argv) > 1 else "scale"
p = synthgen.generate(synthgen.CONFIGS[name])
g = copa.Copa(p, copa.Options.from_config(p.cfg))
torch.cuda.synchronize()
print("init ok")
