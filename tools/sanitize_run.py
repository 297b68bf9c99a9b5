"""Small runs of every kernel family through the C ABI, for compute-sanitizer (tools/sanitize.sh)."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synthgen  # noqa: E402
import paper_1803_04572_b200 as copa  # noqa: E402

CASES = [("tiny", None), ("small", 1500), ("medium", 1500), ("large", 400), ("large_plain", 200),
         ("scale", 1500)]
for name, K in CASES[:int(os.environ.get("NCASES", len(CASES)))]:
    p = synthgen.generate(name, K=K)
    g = copa.Copa(p, copa.Options.from_config(p.cfg))
    f = g.iterate(2)
    U = g.U()
    st = g.stats()
    g.close()
    print(name, f, float(np.abs(U.cpu().numpy()).max()), st["rank_deficient"], flush=True)
