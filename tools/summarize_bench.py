"""Print one line per bench JSON (ms/step, value, e2e, dominant kernel, roofline fraction, phases)."""
import glob
import json
import sys

for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    c = d.get("cpu_baseline") or {}
    print(f"{f:44s} ms/step {d['ms_per_step']:9.3f} value {d['value']:.3e} e2e {e.get('value', 0):.3e} "
          f"dom {r.get('kernel')} frac {r.get('frac', 0):.3f} launches {d.get('gpu_launches')} cpu {c.get('value')}")
    print("    ", {k: round(v["ms_per_launch"], 3) for k, v in (d.get("phases") or {}).items()})
