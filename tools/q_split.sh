#!/bin/bash
# GPU-box helper: the thread/warp split of the small-rank polar (COPA_POLAR_SPLIT, read at init) on
# the plain workloads: the -m gpu suite without the full-size tests, then bench lines per split value.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -rs --deselect tests/test_gpu_fullsize.py > gpurun_out/split_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/split_pytest.log
for s in ${SPLITS:-100000 0 8 16 24 32 48 64}; do
  COPA_POLAR_SPLIT=$s timeout 600 python bench.py --config small --steps 50 --warmup 5 --no-e2e --no-cpu-baseline \
    > gpurun_out/split_small_$s.json 2> gpurun_out/split_small_$s.err
done
for s in 100000 0 8 16; do
  COPA_POLAR_SPLIT=$s timeout 600 python bench.py --config tiny --steps 50 --warmup 5 --no-e2e --no-cpu-baseline \
    > gpurun_out/split_tiny_$s.json 2> gpurun_out/split_tiny_$s.err
done
timeout 900 python bench.py --config large_plain --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/split_large_plain.json 2> gpurun_out/split_large_plain.err
python - <<'EOF' > gpurun_out/split_summary.txt
import glob, json
for f in sorted(glob.glob("gpurun_out/split_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        ph = d.get("phases", {})
        print(f, "ms/iter %.4f" % d["ms_per_step"], " ".join("%s=%.3f" % (k, v["ms_per_launch"]) for k, v in ph.items()))
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
EOF
true
