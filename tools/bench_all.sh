#!/bin/bash
# GPU-box helper: bench lines for the default workload and the other configs (gpurun_out/bench_*.json).
mkdir -p gpurun_out
TAG=${TAG:-r02}
for c in ${CONFIGS:-scale tiny small medium large large_plain small_unconstrained}; do
  extra=""
  [ "$c" != "scale" ] && extra="--no-cpu-baseline"
  timeout 900 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 $extra > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
  echo "$c rc=$?" >> gpurun_out/bench_${TAG}.status
done
