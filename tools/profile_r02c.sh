#!/bin/bash
# GPU-box helper (round 2, final state): the default bench line, its launch list (per-launch
# gpu__time_duration, cold-cache serialised) and full ncu captures of the four iteration kernels
# at Scale, then bench lines of the other workloads.
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 > gpurun_out/p3_bench_scale.json 2> gpurun_out/p3_bench_scale.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p3_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/p3_ncu_launch.log 2>&1
for k in k_scatter_tma k_polar_wide k_passA k_passB_wide; do
  KERNEL=$k CONFIG=scale OUT=p3_$k bash tools/ncu_kernel.sh
done
for c in ${CONFIGS:-medium large tiny small large_plain small_unconstrained medium_l33}; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/p3_bench_$c.json 2> gpurun_out/p3_bench_$c.err
done
true
