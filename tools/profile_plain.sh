#!/bin/bash
# GPU-box helper: launch list of the Small iteration and full ncu captures of the plain-path kernels
# (Small: polar_thread, passB_warp; large_plain: polar_warp).
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/pl_launches_small.csv \
    python bench.py --config small --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/pl_ncu_launch.log 2>&1
KERNEL=k_polar_thread CONFIG=small OUT=pl_polar_thread_small bash tools/ncu_kernel.sh
KERNEL=k_passB_warp CONFIG=small OUT=pl_passB_warp_small bash tools/ncu_kernel.sh
KERNEL=k_polar_warp CONFIG=large_plain OUT=pl_polar_warp_large_plain timeout 900 bash tools/ncu_kernel.sh
true
