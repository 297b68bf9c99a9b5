#!/bin/bash
# GPU-box helper (round 2 profiles): launch list of the default bench command (per-launch
# gpu__time_duration, cold-cache serialised), plus full captures of the top kernels.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_r02.log 2>&1
KERNEL=k_polar_wide CONFIG=scale OUT=r02_scale_polar bash tools/ncu_kernel.sh
KERNEL=k_passA CONFIG=scale OUT=r02_scale_passA bash tools/ncu_kernel.sh
KERNEL=k_passB_wide CONFIG=scale OUT=r02_scale_passBw bash tools/ncu_kernel.sh
