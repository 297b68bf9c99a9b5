#!/bin/bash
# GPU-box helper: ncu --set full captures of the four iteration kernels (one outer iteration) on
# Large and Medium with the round's final code, plus their launch lists.
mkdir -p gpurun_out
for c in medium large; do
  KERNEL='(k_passA|k_polar_wide|k_passB_wide|k_scatter_tma)' COUNT=4 CONFIG=$c OUT=p8_iter_$c timeout 1200 bash tools/ncu_kernel.sh
  rm -f gpurun_out/p8_iter_${c}_src.csv
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p8_launches_$c.csv \
      python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/p8_ncu_launch_$c.log 2>&1
done
true
