#!/bin/bash
# GPU-box helper: one `ncu --set full` capture of kernel $KERNEL in `bench.py --config $CONFIG`,
# exported as details / raw / source CSVs under gpurun_out/ (prefix $OUT).
mkdir -p gpurun_out
OUT=${OUT:-ncu}
ncu --set full --import-source on --clock-control none -k "regex:^${KERNEL}$" -s ${SKIP:-0} -c ${COUNT:-1} \
    -o gpurun_out/${OUT} -f python bench.py --config ${CONFIG:-scale} --steps 1 --warmup 1 --no-e2e \
    --no-cpu-baseline > gpurun_out/${OUT}.log 2>&1
ncu -i gpurun_out/${OUT}.ncu-rep --page details --csv > gpurun_out/${OUT}_details.csv 2>/dev/null
ncu -i gpurun_out/${OUT}.ncu-rep --page raw --csv > gpurun_out/${OUT}_raw.csv 2>/dev/null
ncu -i gpurun_out/${OUT}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${OUT}_src.csv 2>/dev/null
rm -f gpurun_out/${OUT}.ncu-rep
