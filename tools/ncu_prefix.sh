#!/bin/bash
# GPU-box helper: ncu --set full of kernel $KERNEL on a prefix run (tools/run_prefix.py $CONFIG $K).
mkdir -p gpurun_out
OUT=${OUT:-ncu_prefix}
ncu --set full --import-source on --clock-control none -k "regex:${KERNEL}" -s ${SKIP:-1} -c 1 \
    -o gpurun_out/${OUT} -f python tools/run_prefix.py ${CONFIG} ${K:-50000} 2 > gpurun_out/${OUT}.log 2>&1
ncu -i gpurun_out/${OUT}.ncu-rep --page details --csv > gpurun_out/${OUT}_details.csv 2>/dev/null
ncu -i gpurun_out/${OUT}.ncu-rep --page raw --csv > gpurun_out/${OUT}_raw.csv 2>/dev/null
ncu -i gpurun_out/${OUT}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${OUT}_src.csv 2>/dev/null
rm -f gpurun_out/${OUT}.ncu-rep
