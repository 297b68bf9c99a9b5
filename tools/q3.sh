#!/bin/bash
# GPU-box helper: suite, phase tables, and the warp-polar experiment on the small-R workloads.
mkdir -p gpurun_out
bash tools/q2.sh
COPA_POLAR_WARP=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_n3.py -m gpu -q -x -s \
  -k "small or tiny" > gpurun_out/q3_pytest_pw.log 2>&1
echo "pytest rc=$?" >> gpurun_out/q3_pytest_pw.log
for c in small tiny small_unconstrained; do
  timeout 300 bash tools/phases.sh $c 20 COPA_POLAR_WARP=1 >> gpurun_out/q3_phases_pw.txt 2>&1
done
true
