#!/bin/bash
# GPU-box helper: plain-path parity tests, then Small phase tables over the polar long-patient threshold.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -s --deselect tests/test_gpu_fullsize.py \
  -k "small or tiny or shape_sweep or large_plain or single_visit or virtual or nonneg or checkpoint or copa_fit" \
  > gpurun_out/q1_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/q1_pytest.log
COPA_POLAR_LONG_M=0 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_n3.py -m gpu -q -x -s \
  -k "small or tiny" > gpurun_out/q1_pytest_T0.log 2>&1
echo "pytest rc=$?" >> gpurun_out/q1_pytest_T0.log
for T in 100000 12 16 24 32 48; do
  timeout 300 bash tools/phases.sh small 20 COPA_POLAR_LONG_M=$T >> gpurun_out/q1_phases.txt 2>&1
done
timeout 300 bash tools/phases.sh tiny 20 >> gpurun_out/q1_phases.txt 2>&1
timeout 600 bash tools/phases.sh large_plain 3 >> gpurun_out/q1_phases.txt 2>&1
true
