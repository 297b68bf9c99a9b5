#!/bin/bash
# GPU-box helper: the -m gpu suite (minus the full-size file), then phase tables of the workloads.
mkdir -p gpurun_out
OUT=${OUT:-q2}
timeout 1500 python -m pytest tests -m gpu -q -x -s --deselect tests/test_gpu_fullsize.py ${PYTEST_K:+-k "$PYTEST_K"} \
  > gpurun_out/${OUT}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${OUT}_pytest.log
for c in ${CONFIGS:-small tiny medium large scale large_plain}; do
  st=20; [ $c = large_plain ] && st=3
  timeout 600 bash tools/phases.sh $c $st >> gpurun_out/${OUT}_phases.txt 2>&1
done
true
