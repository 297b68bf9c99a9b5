#!/bin/bash
# GPU-box helper (development loop): the fast parity tests of the paths a change touches
# ($TESTS, pytest -k expression), then the phase tables of $CONFIGS (tools/phases.sh).
mkdir -p gpurun_out
OUT=${OUT:-quick}
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -q -x -s ${TESTS:+-k "$TESTS"} \
  --deselect tests/test_gpu_fullsize.py > gpurun_out/${OUT}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${OUT}_pytest.log
for c in ${CONFIGS:-scale}; do
  timeout 600 bash tools/phases.sh $c ${STEPS:-10} >> gpurun_out/${OUT}_phases.txt 2>&1
done
true
