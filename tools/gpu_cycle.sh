#!/bin/bash
# GPU-box helper: -m gpu tests (minus the slow full-size ones unless FULL=1), then bench lines.
mkdir -p gpurun_out
sel="not fullsize"
[ "${FULL:-0}" = "1" ] && sel=""
timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q -x -rs -s ${PYTEST_ARGS} \
  $( [ -n "$sel" ] && echo "--deselect tests/test_gpu_fullsize.py" ) > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
[ "${BENCH:-1}" = "1" ] && CONFIGS="${CONFIGS:-scale small tiny large_plain}" bash tools/bench_all.sh
true
