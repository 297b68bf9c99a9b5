#!/bin/bash
# GPU-box helper: compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over tools/sanitize_run.py.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize.status
done
