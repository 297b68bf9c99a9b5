#!/bin/bash
# GPU-box helper: host facts, then the -m gpu suite (output under gpurun_out/).
mkdir -p gpurun_out
{ nproc; lscpu | grep -i "model name\|^CPU(s)\|Socket\|Thread"; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > gpurun_out/host.txt 2>&1
timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q -x -rs -s ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
