#!/bin/bash
# GPU-box helper (round 2, session 4, final state): the full -m gpu suite (full-size parity included),
# smoke, bench lines of every workload, the launch lists of Scale and Small, and ncu captures of the
# CSC gather of the plain path (128-entry chunks, parallel chunk sum).
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x -rs -s > gpurun_out/p7_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/p7_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p7_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/p7_smoke.log
python bench.py --steps 20 --warmup 3 > gpurun_out/p7_bench_scale.json 2> gpurun_out/p7_bench_scale.err
for c in small tiny small_unconstrained large_plain medium large medium_l33; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/p7_bench_$c.json 2> gpurun_out/p7_bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p7_launches_small.csv \
    python bench.py --config small --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/p7_ncu_launch_small.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p7_launches_scale.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/p7_ncu_launch_scale.log 2>&1
KERNEL=k_scatter_csc CONFIG=small OUT=p7_k_scatter_csc_small bash tools/ncu_kernel.sh
true
