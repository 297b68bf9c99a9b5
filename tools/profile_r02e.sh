#!/bin/bash
# GPU-box helper (round 2, session 4): the full -m gpu suite (full-size parity included) on the code
# with the register-column plain W pass and the parallel fixed-order partial reduce, bench lines of
# every workload, the launch list of Small and an ncu capture of the changed W-pass kernel.
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x -rs -s > gpurun_out/p6_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/p6_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p6_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/p6_smoke.log
python bench.py --steps 20 --warmup 3 > gpurun_out/p6_bench_scale.json 2> gpurun_out/p6_bench_scale.err
for c in small tiny small_unconstrained medium large large_plain medium_l33; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/p6_bench_$c.json 2> gpurun_out/p6_bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p6_launches_small.csv \
    python bench.py --config small --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/p6_ncu_launch.log 2>&1
KERNEL=k_passB_warp CONFIG=small OUT=p6_k_passB_warp_small bash tools/ncu_kernel.sh
KERNEL=k_polar_thread CONFIG=small OUT=p6_k_polar_thread_small bash tools/ncu_kernel.sh
true
