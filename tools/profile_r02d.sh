#!/bin/bash
# GPU-box helper (round 2, session 3 final state): the full -m gpu suite (full-size parity included),
# the default bench line and its launch list, ncu captures of the kernels changed this session
# (plain path), then bench lines of every workload.
mkdir -p gpurun_out
{ nproc; lscpu | grep -i "model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > gpurun_out/p5_host.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -q -x -rs -s > gpurun_out/p5_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/p5_pytest_gpu.log
python bench.py --steps 20 --warmup 3 > gpurun_out/p5_bench_scale.json 2> gpurun_out/p5_bench_scale.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p5_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/p5_ncu_launch.log 2>&1
KERNEL=k_passB_warp CONFIG=small OUT=p5_k_passB_warp_small bash tools/ncu_kernel.sh
KERNEL=k_gram_mma CONFIG=large_plain OUT=p5_k_gram_mma_large_plain bash tools/ncu_kernel.sh
KERNEL=k_polar_warp CONFIG=large_plain OUT=p5_k_polar_warp_large_plain timeout 900 bash tools/ncu_kernel.sh
for c in medium large tiny small large_plain small_unconstrained medium_l33; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/p5_bench_$c.json 2> gpurun_out/p5_bench_$c.err
done
true
