#!/bin/bash
# Rebuild the stale objects of libcopa.so (sources or copa_internal.cuh / copa.h newer than the
# object) in parallel and relink. The full clean build is __graft_entry__.build().
set -e
cd "$(dirname "$0")/../paper_1803_04572_b200"
mkdir -p build
pids=()
for src in csrc/*.cu; do
  f=$(basename $src .cu); o=build/$f.cu.o
  dense=0
  case $f in k_polar_l*|k_passB_*|k_init) [ csrc/k_dense.cuh -nt $o ] && dense=1 ;; esac
  if [ ! -f $o ] || [ $src -nt $o ] || [ csrc/copa_internal.cuh -nt $o ] || [ ../include/copa.h -nt $o ] || [ $dense = 1 ]; then
    echo "compiling $f"
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      -I ../include -c $src -o $o &
    pids+=($!)
  fi
done
for p in "${pids[@]}"; do wait $p; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libcopa.so build/*.o
echo rebuilt
