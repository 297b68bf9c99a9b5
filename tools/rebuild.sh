#!/bin/bash
# Rebuild only the changed objects of libcopa.so (the full build is __graft_entry__.build()).
set -e
cd "$(dirname "$0")/../paper_1803_04572_b200"
mkdir -p build
pids=()
for f in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I ../include --split-compile=0 -c csrc/$f.cu -o build/$f.cu.o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libcopa.so build/*.o
echo rebuilt
