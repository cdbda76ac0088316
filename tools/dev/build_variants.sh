#!/bin/bash
# build tuning variants: tools/dev/build_variants.sh NAME "-DFOO=1 ..." ...
set -e
cd "$(dirname "$0")/../.."
mkdir -p build_var
while [ $# -gt 1 ]; do
  name=$1; defs=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC $defs \
    -o build_var/liberato_gpu_$name.so paper_1111_3297_b200/csrc/erato_gpu.cu &
done
wait
ls build_var
