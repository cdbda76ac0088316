#!/bin/bash
# Build an A/B variant of the extension with extra -D flags:
#   bash tools/build_variant.sh TAG -DEG_FAR_MINB=4 ...   -> paper_1111_3297_b200/liberato_gpu_TAG.so
# then time it with: VARIANTS="ERATO_GPU_SO=paper_1111_3297_b200/liberato_gpu_TAG.so" bash tools/ab.sh
set -e
tag=$1; shift
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  "$@" -o paper_1111_3297_b200/liberato_gpu_$tag.so paper_1111_3297_b200/csrc/erato_gpu.cu
echo paper_1111_3297_b200/liberato_gpu_$tag.so
