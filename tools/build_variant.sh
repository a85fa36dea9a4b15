#!/bin/bash
# Build the current tree's CUDA library under another name (A/B runs): tools/build_variant.sh <name> [nvcc flags]
N=$1; shift
cd "$(dirname "$0")/.." && S=paper_2006_09299_b200/csrc
nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared -Iinclude "$@" \
  $S/kernels.cu $S/api.cu $S/scan.cu $S/generate.cu $S/strips.cu $S/filter.cu $S/pbm.cu $S/into.cu $S/pack.cu $S/strips_multi.cu \
  -o paper_2006_09299_b200/librunlab_gpu_$N.so
