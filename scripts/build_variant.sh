#!/bin/bash
# Build an A/B variant of the library with extra nvcc flags into build_variants/libswamp_gpu_<name>.so
# usage: bash scripts/build_variant.sh <name> "-DFOO -DBAR=2"
set -e
cd "$(dirname "$0")/.."
mkdir -p build_variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++20 \
  -Xcompiler -fPIC -shared $2 -I include -o build_variants/libswamp_gpu_$1.so \
  paper_2206_05761_b200/csrc/swamp_gpu.cu paper_2206_05761_b200/csrc/swamp_io.cpp
echo build_variants/libswamp_gpu_$1.so
