#!/bin/bash
# A/B: build_variants/*.so against the in-tree library, same box, alternating.
# TESTS=0 skips the parity tests.
if [ "${TESTS:-1}" = "1" ]; then
  timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -2
fi
for rep in 1 2; do
  for lib in build_variants/*.so paper_2206_05761_b200/libswamp_gpu.so; do
    TAG=$(basename $lib) SWAMP_GPU_LIB=$PWD/$lib timeout 300 python scripts/ab_time.py 2>&1 | tail -1
  done
done
