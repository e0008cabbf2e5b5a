#!/bin/bash
# A/B: build_variants/*.so against the in-tree library, same box, alternating
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_near.py -x -q 2>&1 | tail -2
for rep in 1 2; do
  for lib in build_variants/*.so paper_2206_05761_b200/libswamp_gpu.so; do
    TAG=$(basename $lib) SWAMP_GPU_LIB=$PWD/$lib timeout 300 python scripts/ab_time.py 2>/dev/null
  done
  TAG=intree_notiles SWAMP_FV1_TILES=0 timeout 300 python scripts/ab_time.py 2>/dev/null
done
