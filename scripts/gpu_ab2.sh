#!/bin/bash
# parity (fast) + A/B against build_variants/libswamp_gpu_head.so
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -2
for r in 1 2; do
  TAG=new timeout 300 python scripts/ab_time.py | tail -1
  TAG=head SWAMP_GPU_LIB=$PWD/build_variants/libswamp_gpu_head.so timeout 300 python scripts/ab_time.py | tail -1
done
