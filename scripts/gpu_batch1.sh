#!/bin/bash
# tests + A/B of the in-tree build against build_variants/libswamp_gpu_head.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -2
for r in 1 2; do
  TAG=new timeout 300 python scripts/ab_time.py | tail -1
  TAG=head SWAMP_GPU_LIB=$PWD/build_variants/libswamp_gpu_head.so timeout 300 python scripts/ab_time.py | tail -1
done
TAG=new timeout 300 python scripts/k3_probe_b2b.py 2>/dev/null | head -1
TAG=head SWAMP_GPU_LIB=$PWD/build_variants/libswamp_gpu_head.so timeout 300 python scripts/k3_probe_b2b.py 2>/dev/null | head -1
timeout 300 python scripts/part_overhead.py | tee gpurun_out/r2g_part_overhead.json
SWAMP_GPU_LIB=$PWD/build_variants/libswamp_gpu_head.so timeout 300 python scripts/part_overhead.py
SWAMP_GPU_LIB=$PWD/build_variants/libswamp_gpu_phaset.so timeout 300 python scripts/fv1_phases.py
