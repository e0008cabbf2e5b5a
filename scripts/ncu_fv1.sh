#!/bin/bash
# ncu --set full of one steady-state step's FV1 kernels (k_fv1_tiles + k_fv1), config 5 and the wet point
TAG=${1:-f}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fv1" -s 16 -c 2 \
    -o gpurun_out/${TAG}_c5 python bench.py --steps 3 --warmup 3 --no-cpu --no-sims --no-wet > gpurun_out/${TAG}_ncu_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fv1" -s 16 -c 2 \
    -o gpurun_out/${TAG}_wet python scripts/ab_time.py > gpurun_out/${TAG}_ncu_wet.log 2>&1
