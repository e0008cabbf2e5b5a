#!/bin/bash
# ncu --set full of one steady-state step's FV1 kernels (k_fv1_tiles + k_fv1), config 5 and the wet point
TAG=${1:-f}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fv1" -s 10 -c 2 \
    -o gpurun_out/${TAG}_c5 python scripts/ncu_case.py river_flood 11 > gpurun_out/${TAG}_ncu_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fv1" -s 10 -c 2 \
    -o gpurun_out/${TAG}_wet python scripts/ncu_case.py monai_runup 11 > gpurun_out/${TAG}_ncu_wet.log 2>&1
