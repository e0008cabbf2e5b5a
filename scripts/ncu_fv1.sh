#!/bin/bash
# ncu --set full of one steady-state k_fv1 launch (config 5 and the wet point), tile path on and off
TAG=${1:-f}
mkdir -p gpurun_out
for T in 1 0; do
  SWAMP_FV1_TILES=$T timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fv1" -s 8 -c 1 \
    -o gpurun_out/${TAG}_fv1_t$T python bench.py --steps 3 --warmup 3 --no-cpu --no-sims --no-wet > gpurun_out/${TAG}_ncu_t$T.log 2>&1
done
