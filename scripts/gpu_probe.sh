#!/bin/bash
# parity + timeline for FV1 occupancy variants + ncu of the MRA kernels
TAG=${1:-p}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for mb in 2 3 4; do echo "MINB=$mb"; SWAMP_FV1_MINB=$mb python scripts/timeline.py 11 | tail -2; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_encode|k_band|k_traverse|k_fv1" -s 20 -c 4 \
  -o gpurun_out/${TAG}_prof python bench.py --steps 3 --warmup 3 --no-cpu --no-sims > /dev/null 2>&1
