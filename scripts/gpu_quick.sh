#!/bin/bash
# Quick GPU iteration: parity tests + bench (no CPU leg) + ncu full capture.
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-sims > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -3 gpurun_out/${TAG}_bench.err
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fv1|k_encode|k_band|k_traverse" -s 20 -c 4 \
    -o gpurun_out/${TAG}_prof python bench.py --steps 3 --warmup 3 --no-cpu --no-sims > gpurun_out/${TAG}_ncu_full.log 2>&1
fi
