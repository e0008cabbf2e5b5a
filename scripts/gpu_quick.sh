#!/bin/bash
# Quick GPU iteration: parity tests + bench (no CPU leg) + device timeline (+ ncu full capture with NCU=1).
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-sims > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -3 gpurun_out/${TAG}_bench.err
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]);print('value',d['value'],'ms/step',d['ms_per_step'],d['stage_ms_per_step'])"
timeout 120 python scripts/timeline.py 11 2>&1 | tail -3
timeout 120 python scripts/k1_probe.py 2>&1 | tail -4
if [ "${NCU:-0}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fv1|k_encode|k_band|k_traverse" -s 20 -c 4 \
    -o gpurun_out/${TAG}_prof python bench.py --steps 3 --warmup 3 --no-cpu --no-sims > gpurun_out/${TAG}_ncu_full.log 2>&1
fi
