#!/bin/bash
# Quick GPU iteration: fast parity tests + bench (no CPU leg / sims) + device timeline (+ ncu full capture with NCU=1).
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-sims > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -3 gpurun_out/${TAG}_bench.err
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]);print('value',d['value'],'ms/step',d['ms_per_step'],d['stage_ms_per_step'],d['work_per_step']);w=d.get('wet_point') or {};print('wet',w.get('ms_per_step'),w.get('stage_ms_per_step'),w.get('counts'))"
SWAMP_FV1_TILES=0 timeout 600 python bench.py --no-cpu --no-sims > gpurun_out/${TAG}_bench_notiles.json 2> /dev/null
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_bench_notiles.json').read().strip().splitlines()[-1]);print('no tiles: value',d['value'],'ms/step',d['ms_per_step'],d['stage_ms_per_step']);w=d.get('wet_point') or {};print('wet',w.get('ms_per_step'),w.get('stage_ms_per_step'))"
if [ "${NCU:-0}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fv1|k_encode|k_band|k_traverse" -s 20 -c 5 \
    -o gpurun_out/${TAG}_prof python bench.py --steps 3 --warmup 3 --no-cpu --no-sims --no-wet > gpurun_out/${TAG}_ncu_full.log 2>&1
fi
