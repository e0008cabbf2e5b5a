#!/bin/bash
# FV1 variants on config 5 and the wet point (stage times), one box
TAG=${1:-tv}
for v in "SWAMP_FV1_TILES=0" "SWAMP_FV1_TILES=1" "SWAMP_FV1_TILES=2" "SWAMP_FV1_TILES=1 SWAMP_FV1_TAIL16=10" "SWAMP_FV1_TILES=0 SWAMP_FV1_STAGE=3"; do
  env $v timeout 300 python bench.py --no-cpu --no-sims --steps 30 > gpurun_out/${TAG}.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open('gpurun_out/${TAG}.json').read().strip().splitlines()[-1]);w=d['wet_point'];print('$v'.ljust(40),'c5 %.1f us fv1 %.1f | wet %.1f us fv1 %.1f'%(d['ms_per_step']*1e3,d['stage_ms_per_step']['ms_fv1']*1e3,w['ms_per_step']*1e3,w['stage_ms_per_step']['ms_fv1']*1e3))"
done
