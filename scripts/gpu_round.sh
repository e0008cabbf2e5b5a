#!/bin/bash
# One GPU session: smoke, GPU tests (fast + slow), bench, bench --impl reference,
# ncu launch list + full capture of the step kernels, racecheck.
# Usage (from the repo root, under gpurun): bash scripts/gpu_round.sh [tag] [skip-slow]
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_gpu.txt
nproc > gpurun_out/${TAG}_nproc.txt; lscpu | head -20 >> gpurun_out/${TAG}_nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
tail -2 gpurun_out/${TAG}_pytest_gpu.log
if [ "${2:-}" != "skip-slow" ]; then
  timeout 1200 python -m pytest tests -m slow -x -q --durations=10 > gpurun_out/${TAG}_pytest_slow.log 2>&1
  tail -2 gpurun_out/${TAG}_pytest_slow.log
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -2 gpurun_out/${TAG}_bench.err
timeout 900 python scripts/cpu_baselines.py > gpurun_out/${TAG}_cpu_baselines.json 2> gpurun_out/${TAG}_cpu_baselines.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 5 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu --no-sims --no-wet > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fv1|k_encode|k_band|k_traverse" -s 20 -c 5 \
    -o gpurun_out/${TAG}_prof python bench.py --steps 3 --warmup 3 --no-cpu --no-sims --no-wet > gpurun_out/${TAG}_ncu_full.log 2>&1
timeout 600 python scripts/part_overhead.py > gpurun_out/${TAG}_part_overhead.json 2>&1
timeout 600 python scripts/ab_small.py > gpurun_out/${TAG}_small.txt 2>&1
TAG=${TAG} bash scripts/sanitize_all.sh > gpurun_out/${TAG}_sanitize.txt 2>&1
ls -la gpurun_out | grep ${TAG}
