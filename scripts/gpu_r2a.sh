#!/bin/bash
# round-2 session A: fast GPU tests, the full-run parity tests, bench (no CPU leg)
TAG=${1:-r2a}
mkdir -p gpurun_out
nproc > gpurun_out/${TAG}_nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q --durations=15 > gpurun_out/${TAG}_pytest_gpu.log 2>&1
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-sims > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -2 gpurun_out/${TAG}_bench.err
timeout 1800 python -m pytest tests -m slow -x -q --durations=15 > gpurun_out/${TAG}_pytest_slow.log 2>&1
tail -3 gpurun_out/${TAG}_pytest_slow.log
