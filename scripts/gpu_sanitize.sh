#!/bin/bash
# compute-sanitizer tier: memcheck, racecheck, synccheck
# over the product kernels at L = 6-8 (default, uniform, inactive-cell and
# partitioned engines), and memcheck over the two-process (CUDA IPC) engine.
TAG=${1:-san}
mkdir -p gpurun_out
CS="compute-sanitizer --print-limit 200 --error-exitcode 9"
for L in 6 8; do
  timeout 900 $CS --tool memcheck --leak-check full python scripts/sanitize_run.py $L > gpurun_out/${TAG}_memcheck_L$L.log 2>&1; echo "memcheck L$L rc=$?"
done
timeout 1200 $CS --tool racecheck --racecheck-report all python scripts/sanitize_run.py 7 > gpurun_out/${TAG}_racecheck_L7.log 2>&1; echo "racecheck rc=$?"
timeout 1200 $CS --tool synccheck python scripts/sanitize_run.py 7 > gpurun_out/${TAG}_synccheck_L7.log 2>&1; echo "synccheck rc=$?"
timeout 900 $CS --tool memcheck --target-processes all python -m pytest tests/test_gpu_ranks.py -x -q > gpurun_out/${TAG}_memcheck_ranks.log 2>&1; echo "memcheck ranks rc=$?"
for f in gpurun_out/${TAG}_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY|passed|failed" $f | tail -4; done
