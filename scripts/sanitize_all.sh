mkdir -p gpurun_out/san
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 600 $CS --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py 6 > gpurun_out/san/${TAG:-r2k}_memcheck_L6.log 2>&1; echo memcheck6 $?
timeout 900 $CS --tool memcheck --error-exitcode 9 python scripts/sanitize_run.py 8 > gpurun_out/san/${TAG:-r2k}_memcheck_L8.log 2>&1; echo memcheck8 $?
timeout 900 $CS --tool racecheck --error-exitcode 9 python scripts/sanitize_run.py 7 > gpurun_out/san/${TAG:-r2k}_racecheck_L7.log 2>&1; echo racecheck7 $?
timeout 900 $CS --tool synccheck --error-exitcode 9 python scripts/sanitize_run.py 7 > gpurun_out/san/${TAG:-r2k}_synccheck_L7.log 2>&1; echo synccheck7 $?
