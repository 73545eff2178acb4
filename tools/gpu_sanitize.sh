#!/bin/bash
# One compute-sanitizer tool per call (B200_PROFILING.md): usage tools/gpu_sanitize.sh memcheck|racecheck|synccheck
mkdir -p gpurun_out
T=${1:-memcheck}
python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/sanitize_plain.log; exit 1; }
timeout 2400 compute-sanitizer --tool $T --print-limit 50 --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_$T.log 2>&1
echo "sanitizer $T rc=$?"
tail -30 gpurun_out/sanitize_$T.log
