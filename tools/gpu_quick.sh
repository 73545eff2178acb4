#!/bin/bash
# Quick GPU iteration: a subset of parity tests, the c5 bench line, the c5 launch list.
# usage: tools/gpu_quick.sh "<pytest -k expr>" [extra bench args]
mkdir -p gpurun_out
K="$1"; shift
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$K" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest_quick.log
fi
timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline "$@" > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"
tail -2 gpurun_out/bench_quick.err; cat gpurun_out/bench_quick.json
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline $*"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "xc_apply/" --csv --log-file gpurun_out/launches_quick.csv $CMD > gpurun_out/ncu_quick.log 2>&1; echo "ncu rc=$?"
