#!/bin/bash
# ncu --set full of the SpMM launch of a config (default c3), after the same command ran clean.
mkdir -p gpurun_out
C=${1:-c3}
CMD="python bench.py --config $C --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain_$C.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_win -s 2 -c 1 -o gpurun_out/prof_spmm_$C $CMD > gpurun_out/ncu_spmm_$C.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_spmm_$C.log
