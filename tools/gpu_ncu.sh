#!/bin/bash
# ncu captures of the apply kernels (run after the same command exited 0).
# usage: tools/gpu_ncu.sh <name> <kernel regex> <count> [bench args...]
NAME=$1; KRE=$2; CNT=$3; shift 3
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline $*"
$CMD > gpurun_out/plain_$NAME.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_$NAME.log; exit 1; }
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "xc_apply/" -k regex:"$KRE" -c $CNT -o gpurun_out/prof_$NAME -f $CMD > gpurun_out/ncu_$NAME.log 2>&1
tail -2 gpurun_out/ncu_$NAME.log
