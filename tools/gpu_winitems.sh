#!/bin/bash
mkdir -p gpurun_out
for c in c3 c4 c5 c2 c8; do
  VARIANTS="XC_WIN_ITEMS_A=48;XC_WIN_ITEMS_A=32;XC_WIN_ITEMS_A=24;XC_WIN_ITEMS_A=16" bash tools/gpu_iter.sh --config $c 2>&1 | grep -v "bench rc"
done
