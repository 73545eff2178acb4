#!/bin/bash
# source-level stall attribution of the c1 small-path kernels
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:small_ -c 4 -o gpurun_out/c1_small -f python bench.py --config c1 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/c1_src.log 2>&1; echo ncu rc=$?
