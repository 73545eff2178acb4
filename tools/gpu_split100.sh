#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "c2r_engine" > gpurun_out/pytest_s.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_s.log
for c in c5 c5n32k c5n128k c3; do VARIANTS="XC_C2R_NOBIG100=1" bash tools/gpu_iter.sh --config $c | grep -v "bench rc"; done
