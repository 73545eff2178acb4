#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "c2r_engine" > gpurun_out/pytest_fused.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_fused.log
grep -q " passed" gpurun_out/pytest_fused.log || exit 1
VARIANTS="XC_FUSED=0;XC_FUSED_LAG=2;XC_FUSED_LAG=6;XC_FUSED_CW=32 XC_FUSED_LAG=2;XC_FUSED_CW=32 XC_FUSED_LAG=3;XC_FUSED_LAG=4 XC_FUSED_CTAS=110" bash tools/gpu_iter.sh
