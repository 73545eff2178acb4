#!/bin/bash
# GPU iteration: (optional) pytest subset, bench lines under env variants, launch list of the default.
# usage: PYTEST_K="expr" VARIANTS="XC_C2R_CHUNK_MB=0;XC_C2R_CHUNK_MB=20" tools/gpu_iter.sh [bench args]
mkdir -p gpurun_out
if [ -n "$PYTEST_K" ]; then
  if [ "$PYTEST_K" = "all" ]; then
    timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"
  else
    timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$PYTEST_K" > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"
  fi
  tail -4 gpurun_out/pytest_iter.log
fi
timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline "$@" > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo "bench rc=$?"
tail -2 gpurun_out/bench_iter.err; python -c "
import json;d=json.load(open('gpurun_out/bench_iter.json'));r=d['roofline'];print('DEFAULT',d['config']['workload'],'%.0f/s'%d['value'],'ms %.3f'%d['ms_per_step'],'spmm %.3f fft %.3f frac %.3f step_frac %.3f'%(r['spmm_ms'],r['fft_ms'],r['frac'],r['step_frac']), 'launches', d['gpu_launches'])"
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  [ -z "$v" ] && continue
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline "$@" > gpurun_out/bench_v.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/bench_v.json'));r=d['roofline'];print('$v','%.0f/s'%d['value'],'ms %.3f'%d['ms_per_step'],'spmm %.3f fft %.3f'%(r['spmm_ms'],r['fft_ms']))"
done
if [ -n "$LAUNCHES" ]; then
  CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline $*"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "xc_apply/" --csv --log-file gpurun_out/launches_iter.csv $CMD > gpurun_out/ncu_iter.log 2>&1; echo "ncu rc=$?"
  python tools/launches.py gpurun_out/launches_iter.csv 9 | tail -30
fi
