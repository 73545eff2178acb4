#!/bin/bash
# c3 / c1 launch lists and bench lines (round-2 small/medium config look)
mkdir -p gpurun_out
for cfg in c3 c1; do
  timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/b_$cfg.json 2> gpurun_out/b_$cfg.err; echo "bench $cfg rc=$?"
  python -c "
import json;d=json.load(open('gpurun_out/b_$cfg.json'));r=d['roofline'];print('$cfg','%.0f/s'%d['value'],'ms %.4f'%d['ms_per_step'],'spmm %.4f fft %.4f frac %.3f'%(r['spmm_ms'],r['fft_ms'],r['frac']), 'launches', d['gpu_launches'])"
  CMD="python bench.py --config $cfg --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --nvtx --nvtx-include "xc_apply/" --csv --log-file gpurun_out/launches_$cfg.csv $CMD > gpurun_out/ncu_$cfg.log 2>&1; echo "ncu rc=$?"
  python tools/launches.py gpurun_out/launches_$cfg.csv 9 | tail -30
done
