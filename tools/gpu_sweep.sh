#!/bin/bash
# bench one config under environment variants: CFG=c3 VARS="A=1 B=2;C=3" tools/gpu_sweep.sh
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "$VARS"
for cfg in ${CFGS:-c3}; do
for v in "" "${VS[@]}"; do
  env $v timeout 300 python bench.py --config $cfg --steps ${STEPS:-50} --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "
import json;d=json.load(open('gpurun_out/sw.json'));r=d['roofline'];print('$cfg [$v]','%.0f/s'%d['value'],'ms %.4f'%d['ms_per_step'],'spmm %.4f fft %.4f frac %.3f'%(r['spmm_ms'],r['fft_ms'],r['frac']))" || tail -2 gpurun_out/sw.err
done
done
