#!/bin/bash
# A/B of two builds (libxc_base.so / libxc_new.so) under an environment ($ENVV), CFGS configs, ROUNDS
mkdir -p gpurun_out
L=paper_2004_11610_b200
for r in $(seq ${ROUNDS:-2}); do
for v in base new; do
  cp $L/libxc_$v.so $L/libxc.so
  for cfg in ${CFGS:-c5}; do
    env $ENVV timeout 300 python bench.py --config $cfg --steps ${STEPS:-20} --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
    python -c "
import json;d=json.load(open('gpurun_out/ab.json'));r=d['roofline'];print('$v $cfg','%.0f/s'%d['value'],'ms %.4f'%d['ms_per_step'],'spmm %.4f fft %.4f frac %.3f'%(r['spmm_ms'],r['fft_ms'],r['frac']))" || tail -2 gpurun_out/ab.err
  done
done
done
cp $L/libxc_new.so $L/libxc.so
if [ -n "$LAUNCHES" ]; then
  env $ENVV timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "xc_apply/" --csv --log-file gpurun_out/launches_ab.csv python bench.py --config c5 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
  python tools/launches.py gpurun_out/launches_ab.csv 9 | head -12
fi
